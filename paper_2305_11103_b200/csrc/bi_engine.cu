// Native step scheduler for the 2^k-diagonal-block engine (run_inversion).
//
// Reference: /root/reference/pkg/src/blockinv/engine.py:73-162 (stepid ->
// loopid -> action), :289-446 (the three actions), storage.py:166-262,
// 391-411 (M_inv and the provisional sets T_l).
//
// B200 design:
//  * device-resident, coordinate-aligned layout: M and M_inv are padded
//    row-major n x n buffers; T_l is stored as the batch of level-l quad
//    squares (side = quad span, contiguous, ld padded to 4) with S_D at A's
//    position, R at B's, L at C's and S_A at D's -- every operand of every
//    step is a window at the same block coordinates as in M;
//  * each step is a fixed list of device ops built once at bind time:
//      diag      -> K3 batched pivoted GJ over all N_b x batch leaves
//      arrows    -> K1 launch {R=-A^-1 B, L=-D^-1 C}, K1 launch {S_D=A+B L, S_A=D+C R}
//      assemble  -> diag on T_cid S, then per pass one K1 launch {down, up}
//    GEMM descriptors of equal shape and constant pointer stride are merged
//    into strided batches; everything is uploaded once and the whole step
//    range is replayed as one CUDA graph;
//  * singular leaves are recorded per diag step on the device and resolved
//    to (step, quad, matrix) after the range (no host syncs inside it).
#include <algorithm>
#include <array>
#include <chrono>
#include <cstdio>
#include <functional>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <condition_variable>
#include <mutex>
#include <thread>
#include <tuple>
#include <vector>

#include "../../include/blockinv_b200.h"
#include "bi_common.cuh"
#include "bi_shard_internal.cuh"

namespace bi {

struct StepAct {
  int kind;  // 0 diag, 1 arrows, 2 assemble
  int from_tset;
  int cid, sid, depth;
};

static int loopid_decode(int stepid, int nblocks, StepAct* out) {
  // engine.py:77-90 (loopid) and :117-157 (decode rules)
  int width = 0;
  while ((1 << width) < nblocks) ++width;
  width += 1;
  std::vector<int> nz;
  for (int b = width - 1; b >= 0; --b)
    if ((stepid >> b) & 1) nz.push_back(b + 1);
  if (nz.empty()) return 2;
  const int last = nz.back();
  StepAct a{};
  if (nz.size() == 1) {
    a.kind = last == 1 ? 0 : 1;
    a.from_tset = 0;
    a.sid = last - 1;
  } else {
    a.cid = nz[nz.size() - 2] - 1;
    a.from_tset = 1;
    if (last == 1) {
      int run = 1;
      while (run < (int)nz.size() && nz[nz.size() - run - 1] == run + 1) ++run;
      a.kind = 2;
      a.depth = run - 1;
    } else {
      a.kind = 1;
      a.sid = last - 1;
    }
  }
  *out = a;
  return 0;
}

// Merge consecutive descriptors that differ only by a constant pointer stride.
static std::vector<GemmDesc> merge_descs(const std::vector<GemmDesc>& in) {
  std::vector<GemmDesc> out;
  for (const GemmDesc& d : in) {
    if (!out.empty()) {
      GemmDesc& p = out.back();
      const bool same = p.M == d.M && p.N == d.N && p.K == d.K && p.lda == d.lda && p.ldb == d.ldb &&
                        p.ldc == d.ldc && p.ldd == d.ldd && p.neg == d.neg && p.skip_len == d.skip_len &&
                        p.skip_at == d.skip_at && (p.C == nullptr) == (d.C == nullptr);
      if (same) {
        const int64_t dA = d.A - p.A, dB = d.B - p.B, dD = d.D - p.D, dC = d.C ? d.C - p.C : 0;
        // TMA batch strides are unsigned: keep descriptors apart rather than
        // produce a negative A/B stride (the launch would lose the TMA path)
        if (dA < 0 || dB < 0) goto no_merge;
        if (p.batch == 1) {
          p.sA = dA;
          p.sB = dB;
          p.sC = dC;
          p.sD = dD;
          p.batch = 2;
          continue;
        }
        const int64_t b = p.batch;
        if (dA == b * p.sA && dB == b * p.sB && dD == b * p.sD && dC == b * p.sC) {
          p.batch += 1;
          continue;
        }
      }
    }
  no_merge:
    GemmDesc c = d;
    c.batch = 1;
    c.sA = c.sB = c.sC = c.sD = 0;
    out.push_back(c);
  }
  return out;
}

}  // namespace bi

using namespace bi;

namespace {

struct Op {
  int kind;      // 0 = inversion group, 1 = gemm launch, 2 = copy M -> M_inv (pivot-A)
  int index;     // inv group index / gemm launch index / lane
};

struct GemmLaunchRec {
  int first, count;  // into the descriptor table
};

struct InvRec {
  InvGroup g;           // device pointers filled at bind
  int diag_step_index;  // which diag step (for info reporting)
  std::vector<int> item_block;   // block index p of each item
  std::vector<int> item_matrix;  // matrix index z of each item
  int info_offset;      // into the info region (ints)
  int lane;             // which lane (scratch region / stream)
  bool in_place = false;  // pivot-A: leaf inverted in place inside M_inv
  // host mirrors of the pointer tables (blocks above kInvMaxDirect run a host-driven recursion)
  std::vector<const double*> h_src;
  std::vector<int64_t> h_srcld;
  std::vector<double*> h_dst;
  std::vector<int64_t> h_dstld;
};

struct Window {
  double* p;
  int64_t ld;
};

struct GraphKey {
  int first, last;
  const void* in;
  const void* out;
  int64_t ld_in, s_in, ld_out, s_out;
  bool operator<(const GraphKey& o) const {
    return std::tie(first, last, in, out, ld_in, s_in, ld_out, s_out) <
           std::tie(o.first, o.last, o.in, o.out, o.ld_in, o.s_in, o.ld_out, o.s_out);
  }
};

}  // namespace

struct bi_engine {
  int nb = 0, Z = 0, k = 0, nsteps = 0;
  int schedule = 0;                  // BI_SCHEDULE_EQ7 / BI_SCHEDULE_PIVOT_A
  std::vector<int64_t> pa_depth_off;  // pivot-A: per recursion depth, T_b/T_c offset (elements)
  std::vector<int64_t> sizes, off;
  int64_t n = 0;
  // bound buffers
  const double* M = nullptr;
  int64_t ldm = 0, sm = 0;
  double* Minv = nullptr;
  int64_t ldi = 0, si = 0;
  char* ws = nullptr;
  int64_t ws_bytes = 0;
  // layout
  struct Sq {
    int64_t off, side, ld;
    int64_t col_origin;  // matrix column of the square's column 0 (the quad's first column, or
                         // this rank's first column for a column-sharded global-level quad)
    bool present;        // false: the quad holds none of this rank's columns
  };
  std::vector<std::vector<Sq>> tsq;  // [level][quad]
  int64_t t_matrix = 0;              // elements per matrix (all levels)
  int64_t t_bytes = 0, inv_scratch = 0, info_ints = 0, meta_bytes = 0;
  double* T = nullptr;
  static constexpr int kMaxLanes = 8;
  void* inv_base[kMaxLanes] = {};
  int nlanes = 1;
  int lane_priority[kMaxLanes] = {};
  int leaf_priority = 0;
  int gemm_cap = 0;  // engine GEMM grid cap (SMs left for the leaf chains)
  int skew_mode = 1;  // lane start: 0 together, 1 after lane l-1's first step, 2 after lane 0's
  struct Policy {
    int lane_priority[kMaxLanes] = {};
    int leaf_priority = 0;
    int skew = 1;
    int gemm_cap = 0;
  } pol[2];  // [0] device-resident runs, [1] runs with host read-back
  void set_policy(int i) {
    for (int l = 0; l < kMaxLanes; ++l) lane_priority[l] = pol[i].lane_priority[l];
    leaf_priority = pol[i].leaf_priority;
    skew_mode = pol[i].skew;
    gemm_cap = pol[i].gemm_cap;
  }
  int zlo[kMaxLanes] = {}, zhi[kMaxLanes] = {};
  // ---- column-sharded rank of a P-GPU run (bi_engine_create_shard).
  // P == 1: the whole matrix.  Rank r owns block columns [h0, h1) of M, M_inv
  // and every T_l; local levels (2^l <= N_b/P) need nothing from other ranks,
  // a global-level action first assembles its replicated operand X from the
  // group's column slabs (an "exchange"), then runs on this rank's columns.
  int P = 1, rank = 0, nbp = 0, h0 = 0, h1 = 0;
  int64_t col0 = 0, w = 0, wmax = 0;  // first owned column, owned width, widest rank
  int shard_flags = 0;
  struct Xchg {
    int level = 0, kind = 0;       // kind 0: arrows ([A^-1; C] / [B; D^-1]), 1: up/down pass (L / R)
    int g0 = 0, gs = 0;            // group: ranks [g0, g0 + gs)
    bool in_a = false;             // this rank's columns lie in the quad's A half
    const double* top = nullptr;   // this rank's send parts: rows x w windows
    int64_t top_ld = 0, top_rows = 0;
    const double* bot = nullptr;
    int64_t bot_ld = 0, bot_rows = 0;
    int from0 = 0, from1 = 0;      // ranks whose send parts form X (columns side by side)
    int64_t x_col0 = 0;            // matrix column of X's column 0
    int64_t rows = 0, xcols = 0, ldx = 0;
  };
  std::vector<Xchg> xchgs;
  int64_t x_elems = 0, send_elems = 0, recv_elems = 0;
  double* X = nullptr;
  double* sendbuf = nullptr;
  double* recvbuf = nullptr;
  struct FlatOp {
    int stepid;
    Op op;  // kind 3: exchange (index into xchgs)
  };
  std::vector<FlatOp> flat;         // lane 0's ops of steps 1..N_s in order
  std::vector<int> step_first_op;   // [stepid] -> first index into flat (N_s + 2 entries)
  std::map<std::pair<int, int>, cudaGraphExec_t> seg_graphs;
  std::map<int, void*> group_comms;  // NCCL transport: group size -> ncclComm_t (bi_nccl.cu)
  int device = 0;
  int* info = nullptr;
  GemmDesc* d_descs = nullptr;
  void* d_ptrs = nullptr;
  // schedule
  std::vector<std::vector<Op>> lane_ops[kMaxLanes];  // [lane][stepid]
  std::vector<GemmDesc> descs;            // host copy of the table
  std::vector<GemmLaunchRec> launches;
  std::vector<InvRec> invs;
  std::vector<int> diag_steps;            // stepids of diag actions
  bool bound = false;
  cudaStream_t last_stream = nullptr;
  cudaStream_t capture_stream = nullptr;
  cudaStream_t aux_stream[kMaxLanes] = {};  // lanes 1.. (lane 0 runs on the caller's stream)
  cudaEvent_t ev_fork = nullptr, ev_skew[kMaxLanes] = {}, ev_join[kMaxLanes] = {};
  // BI_ENGINE_TIMELINE=1: timing events after every step of every lane
  // (captured as external event-record nodes), read by bi_engine_timeline
  bool timeline = false;
  cudaEvent_t tl_start = nullptr;
  std::vector<cudaEvent_t> tl_ev;  // [lane * (nsteps + 1) + stepid]
  cudaStream_t copy_stream = nullptr;       // host->device input copies
  cudaStream_t d2h_stream[kMaxLanes] = {};  // per-lane read-back (page-locked output)
  cudaEvent_t ev_d2h_a[kMaxLanes] = {}, ev_d2h_b[kMaxLanes] = {};
  static constexpr int kOutChunks = 16;  // max row chunks of the last top-level pass, each read back at once
  cudaEvent_t ev_chunk[kMaxLanes][kOutChunks] = {};
  std::vector<cudaEvent_t> ev_h2d;          // per (matrix, level): that level's input blocks copied
  std::map<GraphKey, cudaGraphExec_t> graphs;
  int last_first = 1, last_last = 0;

  void* meta_dev = nullptr;
  int64_t meta_cap = 0;
  // page-locked staging for pageable host buffers (bi_engine_run_host):
  // [Z][n][ldm] input, [Z][n][ldi] output, allocated on first use
  double* stage_in = nullptr;
  double* stage_out = nullptr;
  int64_t stage_in_bytes = 0, stage_out_bytes = 0;
  cudaEvent_t ev_level[32] = {};  // H2D of input level l done (pipelined host path)
  // bounded page-locked ring for host buffers above the staging limit
  static constexpr int kRingSlots = 4;
  int64_t ring_bytes = 0;  // slot size: 256 MB (BI_RING_MB overrides; tests use tiny slots)
  char* ring[kRingSlots] = {};
  cudaEvent_t ring_ev[kRingSlots] = {};
  bool ring_busy[kRingSlots] = {};

  ~bi_engine() {
    for (auto& kv : seg_graphs) cudaGraphExecDestroy(kv.second);
    if (stage_in) cudaFreeHost(stage_in);
    if (stage_out) cudaFreeHost(stage_out);
    for (int i = 0; i < kRingSlots; ++i) {
      if (ring[i]) cudaFreeHost(ring[i]);
      if (ring_ev[i]) cudaEventDestroy(ring_ev[i]);
    }
    for (cudaEvent_t ev : ev_level)
      if (ev) cudaEventDestroy(ev);
    for (auto& kv : graphs) cudaGraphExecDestroy(kv.second);
    if (capture_stream) cudaStreamDestroy(capture_stream);
    for (int l = 0; l < kMaxLanes; ++l) {
      if (aux_stream[l]) cudaStreamDestroy(aux_stream[l]);
      if (ev_skew[l]) cudaEventDestroy(ev_skew[l]);
      if (ev_join[l]) cudaEventDestroy(ev_join[l]);
    }
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (tl_start) cudaEventDestroy(tl_start);
    for (cudaEvent_t ev : tl_ev) cudaEventDestroy(ev);
    if (copy_stream) cudaStreamDestroy(copy_stream);
    for (int l = 0; l < kMaxLanes; ++l) {
      if (d2h_stream[l]) cudaStreamDestroy(d2h_stream[l]);
      if (ev_d2h_a[l]) cudaEventDestroy(ev_d2h_a[l]);
      if (ev_d2h_b[l]) cudaEventDestroy(ev_d2h_b[l]);
      for (int c = 0; c < kOutChunks; ++c)
        if (ev_chunk[l][c]) cudaEventDestroy(ev_chunk[l][c]);
    }
    for (cudaEvent_t ev : ev_h2d) cudaEventDestroy(ev);
    if (meta_dev) cudaFree(meta_dev);
  }

  Window tset_window(int level, int z, int r0, int r1, int c0, int c1) const {
    const int lo = std::min(r0, c0);
    const int qp = lo >> level;
    const Sq& s = tsq[level][qp];
    const int64_t origin = off[(size_t)qp << level];
    double* base = T + (int64_t)z * t_matrix + s.off;
    (void)r1;
    (void)c1;
    return Window{base + (off[r0] - origin) * s.ld + (off[c0] - s.col_origin), s.ld};
  }
  // M and M_inv hold this rank's columns [col0, col0 + w) (all of them for P = 1)
  Window m_window(int z, int r0, int c0) const {
    return Window{const_cast<double*>(M) + (int64_t)z * sm + off[r0] * ldm + (off[c0] - col0), ldm};
  }
  Window minv_window(int z, int r0, int c0) const {
    return Window{Minv + (int64_t)z * si + off[r0] * ldi + (off[c0] - col0), ldi};
  }
  bool is_global(int level) const { return (1 << level) > nbp; }
  Window source(const StepAct& a, int z, int r0, int r1, int c0, int c1) const {
    return a.from_tset ? tset_window(a.cid, z, r0, r1, c0, c1) : m_window(z, r0, c0);
  }
};

static int64_t align256(int64_t v) { return round_up(v, 256); }

extern "C" int bi_engine_create(bi_engine** out, int nblocks, const int64_t* sizes, int batch) {
  return bi_engine_create_ex(out, nblocks, sizes, batch, BI_SCHEDULE_EQ7);
}

// pivot-A recursion tree over blocks [b0, b1): per depth, the largest T_b
// (p x ld(q)) + T_c (q x ld(p)) footprint of its nodes
static void pivot_a_footprint(const std::vector<int64_t>& off, int b0, int b1, int depth,
                              std::vector<int64_t>& per_depth) {
  if (b1 - b0 < 2) return;
  const int mid = (b0 + b1) / 2;
  const int64_t p = off[mid] - off[b0], q = off[b1] - off[mid];
  if ((int)per_depth.size() <= depth) per_depth.resize(depth + 1, 0);
  per_depth[depth] = std::max(per_depth[depth], round_up(p * round_up(q, 4), 32) + round_up(q * round_up(p, 4), 32));
  pivot_a_footprint(off, b0, mid, depth + 1, per_depth);
  pivot_a_footprint(off, mid, b1, depth + 1, per_depth);
}

static int create_common(bi_engine** out, int nblocks, const int64_t* sizes, int batch, int schedule, int nranks,
                         int rank, int flags) {
  BI_REQUIRE(out != nullptr && sizes != nullptr, "null argument");
  BI_REQUIRE(schedule == BI_SCHEDULE_EQ7 || schedule == BI_SCHEDULE_PIVOT_A, "unknown schedule");
  BI_REQUIRE(nblocks >= 1 && (nblocks & (nblocks - 1)) == 0,
             "number of diagonal blocks must be a power of two");
  BI_REQUIRE(batch >= 1, "batch must be >= 1");
  auto e = std::make_unique<bi_engine>();
  e->nb = nblocks;
  e->Z = batch;
  while ((1 << e->k) < nblocks) ++e->k;
  e->schedule = schedule;
  e->nsteps = schedule == BI_SCHEDULE_PIVOT_A ? 1 : 2 * nblocks - 1;
  e->off.push_back(0);
  int64_t maxb = 0;
  for (int i = 0; i < nblocks; ++i) {
    BI_REQUIRE(sizes[i] >= 1, "block sizes must be >= 1");
    e->sizes.push_back(sizes[i]);
    e->off.push_back(e->off.back() + sizes[i]);
    maxb = std::max(maxb, sizes[i]);
  }
  (void)maxb;  // blocks above kInvMaxDirect invert by a pivot-A recursion with K3 leaves
  e->n = e->off.back();
  BI_REQUIRE(nranks >= 1 && (nranks & (nranks - 1)) == 0 && nblocks % nranks == 0 && rank >= 0 && rank < nranks,
             "the rank count must be a power of two dividing the number of diagonal blocks");
  e->P = nranks;
  e->rank = rank;
  e->shard_flags = flags;
  e->nbp = nblocks / nranks;
  e->h0 = rank * e->nbp;
  e->h1 = e->h0 + e->nbp;
  e->col0 = e->off[e->h0];
  e->w = e->off[e->h1] - e->col0;
  for (int r = 0; r < nranks; ++r)
    e->wmax = std::max(e->wmax, e->off[(size_t)(r + 1) * e->nbp] - e->off[(size_t)r * e->nbp]);
  // T-set layout (per matrix): every level-l quad holding some of this rank's
  // columns; a quad wider than the home range keeps only the home columns
  e->tsq.resize(e->k + 1);
  int64_t t = 0;
  for (int lv = 1; lv <= e->k; ++lv) {
    const int nq = nblocks >> lv;
    for (int g = 0; g < nq; ++g) {
      const int first = g << lv, last = (g + 1) << lv;
      const int64_t side = e->off[last] - e->off[first];
      if (last <= e->h0 || first >= e->h1) {
        e->tsq[lv].push_back({-1, side, 0, 0, false});
        continue;
      }
      const int c_lo = std::max(first, e->h0), c_hi = std::min(last, e->h1);
      const int64_t cols = e->off[c_hi] - e->off[c_lo];
      const int64_t ld = round_up(cols, 4);
      e->tsq[lv].push_back({t, side, ld, e->off[c_lo], true});
      t += round_up(side * ld, 32);
    }
  }
  // global-level exchange buffers: X (the replicated operand of one action)
  // and, with BI_SHARD_STAGING, contiguous send / all-gather receive areas
  for (int lv = 1; lv <= e->k; ++lv) {
    if ((1 << lv) <= e->nbp) continue;
    const int g = e->h0 >> lv, first = g << lv, mid = first + (1 << (lv - 1)), last = (g + 1) << lv;
    const int64_t ha = e->off[mid] - e->off[first], hd = e->off[last] - e->off[mid];
    const bool in_a = e->h1 <= mid;
    const int gs = (1 << lv) / e->nbp;
    const int64_t xa = (ha + hd) * round_up(in_a ? hd : ha, 4);           // arrows
    const int64_t xu = in_a ? hd * round_up(ha, 4) : ha * round_up(hd, 4);  // up/down pass
    e->x_elems = std::max(e->x_elems, std::max(xa, xu));
    e->send_elems = std::max(e->send_elems, (ha + hd) * e->wmax);
    e->recv_elems = std::max(e->recv_elems, (int64_t)gs * (ha + hd) * e->wmax);
  }
  if (!(flags & BI_SHARD_STAGING)) e->send_elems = e->recv_elems = 0;
  if (schedule == BI_SCHEDULE_PIVOT_A) {  // no T-sets: per-depth T_b / T_c temporaries instead
    std::vector<int64_t> per_depth;
    pivot_a_footprint(e->off, 0, nblocks, 0, per_depth);
    t = 0;
    e->pa_depth_off.clear();
    for (int64_t f : per_depth) {
      e->pa_depth_off.push_back(t);
      t += f;
    }
  }
  e->t_matrix = t;
  e->t_bytes = align256(t * 8 * (int64_t)batch);
  // Lanes: with >= 2 matrices the batch is split in two halves that run on two
  // streams, lane 1 one step behind lane 0, so latency-bound leaf steps of
  // one lane overlap GEMM-bound steps of the other (BI_ENGINE_LANES=1 disables).
  const char* lanes_env = getenv("BI_ENGINE_LANES");
  int want = lanes_env ? atoi(lanes_env) : bi_engine::kMaxLanes;
  want = std::max(1, std::min(want, bi_engine::kMaxLanes));
  e->nlanes = std::min(want, batch);
  for (int l = 0; l < e->nlanes; ++l) {  // contiguous, near-equal matrix ranges
    e->zlo[l] = (int)((int64_t)batch * l / e->nlanes);
    e->zhi[l] = (int)((int64_t)batch * (l + 1) / e->nlanes);
  }
  // leaf scratch (per lane): the largest equal-size group of one diag step
  std::map<int64_t, int> cnt;
  int lane_max = 0;
  for (int l = 0; l < e->nlanes; ++l) lane_max = std::max(lane_max, e->zhi[l] - e->zlo[l]);
  for (int p = e->h0; p < e->h1; ++p) {
    const int64_t s = e->sizes[p];
    if (schedule == BI_SCHEDULE_PIVOT_A) cnt[s] = lane_max;  // one leaf at a time per lane
    else cnt[s] += lane_max;
  }
  int64_t scratch = 0;
  for (auto& kv : cnt) scratch = std::max(scratch, inv_group_scratch_bytes((int)kv.first, kv.second));
  e->inv_scratch = align256(scratch);
  // Eq. 7: nblocks diag steps x leaves; pivot-A: every block is a leaf once
  e->info_ints = (int64_t)(schedule == BI_SCHEDULE_PIVOT_A ? 1 : nblocks) * nblocks * batch;
  // metadata upper bound (descriptors + pointer tables); computed exactly at bind
  *out = e.release();
  return 0;
}

extern "C" int bi_engine_create_ex(bi_engine** out, int nblocks, const int64_t* sizes, int batch, int schedule) {
  return create_common(out, nblocks, sizes, batch, schedule, 1, 0, 0);
}

extern "C" int bi_engine_create_shard(bi_engine** out, int nblocks, const int64_t* sizes, int nranks, int rank,
                                      int flags) {
  return create_common(out, nblocks, sizes, 1, BI_SCHEDULE_EQ7, nranks, rank, flags);
}

extern "C" int64_t bi_engine_workspace_bytes(const bi_engine* e) {
  if (!e) return -1;
  // schedule metadata (descriptor and pointer tables) is engine-owned device memory
  return e->t_bytes + e->nlanes * e->inv_scratch + align256(e->info_ints * 4) + align256(e->x_elems * 8) +
         align256(e->send_elems * 8) + align256(e->recv_elems * 8);
}

static int build_pivot_a(bi_engine* e);

static int build_schedule(bi_engine* e) {
  if (e->schedule == BI_SCHEDULE_PIVOT_A) return build_pivot_a(e);
  for (int l = 0; l < bi_engine::kMaxLanes; ++l) e->lane_ops[l].assign(e->nsteps + 1, {});
  e->descs.clear();
  e->launches.clear();
  e->invs.clear();
  e->diag_steps.clear();
  const int nb = e->nb;
  const auto& off = e->off;
  auto add_launch = [&](const std::vector<GemmDesc>& raw) -> int {
    std::vector<GemmDesc> m = merge_descs(raw);
    GemmLaunchRec rec{(int)e->descs.size(), (int)m.size()};
    finalize_descs(m.data(), (int)m.size());
    e->descs.insert(e->descs.end(), m.begin(), m.end());
    e->launches.push_back(rec);
    return (int)e->launches.size() - 1;
  };
  auto gemm = [](Window a, Window b, const double* c, int64_t ldc, Window d, int64_t M, int64_t N,
                 int64_t K, int neg) {
    GemmDesc g{};
    g.A = a.p;
    g.lda = a.ld;
    g.B = b.p;
    g.ldb = b.ld;
    g.C = c;
    g.ldc = c ? ldc : 0;
    g.D = d.p;
    g.ldd = d.ld;
    g.M = (int)M;
    g.N = (int)N;
    g.K = (int)K;
    g.batch = 1;
    g.neg = neg;
    g.skip_at = INT32_MAX;
    g.skip_len = 0;
    return g;
  };
  e->xchgs.clear();
  // one global-level exchange of this rank (its group, send parts, X layout)
  auto add_xchg = [&](int lv, int kind, const StepAct& a) -> int {
    bi_engine::Xchg x;
    x.level = lv;
    x.kind = kind;
    const int g = e->h0 >> lv, first = g << lv, mid = first + (1 << (lv - 1)), last = (g + 1) << lv;
    const int64_t ha = off[mid] - off[first], hd = off[last] - off[mid];
    x.gs = (1 << lv) / e->nbp;
    x.g0 = e->rank / x.gs * x.gs;
    x.in_a = e->h1 <= mid;
    const int half = x.gs / 2;
    auto part = [](Window wdw, const double*& p, int64_t& ld) {
      p = wdw.p;
      ld = wdw.ld;
    };
    if (kind == 0) {  // arrows: A-half ranks send [A^-1 ; C], D-half ranks [B ; D^-1]; X = the other half's
      if (x.in_a) {
        part(e->minv_window(0, first, e->h0), x.top, x.top_ld);
        part(e->source(a, 0, mid, last, e->h0, e->h1), x.bot, x.bot_ld);
        x.from0 = x.g0 + half;
        x.from1 = x.g0 + x.gs;
        x.x_col0 = off[mid];
        x.xcols = hd;
      } else {
        part(e->source(a, 0, first, mid, e->h0, e->h1), x.top, x.top_ld);
        part(e->minv_window(0, mid, e->h0), x.bot, x.bot_ld);
        x.from0 = x.g0;
        x.from1 = x.g0 + half;
        x.x_col0 = off[first];
        x.xcols = ha;
      }
      x.top_rows = ha;
      x.bot_rows = hd;
      x.rows = ha + hd;
    } else {  // up/down pass: A-half ranks share their L columns, D-half ranks their R columns
      // The exchange stays inside the rank's own half of the group: only those
      // ranks read its part, and only they send parts of the same height (L is
      // hd x ha, R is ha x hd: with ragged block orders the halves differ, and
      // an all-gather needs equal contributions).  A half of one rank
      // (gs == 1) is a local copy.
      if (x.in_a) {
        part(e->tset_window(lv, 0, mid, last, e->h0, e->h1), x.top, x.top_ld);
        x.top_rows = hd;
        x.x_col0 = off[first];
        x.xcols = ha;
      } else {
        part(e->tset_window(lv, 0, first, mid, e->h0, e->h1), x.top, x.top_ld);
        x.top_rows = ha;
        x.g0 += half;
        x.x_col0 = off[mid];
        x.xcols = hd;
      }
      x.gs = half;
      x.from0 = x.g0;
      x.from1 = x.g0 + x.gs;
      x.rows = x.top_rows;
    }
    x.ldx = round_up(x.xcols, 4);
    e->xchgs.push_back(x);
    return (int)e->xchgs.size() - 1;
  };
  int info_cursor = 0;
  for (int stepid = 1; stepid <= e->nsteps; ++stepid) {
    StepAct a;
    loopid_decode(stepid, nb, &a);
    if (a.kind == 0 || a.kind == 2) e->diag_steps.push_back(stepid);
  }
  for (int lane = 0; lane < e->nlanes; ++lane) {
  const int Z0 = e->zlo[lane], Z1 = e->zhi[lane];
  int diag_index = 0;
  for (int stepid = 1; stepid <= e->nsteps; ++stepid) {
    StepAct a;
    loopid_decode(stepid, nb, &a);
    auto& ops = e->lane_ops[lane][stepid];
    if (a.kind == 0 || a.kind == 2) {
      // diag: group leaves (z, p) by block size
      std::map<int64_t, std::vector<std::pair<int, int>>> groups;
      for (int z = Z0; z < Z1; ++z)
        for (int p = e->h0; p < e->h1; ++p) groups[e->sizes[p]].push_back({z, p});
      for (auto& kv : groups) {
        InvRec r{};
        r.g.n = (int)kv.first;
        r.g.count = (int)kv.second.size();
        r.diag_step_index = diag_index;
        r.lane = lane;
        r.info_offset = info_cursor;
        info_cursor += r.g.count;
        for (auto& zp : kv.second) {
          r.item_matrix.push_back(zp.first);
          r.item_block.push_back(zp.second);
        }
        e->invs.push_back(std::move(r));
        ops.push_back({0, (int)e->invs.size() - 1});
      }
      ++diag_index;
      if (a.kind == 2) {
        for (int lv = 1; lv <= a.depth; ++lv) {
          if (e->is_global(lv)) {  // exchange L / R inside the group, then this rank's columns
            const int xi = add_xchg(lv, 1, a);
            const auto& x = e->xchgs[xi];
            const int g = e->h0 >> lv, first = g << lv, mid = first + (1 << (lv - 1)), last = (g + 1) << lv;
            const int64_t ha = off[mid] - off[first], hd = off[last] - off[mid];
            const Window X{e->X, x.ldx};
            std::vector<GemmDesc> raw;
            if (x.in_a)  // Minv[D, my A cols] = L Minv[A, my A cols]
              raw.push_back(gemm(X, e->minv_window(0, first, e->h0), nullptr, 0, e->minv_window(0, mid, e->h0), hd,
                                 e->w, ha, 0));
            else  // Minv[A, my D cols] = R Minv[D, my D cols]
              raw.push_back(gemm(X, e->minv_window(0, mid, e->h0), nullptr, 0, e->minv_window(0, first, e->h0), ha,
                                 e->w, hd, 0));
            ops.push_back({3, xi});
            ops.push_back({1, add_launch(raw)});
            continue;
          }
          std::vector<GemmDesc> raw;
          for (int z = Z0; z < Z1; ++z)
            for (int g = (e->h0 >> lv); g < (e->h1 >> lv); ++g) {
              const int first = g << lv, mid = first + (1 << (lv - 1)), last = (g + 1) << lv;
              const int64_t ha = off[mid] - off[first], hd = off[last] - off[mid];
              // down: Minv[D, A] = L * Minv[A, A]
              raw.push_back(gemm(e->tset_window(lv, z, mid, last, first, mid), e->minv_window(z, first, first),
                                 nullptr, 0, e->minv_window(z, mid, first), hd, ha, ha, 0));
            }
          for (int z = Z0; z < Z1; ++z)
            for (int g = (e->h0 >> lv); g < (e->h1 >> lv); ++g) {
              const int first = g << lv, mid = first + (1 << (lv - 1)), last = (g + 1) << lv;
              const int64_t ha = off[mid] - off[first], hd = off[last] - off[mid];
              // up: Minv[A, D] = R * Minv[D, D]
              raw.push_back(gemm(e->tset_window(lv, z, first, mid, mid, last), e->minv_window(z, mid, mid),
                                 nullptr, 0, e->minv_window(z, first, mid), ha, hd, hd, 0));
            }
          ops.push_back({1, add_launch(raw)});
        }
      }
    } else if (e->is_global(a.sid)) {
      // global arrows: X = the other half's [B ; D^-1] (A-half ranks) or
      // [A^-1 ; C] (D-half ranks); then this rank's columns of L, S_D / R, S_A
      const int lv = a.sid;
      const int xi = add_xchg(lv, 0, a);
      const auto& x = e->xchgs[xi];
      const int g = e->h0 >> lv, first = g << lv, mid = first + (1 << (lv - 1)), last = (g + 1) << lv;
      const int64_t ha = off[mid] - off[first], hd = off[last] - off[mid];
      const Window X0{e->X, x.ldx}, X1{e->X + ha * x.ldx, x.ldx};
      std::vector<GemmDesc> l1, l2;
      if (x.in_a) {
        const Window Lm = e->tset_window(lv, 0, mid, last, e->h0, e->h1);
        l1.push_back(gemm(X1, e->source(a, 0, mid, last, e->h0, e->h1), nullptr, 0, Lm, hd, e->w, hd, 1));  // -D^-1 C
        const Window Am = e->source(a, 0, first, mid, e->h0, e->h1);
        l2.push_back(gemm(X0, Lm, Am.p, Am.ld, e->tset_window(lv, 0, first, mid, e->h0, e->h1), ha, e->w, hd,
                          0));  // S_D = A + B L
      } else {
        const Window Rm = e->tset_window(lv, 0, first, mid, e->h0, e->h1);
        l1.push_back(gemm(X0, e->source(a, 0, first, mid, e->h0, e->h1), nullptr, 0, Rm, ha, e->w, ha, 1));  // -A^-1 B
        const Window Dm = e->source(a, 0, mid, last, e->h0, e->h1);
        l2.push_back(gemm(X1, Rm, Dm.p, Dm.ld, e->tset_window(lv, 0, mid, last, e->h0, e->h1), hd, e->w, ha,
                          0));  // S_A = D + C R
      }
      ops.push_back({3, xi});
      ops.push_back({1, add_launch(l1)});
      ops.push_back({1, add_launch(l2)});
    } else {
      const int lv = a.sid;
      std::vector<GemmDesc> l1, l2;
      // Quad order: sources in T_cid put 2^(cid-sid) level-sid quads on the
      // diagonal of each T_cid square -- a uniform stride inside a square, a
      // jump between squares.  Visiting the quads as (position in square,
      // square) when there are fewer positions than squares makes every
      // position class one strided batch, so a launch carries at most 4
      // descriptors per product and stays on the TMA path (ncu r02: 88
      // launches had fallen back to the cp.async descriptor-table kernel).
      const int qlo = e->h0 >> lv, qn = (e->h1 >> lv) - qlo;
      const int per_sq = (a.from_tset && !e->is_global(a.cid)) ? std::min(qn, 1 << (a.cid - lv)) : 1;
      const int nsq = qn / per_sq;
      const bool by_pos = per_sq > 1 && per_sq <= nsq;
      auto quad_at = [&](int i) { return qlo + (by_pos ? (i % nsq) * per_sq + i / nsq : i); };
      for (int kind = 0; kind < 2; ++kind)
        for (int z = Z0; z < Z1; ++z)
          for (int gi = 0; gi < qn; ++gi) {
            const int g = quad_at(gi);
            const int first = g << lv, mid = first + (1 << (lv - 1)), last = (g + 1) << lv;
            const int64_t ha = off[mid] - off[first], hd = off[last] - off[mid];
            Window B = e->source(a, z, first, mid, mid, last);
            Window C = e->source(a, z, mid, last, first, mid);
            Window R = e->tset_window(lv, z, first, mid, mid, last);
            Window L = e->tset_window(lv, z, mid, last, first, mid);
            if (kind == 0) {  // R = -A^-1 B
              l1.push_back(gemm(e->minv_window(z, first, first), B, nullptr, 0, R, ha, hd, ha, 1));
            } else {  // L = -D^-1 C
              l1.push_back(gemm(e->minv_window(z, mid, mid), C, nullptr, 0, L, hd, ha, hd, 1));
            }
          }
      for (int kind = 0; kind < 2; ++kind)
        for (int z = Z0; z < Z1; ++z)
          for (int gi = 0; gi < qn; ++gi) {
            const int g = quad_at(gi);
            const int first = g << lv, mid = first + (1 << (lv - 1)), last = (g + 1) << lv;
            const int64_t ha = off[mid] - off[first], hd = off[last] - off[mid];
            Window Aw = e->source(a, z, first, mid, first, mid);
            Window B = e->source(a, z, first, mid, mid, last);
            Window C = e->source(a, z, mid, last, first, mid);
            Window Dw = e->source(a, z, mid, last, mid, last);
            Window R = e->tset_window(lv, z, first, mid, mid, last);
            Window L = e->tset_window(lv, z, mid, last, first, mid);
            Window SD = e->tset_window(lv, z, first, mid, first, mid);
            Window SA = e->tset_window(lv, z, mid, last, mid, last);
            if (kind == 0) {  // S_D = A + B L
              l2.push_back(gemm(B, L, Aw.p, Aw.ld, SD, ha, ha, hd, 0));
            } else {  // S_A = D + C R
              l2.push_back(gemm(C, R, Dw.p, Dw.ld, SA, hd, hd, ha, 0));
            }
          }
      ops.push_back({1, add_launch(l1)});
      ops.push_back({1, add_launch(l2)});
    }
  }
  }
  return 0;
}

// ---------------------------------------------------------------------------
// pivot-A schedule: the 2n^3 recursion of invertor_by_a
// (recursive.py:83-123) at block granularity, in place in M_inv, batched over
// the lane's matrices.  Node over blocks [b0, b1) split at mid (p, q rows):
//   recurse on A                          -> A = A^-1
//   T_b = -A B,  T_c = -C A               (one launch)
//   D  += C T_b                           (S_A = D - C A^-1 B)
//   recurse on D                          -> D = S_A^-1
//   C   = D T_c,  B = T_b D               (one launch: -S^-1 C A^-1, -A^-1 B S^-1)
//   A  += T_b C                           (A^-1 + A^-1 B S^-1 C A^-1)
// 12 p q (p + q) / 2 ... = 6pq(p+q) flops per node, 2n^3 in total with the
// leaves; T_b / T_c live in per-depth workspace regions.
// ---------------------------------------------------------------------------
static int build_pivot_a(bi_engine* e) {
  for (int l = 0; l < bi_engine::kMaxLanes; ++l) e->lane_ops[l].assign(e->nsteps + 1, {});
  e->descs.clear();
  e->launches.clear();
  e->invs.clear();
  e->diag_steps.assign(1, 1);
  const auto& off = e->off;
  auto add_launch = [&](const std::vector<GemmDesc>& raw) -> int {
    std::vector<GemmDesc> m = merge_descs(raw);
    GemmLaunchRec rec{(int)e->descs.size(), (int)m.size()};
    finalize_descs(m.data(), (int)m.size());
    e->descs.insert(e->descs.end(), m.begin(), m.end());
    e->launches.push_back(rec);
    return (int)e->launches.size() - 1;
  };
  auto gemm = [](const double* a, int64_t lda, const double* b, int64_t ldb, const double* c, int64_t ldc,
                 double* d, int64_t ldd, int64_t M, int64_t N, int64_t K, int neg) {
    GemmDesc g{};
    g.A = a;
    g.lda = lda;
    g.B = b;
    g.ldb = ldb;
    g.C = c;
    g.ldc = c ? ldc : 0;
    g.D = d;
    g.ldd = ldd;
    g.M = (int)M;
    g.N = (int)N;
    g.K = (int)K;
    g.batch = 1;
    g.neg = neg;
    g.skip_at = INT32_MAX;
    g.skip_len = 0;
    return g;
  };
  int info_cursor = 0;
  for (int lane = 0; lane < e->nlanes; ++lane) {
    const int Z0 = e->zlo[lane], Z1 = e->zhi[lane];
    auto& ops = e->lane_ops[lane][1];
    ops.push_back({2, lane});
    auto mi = [&](int z, int br, int bc) { return e->Minv + (int64_t)z * e->si + off[br] * e->ldi + off[bc]; };
    std::function<void(int, int, int)> node = [&](int b0, int b1, int depth) {
      if (b1 - b0 == 1) {
        InvRec r{};
        r.g.n = (int)e->sizes[b0];
        r.g.count = Z1 - Z0;
        r.diag_step_index = 0;
        r.lane = lane;
        r.info_offset = info_cursor;
        r.in_place = true;
        info_cursor += r.g.count;
        for (int z = Z0; z < Z1; ++z) {
          r.item_matrix.push_back(z);
          r.item_block.push_back(b0);
        }
        e->invs.push_back(std::move(r));
        ops.push_back({0, (int)e->invs.size() - 1});
        return;
      }
      const int mid = (b0 + b1) / 2;
      const int64_t p = off[mid] - off[b0], q = off[b1] - off[mid];
      const int64_t ldb_t = round_up(q, 4), ldc_t = round_up(p, 4);
      const int64_t ld = e->ldi;
      auto tb = [&](int z) { return e->T + (int64_t)z * e->t_matrix + e->pa_depth_off[depth]; };
      auto tc = [&](int z) { return tb(z) + round_up(p * ldb_t, 32); };
      node(b0, mid, depth + 1);
      std::vector<GemmDesc> l1, l2, l3, l4;
      for (int z = Z0; z < Z1; ++z) {
        double *A = mi(z, b0, b0), *B = mi(z, b0, mid), *C = mi(z, mid, b0), *D = mi(z, mid, mid);
        l1.push_back(gemm(A, ld, B, ld, nullptr, 0, tb(z), ldb_t, p, q, p, 1));   // T_b = -A^-1 B
        l1.push_back(gemm(C, ld, A, ld, nullptr, 0, tc(z), ldc_t, q, p, p, 1));   // T_c = -C A^-1
        l2.push_back(gemm(C, ld, tb(z), ldb_t, D, ld, D, ld, q, q, p, 0));        // S_A = D + C T_b
        l3.push_back(gemm(D, ld, tc(z), ldc_t, nullptr, 0, C, ld, q, p, q, 0));   // C = S^-1 T_c
        l3.push_back(gemm(tb(z), ldb_t, D, ld, nullptr, 0, B, ld, p, q, q, 0));   // B = T_b S^-1
        l4.push_back(gemm(tb(z), ldb_t, C, ld, A, ld, A, ld, p, p, q, 0));        // A += T_b C
      }
      ops.push_back({1, add_launch(l1)});
      ops.push_back({1, add_launch(l2)});
      node(mid, b1, depth + 1);
      ops.push_back({1, add_launch(l3)});
      ops.push_back({1, add_launch(l4)});
    };
    node(0, e->nb, 0);
  }
  return 0;
}

extern "C" int bi_engine_bind(bi_engine* e, const double* m, int64_t ldm, int64_t stride_m, double* minv,
                              int64_t ldi, int64_t stride_i, void* workspace, int64_t workspace_bytes,
                              void* stream) {
  BI_REQUIRE(e != nullptr, "null engine");
  BI_REQUIRE(m && minv && workspace, "null buffer");
  BI_REQUIRE(ldm >= e->w && ldi >= e->w, "leading dimension smaller than the owned columns");
  BI_REQUIRE(workspace_bytes >= bi_engine_workspace_bytes(e), "workspace too small");
  for (auto& kv : e->graphs) cudaGraphExecDestroy(kv.second);
  e->graphs.clear();
  e->M = m;
  e->ldm = ldm;
  e->sm = stride_m;
  e->Minv = minv;
  e->ldi = ldi;
  e->si = stride_i;
  e->ws = static_cast<char*>(workspace);
  e->ws_bytes = workspace_bytes;
  char* p = e->ws;
  e->T = reinterpret_cast<double*>(p);
  p += e->t_bytes;
  for (int l = 0; l < e->nlanes; ++l) {
    e->inv_base[l] = p;
    p += e->inv_scratch;
  }
  e->info = reinterpret_cast<int*>(p);
  p += align256(e->info_ints * 4);
  e->X = reinterpret_cast<double*>(p);
  p += align256(e->x_elems * 8);
  e->sendbuf = reinterpret_cast<double*>(p);
  p += align256(e->send_elems * 8);
  e->recvbuf = reinterpret_cast<double*>(p);
  p += align256(e->recv_elems * 8);
  cudaGetDevice(&e->device);
  for (auto& kv : e->seg_graphs) cudaGraphExecDestroy(kv.second);
  e->seg_graphs.clear();
  BI_CUDA_TRY(init_attributes());
  {
    // BI_PRIORITY_MODE: 0 none; 1 lane order (lane 0 highest); 2 leaf kernels
    // above the GEMMs; 3 leaf kernels highest, then the GEMMs of later-starting
    // lanes; 4 leaf kernels highest, then the GEMMs in lane order.
    // Two scheduling policies (measured, profiles/r01_engine_policies.txt):
    //  * device-resident runs: leaf kernels at the highest priority, GEMMs
    //    equal, lanes start together (mode 2, skew 0);
    //  * runs that read the inverses back to the host: lane 0 highest, lanes
    //    start together (mode 1, skew 0) -- lanes finish staggered, so the
    //    per-lane read-backs (PCIe-bound, ~2.3 ms each at cfg2) overlap compute.
    // BI_PRIORITY_MODE / BI_ENGINE_SKEW override both.
    const char* pe = getenv("BI_PRIORITY_MODE");
    const char* sk = getenv("BI_ENGINE_SKEW");
    int least = 0, greatest = 0;
    cudaDeviceGetStreamPriorityRange(&least, &greatest);
    for (int pol = 0; pol < 2; ++pol) {
      const int mode = pe ? atoi(pe) : (pol == 0 ? 2 : 1);
      // mode 3: leaf kernels highest, then the GEMMs of later-starting lanes
      for (int l = 0; l < e->nlanes; ++l) {
        int pr = 0;
        if (mode == 1 && e->nlanes > 1) pr = std::min(greatest + l, least);
        if (mode == 3 && e->nlanes > 1) pr = std::min(greatest + 1 + (e->nlanes - 1 - l), least);
        if (mode == 4 && e->nlanes > 1) pr = std::min(greatest + 1 + l, least);
        e->pol[pol].lane_priority[l] = pr;
      }
      e->pol[pol].leaf_priority = (mode >= 2 && mode <= 4) ? greatest : 0;
      e->pol[pol].skew = sk ? atoi(sk) : 0;
    }
    int dev = 0, nsm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const char* rs = getenv("BI_RESERVE_SMS");
    // BI_RESERVE_SMS: SMs kept out of a persistent (grid-capped) engine GEMM.
    // Device-resident runs: no cap -- one CTA per tile, so SMs free up at
    // every tile end and the top-priority leaf kernels of other lanes get them
    // at once instead of waiting out a persistent GEMM (27.4 -> 27.0 ms).
    // Host read-back runs keep 16 SMs out of a persistent grid (their lanes
    // run in lane-priority order; e2e 31.2 -> 31.0 ms).
    for (int pol = 0; pol < 2; ++pol) {
      const int reserve = rs ? atoi(rs) : (pol == 0 || e->nlanes == 1 ? 0 : 16);
      e->pol[pol].gemm_cap = (reserve > 0 && reserve < nsm) ? nsm - reserve : 0;
    }
    e->set_policy(0);
  }
  if (!e->d2h_stream[0]) {
    for (int l = 0; l < e->nlanes; ++l) {
      BI_CUDA_TRY(cudaStreamCreateWithFlags(&e->d2h_stream[l], cudaStreamNonBlocking));
      BI_CUDA_TRY(cudaEventCreateWithFlags(&e->ev_d2h_a[l], cudaEventDisableTiming));
      BI_CUDA_TRY(cudaEventCreateWithFlags(&e->ev_d2h_b[l], cudaEventDisableTiming));
      for (int c = 0; c < bi_engine::kOutChunks; ++c)
        BI_CUDA_TRY(cudaEventCreateWithFlags(&e->ev_chunk[l][c], cudaEventDisableTiming));
      if (!e->ev_join[l]) BI_CUDA_TRY(cudaEventCreateWithFlags(&e->ev_join[l], cudaEventDisableTiming));
    }
  }
  if (!e->copy_stream) {
    BI_CUDA_TRY(cudaStreamCreateWithFlags(&e->copy_stream, cudaStreamNonBlocking));
    e->ev_h2d.assign((size_t)e->Z * (e->k + 1), nullptr);
    for (auto& ev : e->ev_h2d) BI_CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  }
  if (!e->ev_fork) BI_CUDA_TRY(cudaEventCreateWithFlags(&e->ev_fork, cudaEventDisableTiming));
  {
    const char* tl = getenv("BI_ENGINE_TIMELINE");
    e->timeline = tl && atoi(tl) != 0;
    if (e->timeline && !e->tl_start) {
      BI_CUDA_TRY(cudaEventCreate(&e->tl_start));
      e->tl_ev.assign((size_t)e->nlanes * (e->nsteps + 1), nullptr);
      for (auto& ev : e->tl_ev) BI_CUDA_TRY(cudaEventCreate(&ev));
    }
  }
  if (e->nlanes > 1 && !e->ev_skew[0]) {
    for (int l = 0; l < e->nlanes; ++l) {
      if (l > 0) BI_CUDA_TRY(cudaStreamCreateWithFlags(&e->aux_stream[l], cudaStreamNonBlocking));
      BI_CUDA_TRY(cudaEventCreateWithFlags(&e->ev_skew[l], cudaEventDisableTiming));
      BI_CUDA_TRY(cudaEventCreateWithFlags(&e->ev_join[l], cudaEventDisableTiming));
    }
  }

  int rc = build_schedule(e);
  if (rc) return rc;
  // inversion groups: scratch, info, pointer tables, panel descriptors
  std::vector<char> host_meta;
  auto reserve = [&](int64_t bytes) {
    int64_t o = align256((int64_t)host_meta.size());
    host_meta.resize(o + bytes);
    return o;
  };
  // panel descriptors appended to e->descs
  struct PtrTab {
    int64_t src, srcld, dst, dstld;
  };
  std::vector<PtrTab> tabs;
  for (InvRec& r : e->invs) {
    inv_group_layout(r.g, e->inv_base[r.lane]);
    r.g.info = e->info + r.info_offset;
    tabs.push_back({reserve(r.g.count * 8), reserve(r.g.count * 8), reserve(r.g.count * 8),
                    reserve(r.g.count * 8)});
  }
  const int64_t desc_off = reserve((int64_t)e->descs.size() * sizeof(GemmDesc));
  if ((int64_t)host_meta.size() > e->meta_cap) {
    if (e->meta_dev) cudaFree(e->meta_dev);
    e->meta_dev = nullptr;
    e->meta_cap = 0;
    BI_CUDA_TRY(cudaMalloc(&e->meta_dev, host_meta.size()));
    e->meta_cap = (int64_t)host_meta.size();
  }
  char* meta = static_cast<char*>(e->meta_dev);
  // fill tables (device addresses relative to meta)
  int diag_i = 0;
  for (size_t i = 0; i < e->invs.size(); ++i) {
    InvRec& r = e->invs[i];
    const int stepid = e->diag_steps[r.diag_step_index];
    StepAct a;
    loopid_decode(stepid, e->nb, &a);
    auto* src = reinterpret_cast<const double**>(host_meta.data() + tabs[i].src);
    auto* srcld = reinterpret_cast<int64_t*>(host_meta.data() + tabs[i].srcld);
    auto* dst = reinterpret_cast<double**>(host_meta.data() + tabs[i].dst);
    auto* dstld = reinterpret_cast<int64_t*>(host_meta.data() + tabs[i].dstld);
    for (int it = 0; it < r.g.count; ++it) {
      const int z = r.item_matrix[it], pb = r.item_block[it];
      Window s = r.in_place ? e->minv_window(z, pb, pb) : e->source(a, z, pb, pb + 1, pb, pb + 1);
      Window d = e->minv_window(z, pb, pb);
      src[it] = s.p;
      srcld[it] = s.ld;
      dst[it] = d.p;
      dstld[it] = d.ld;
    }
    r.h_src.assign(src, src + r.g.count);
    r.h_srcld.assign(srcld, srcld + r.g.count);
    r.h_dst.assign(dst, dst + r.g.count);
    r.h_dstld.assign(dstld, dstld + r.g.count);
    r.g.h_src_ptrs = r.h_src.data();
    r.g.h_src_lds = r.h_srcld.data();
    r.g.h_dst_ptrs = r.h_dst.data();
    r.g.h_dst_lds = r.h_dstld.data();
    r.g.src_ptrs = reinterpret_cast<const double* const*>(meta + tabs[i].src);
    r.g.src_lds = reinterpret_cast<const int64_t*>(meta + tabs[i].srcld);
    r.g.dst_ptrs = reinterpret_cast<double* const*>(meta + tabs[i].dst);
    r.g.dst_lds = reinterpret_cast<const int64_t*>(meta + tabs[i].dstld);
    ++diag_i;
  }
  std::memcpy(host_meta.data() + desc_off, e->descs.data(), e->descs.size() * sizeof(GemmDesc));
  e->d_descs = reinterpret_cast<GemmDesc*>(meta + desc_off);
  BI_CUDA_TRY(cudaMemcpyAsync(meta, host_meta.data(), host_meta.size(), cudaMemcpyHostToDevice,
                              static_cast<cudaStream_t>(stream)));
  BI_CUDA_TRY(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
  // flat op list of the (single) lane: the shard segment driver walks it
  e->flat.clear();
  e->step_first_op.assign(e->nsteps + 2, 0);
  for (int st = 1; st <= e->nsteps; ++st) {
    e->step_first_op[st] = (int)e->flat.size();
    for (const Op& op : e->lane_ops[0][st]) e->flat.push_back({st, op});
  }
  e->step_first_op[e->nsteps + 1] = (int)e->flat.size();
  e->bound = true;
  return 0;
}

struct HostIO;
static cudaError_t copy_top_quads(bi_engine* e, int lane, const HostIO* io, bool diag, cudaStream_t st);

// BI_OUT_CHUNKS (default 8, max 16): row chunks of the last top-level pass, each read
// back as soon as written (cfg4 run_inversion(m): 4 -> 408.4 / 407.4 ms, 8 -> 404.9 / 405.2, 16 -> 407.8)
static int out_chunks() {
  static const int c = [] {
    const char* v = getenv("BI_OUT_CHUNKS");
    const int x = v ? atoi(v) : 8;
    return x < 1 ? 1 : (x > bi_engine::kOutChunks ? bi_engine::kOutChunks : x);
  }();
  return c;
}

static cudaError_t pass_in_chunks(bi_engine* e, int lane, const GemmLaunchRec& L, const HostIO* io,
                                  cudaStream_t s);

// BI_LEAF_GEMM_CAP: SMs the leaf chain's own trailing-update GEMMs may use
// (persistent grid of 2 CTAs per SM); 0 = uncapped.  A narrow grid starts
// as soon as a few SMs free up instead of waiting for a GPU's worth of
// another lane's GEMM tiles to retire.
static int leaf_gemm_cap() {
  static const int cap = [] {
    const char* v = getenv("BI_LEAF_GEMM_CAP");
    return v ? atoi(v) : 0;
  }();
  return cap;
}

// BI_ENGINE_PDL (default 0): measured within noise (cfg4 394.6 / 396.3 ms off,
// 395.3 / 394.7 on; cfg2 27.0 / 26.9 vs 26.7 / 26.9; profiles/r02_k1_tiles.txt)
static int engine_pdl() {
  static const int on = [] {
    const char* v = getenv("BI_ENGINE_PDL");
    return v ? atoi(v) : 0;
  }();
  return on;
}

static cudaError_t enqueue_lane(bi_engine* e, int lane, int first, int last, cudaStream_t s, int mask,
                                cudaEvent_t after_first = nullptr, bool wait_input = false,
                                const HostIO* split_io = nullptr) {
  // Lane priority: lane 0 highest.  The leading lane then runs as if alone
  // and the others fill the SMs its latency-bound leaf phases leave idle.
  PriorityScope lane_prio(e->lane_priority[lane]);
  for (int stepid = first; stepid <= last; ++stepid) {
    const auto& step_ops = e->lane_ops[lane][stepid];
    if (wait_input && (stepid & (stepid - 1)) == 0) {
      // Eq. 7: step 2^l is the first to read M at level l (diag blocks for
      // l = 0, the level-l quads' off-diagonal blocks for l >= 1).  pivot-A
      // copies the whole input into M_inv first: wait for every level.
      int lv = 0;
      while ((1 << lv) < stepid) ++lv;
      const int lv_hi = e->schedule == BI_SCHEDULE_PIVOT_A ? e->k : lv;
      for (int z = e->zlo[lane]; z < e->zhi[lane]; ++z)
        for (int l = (e->schedule == BI_SCHEDULE_PIVOT_A ? 0 : lv); l <= lv_hi; ++l) {
          cudaError_t err = cudaStreamWaitEvent(s, e->ev_h2d[(size_t)z * (e->k + 1) + l], 0);
          if (err != cudaSuccess) return err;
        }
    }
    for (const Op& op : step_ops) {
      if (op.kind == 3) continue;  // exchanges: shard driver only (P > 1)
      if (!(mask & (op.kind == 0 ? 2 : 1))) continue;
      cudaError_t err;
      if (split_io && stepid == e->nsteps && &op == &step_ops.back() && op.kind == 1) {
        // last step, before its top-level up/down pass: the diagonal quads are
        // final -- read them back while the pass runs
        err = cudaEventRecord(e->ev_d2h_a[lane], s);
        if (err == cudaSuccess) err = cudaStreamWaitEvent(e->d2h_stream[lane], e->ev_d2h_a[lane], 0);
        if (err == cudaSuccess) err = copy_top_quads(e, lane, split_io, true, e->d2h_stream[lane]);
        if (err != cudaSuccess) return err;
      }
      if (op.kind == 2) {  // pivot-A: the lane's inputs into M_inv (inverted in place)
        err = cudaSuccess;
        for (int z = e->zlo[lane]; z < e->zhi[lane] && err == cudaSuccess; ++z)
          err = cudaMemcpy2DAsync(e->Minv + (int64_t)z * e->si, e->ldi * 8, e->M + (int64_t)z * e->sm, e->ldm * 8,
                                  e->n * 8, e->n, cudaMemcpyDeviceToDevice, s);
      } else if (op.kind == 0) {
        static const bool skip_leaves = [] {  // timing experiments only: results are wrong
          const char* v = getenv("BI_DEBUG_SKIP_LEAVES");
          return v && atoi(v) != 0;
        }();
        if (skip_leaves) continue;
        PriorityScope leaf_prio(e->leaf_priority ? e->leaf_priority : g_launch_priority);
        GemmCapScope leaf_cap(leaf_gemm_cap());
        err = launch_inv_group(e->invs[op.index].g, s);
      } else if (split_io && stepid == e->nsteps && &op == &step_ops.back() &&
                 e->launches[op.index].count <= kGemmInline) {
        // the last top-level pass writes the off-diagonal top quads: run it in
        // row chunks and read each chunk back as soon as it is written, so
        // only the last chunk's copy trails the lane's compute
        GemmCapScope cap(e->gemm_cap);
        err = pass_in_chunks(e, lane, e->launches[op.index], split_io, s);
      } else {
        GemmCapScope cap(e->gemm_cap);
        // programmatic dependent launch between consecutive engine kernels: the
        // next GEMM's CTAs are placed (and run their prologue) during the
        // previous kernel's tail; griddepcontrol.wait in every kernel keeps the
        // data dependency (BI_ENGINE_PDL, default 1)
        PdlScope pdl(engine_pdl());
        const GemmLaunchRec& L = e->launches[op.index];
        err = launch_gemm(e->descs.data() + L.first, e->d_descs + L.first, L.count, s);
      }
      if (err != cudaSuccess) return err;
    }
    if (after_first && stepid == first) {
      cudaError_t err = cudaEventRecord(after_first, s);
      if (err != cudaSuccess) return err;
    }
    if (e->timeline) {
      cudaError_t err = cudaEventRecordWithFlags(e->tl_ev[(size_t)lane * (e->nsteps + 1) + stepid], s,
                                                 cudaEventRecordExternal);
      if (err != cudaSuccess) return err;
    }
  }
  return cudaSuccess;
}

// Optional host I/O around a step range: per-matrix H2D on a copy stream,
// M_inv zero-fill per lane, per-matrix D2H as soon as its lane finishes.
struct HostIO {
  const double* in;
  int64_t ld_in, s_in;
  double* out;
  int64_t ld_out, s_out;
  bool split_out = false;  // page-locked output of a full Eq. 7 run: read back in two halves
};

// Read-back of the quads of the top level: diag = the two diagonal quads (final
// before the top-level up/down pass of the last step), else the two
// off-diagonal quads (final after it).
// Row-chunked last pass with per-chunk read-back (see enqueue_lane).  Each
// descriptor's output lies in M_inv; rows [r0, r1) of every descriptor form
// chunk c, copied to the host rows at the same coordinates.
static cudaError_t pass_in_chunks(bi_engine* e, int lane, const GemmLaunchRec& L, const HostIO* io,
                                  cudaStream_t s) {
  cudaError_t err = cudaSuccess;
  const int C = out_chunks();
  for (int c = 0; c < C && err == cudaSuccess; ++c) {
    GemmDesc d[kGemmInline];
    int nd = 0;
    for (int i = 0; i < L.count; ++i) {
      GemmDesc x = e->descs[L.first + i];
      const int r0 = (int)((int64_t)x.M * c / C), r1 = (int)((int64_t)x.M * (c + 1) / C);
      if (r1 <= r0) continue;
      x.A += (int64_t)r0 * x.lda;
      if (x.C) x.C += (int64_t)r0 * x.ldc;
      x.D += (int64_t)r0 * x.ldd;
      x.M = r1 - r0;
      d[nd++] = x;
    }
    if (nd == 0) continue;
    finalize_descs(d, nd);
    err = launch_gemm(d, nullptr, nd, s);
    if (err == cudaSuccess) err = cudaEventRecord(e->ev_chunk[lane][c], s);
    if (err == cudaSuccess) err = cudaStreamWaitEvent(e->d2h_stream[lane], e->ev_chunk[lane][c], 0);
    for (int i = 0; i < nd && err == cudaSuccess; ++i)
      for (int b = 0; b < d[i].batch && err == cudaSuccess; ++b) {
        const double* dev = d[i].D + (int64_t)b * d[i].sD;
        const int64_t off = dev - e->Minv;  // inside matrix z's M_inv
        const int64_t z = off / e->si, rem = off - z * e->si, row = rem / e->ldi, col = rem - row * e->ldi;
        err = cudaMemcpy2DAsync(io->out + z * io->s_out + row * io->ld_out + col, io->ld_out * 8, dev,
                                d[i].ldd * 8, (size_t)d[i].N * 8, (size_t)d[i].M, cudaMemcpyDeviceToHost,
                                e->d2h_stream[lane]);
      }
  }
  return err;
}

static cudaError_t copy_top_quads(bi_engine* e, int lane, const HostIO* io, bool diag, cudaStream_t st) {
  cudaError_t err = cudaSuccess;
  const int mid = e->nb / 2;
  const int64_t h0 = e->off[mid], h1 = e->n - e->off[mid];
  for (int z = e->zlo[lane]; z < e->zhi[lane] && err == cudaSuccess; ++z) {
    for (int part = 0; part < 2 && err == cudaSuccess; ++part) {
      // diag: (0,0) [h0 x h0] and (h0,h0) [h1 x h1]; off: (0,h0) [h0 x h1] and (h0,0) [h1 x h0]
      const int64_t r0 = part == 0 ? 0 : h0;
      const int64_t c0 = diag ? r0 : (part == 0 ? h0 : 0);
      const int64_t rows = part == 0 ? h0 : h1;
      const int64_t cols = diag ? rows : (part == 0 ? h1 : h0);
      err = cudaMemcpy2DAsync(io->out + (int64_t)z * io->s_out + r0 * io->ld_out + c0, io->ld_out * 8,
                              e->Minv + (int64_t)z * e->si + r0 * e->ldi + c0, e->ldi * 8, cols * 8, rows,
                              cudaMemcpyDeviceToHost, st);
    }
  }
  return err;
}

static cudaError_t lane_io_pre(bi_engine* e, int lane, cudaStream_t ls, int first, const HostIO* io) {
  cudaError_t err = cudaSuccess;
  for (int z = e->zlo[lane]; z < e->zhi[lane] && err == cudaSuccess; ++z) {
    if (io && first == 1 && e->schedule == BI_SCHEDULE_EQ7)
      err = cudaMemset2DAsync(e->Minv + (int64_t)z * e->si, e->ldi * 8, 0, e->n * 8, e->n, ls);
  }
  return err;
}

static cudaError_t lane_io_post(bi_engine* e, int lane, cudaStream_t ls, const HostIO* io) {
  cudaError_t err = cudaSuccess;
  if (!io || !io->out) return err;
  if (io->split_out) {  // the off-diagonal top quads, after the lane's last op
    // (the lane stream is joined through the read-back stream either way)
    err = cudaEventRecord(e->ev_d2h_b[lane], ls);
    if (err == cudaSuccess) err = cudaStreamWaitEvent(e->d2h_stream[lane], e->ev_d2h_b[lane], 0);
    const auto& ops = e->lane_ops[lane][e->nsteps];
    const bool chunked = !ops.empty() && ops.back().kind == 1 && e->launches[ops.back().index].count <= kGemmInline;
    if (err == cudaSuccess && !chunked) err = copy_top_quads(e, lane, io, false, e->d2h_stream[lane]);
    return err;
  }
  for (int z = e->zlo[lane]; z < e->zhi[lane] && err == cudaSuccess; ++z)
    err = cudaMemcpy2DAsync(io->out + (int64_t)z * io->s_out, io->ld_out * 8, e->Minv + (int64_t)z * e->si,
                            e->ldi * 8, e->n * 8, e->n, cudaMemcpyDeviceToHost, ls);
  return err;
}

static cudaError_t enqueue_steps(bi_engine* e, int first, int last, cudaStream_t s, int mask = 3,
                                 const HostIO* io = nullptr) {
  cudaError_t err = cudaSuccess;
  cudaEvent_t last_h2d = nullptr;  // the copy stream's final piece (joined into `s` at the end)
  e->set_policy(io && io->out ? 1 : 0);
  const bool fork = e->nlanes > 1 || (io && io->in);
  if (e->timeline) err = cudaEventRecordWithFlags(e->tl_start, s, cudaEventRecordExternal);
  if (fork && err == cudaSuccess) err = cudaEventRecord(e->ev_fork, s);
  if (io && io->in && err == cudaSuccess) {
    // Input in level order across the batch: every matrix's diagonal blocks
    // (all step 1 reads), then level by level the quads' off-diagonal B and
    // C blocks (first read by step 2^l).  Lanes start after a few MB instead
    // of after their whole matrix, and the rest streams under the compute.
    err = cudaStreamWaitEvent(e->copy_stream, e->ev_fork, 0);
    auto copy_block = [&](int z, int r0, int r1, int c0, int c1) {
      const int64_t ro = e->off[r0], co = e->off[c0];
      return cudaMemcpy2DAsync(const_cast<double*>(e->M) + (int64_t)z * e->sm + ro * e->ldm + co, e->ldm * 8,
                               io->in + (int64_t)z * io->s_in + ro * io->ld_in + co, io->ld_in * 8,
                               (e->off[c1] - co) * 8, e->off[r1] - ro, cudaMemcpyHostToDevice, e->copy_stream);
    };
    // (matrix, level) pieces in order of the step that first needs them: lane
    // l starts ~l steps late (skew), and reads level lv at step 2^lv
    std::vector<std::pair<int, int>> order;  // (z, lv)
    for (int lv = 0; lv <= e->k; ++lv)
      for (int z = 0; z < e->Z; ++z) order.push_back({z, lv});
    auto lane_of = [&](int z) {
      int l = 0;
      while (l + 1 < e->nlanes && z >= e->zhi[l]) ++l;
      return l;
    };
    std::stable_sort(order.begin(), order.end(), [&](const std::pair<int, int>& x, const std::pair<int, int>& y) {
      return lane_of(x.first) + (1 << x.second) < lane_of(y.first) + (1 << y.second);
    });
    for (const auto& zl : order) {
      const int z = zl.first, lv = zl.second;
      if (err != cudaSuccess) break;
      {
        if (lv == 0) {
          for (int p = 0; p < e->nb && err == cudaSuccess; ++p) err = copy_block(z, p, p + 1, p, p + 1);
        } else {
          for (int g = 0; g < (e->nb >> lv) && err == cudaSuccess; ++g) {
            const int first = g << lv, mid = first + (1 << (lv - 1)), last = (g + 1) << lv;
            err = copy_block(z, first, mid, mid, last);
            if (err == cudaSuccess) err = copy_block(z, mid, last, first, mid);
          }
        }
        if (err == cudaSuccess) err = cudaEventRecord(e->ev_h2d[(size_t)z * (e->k + 1) + lv], e->copy_stream);
        last_h2d = e->ev_h2d[(size_t)z * (e->k + 1) + lv];
      }
    }
  }
  // Lanes: lane l runs on its own stream, starting after lane l-1 completes
  // its first step (a one-step skew per lane); all lanes join back into `s`.
  for (int l = 0; l < e->nlanes && err == cudaSuccess; ++l) {
    cudaStream_t ls = l == 0 ? s : e->aux_stream[l];
    if (l > 0) {
      err = cudaStreamWaitEvent(ls, e->ev_fork, 0);
      if (err == cudaSuccess && e->skew_mode == 1) err = cudaStreamWaitEvent(ls, e->ev_skew[l - 1], 0);
      if (err == cudaSuccess && e->skew_mode == 2) err = cudaStreamWaitEvent(ls, e->ev_skew[0], 0);
    }
    if (err == cudaSuccess) err = lane_io_pre(e, l, ls, first, io);
    if (err == cudaSuccess)
      err = enqueue_lane(e, l, first, last, ls, mask, e->nlanes > 1 ? e->ev_skew[l] : nullptr, io && io->in,
                         (io && io->split_out) ? io : nullptr);
  }
  // read-back after every lane is enqueued (a pageable D2H blocks the host)
  const bool split = io && io->split_out;
  for (int l = 0; l < e->nlanes && err == cudaSuccess; ++l) {
    cudaStream_t ls = l == 0 ? s : e->aux_stream[l];
    err = lane_io_post(e, l, ls, io);
    if (err == cudaSuccess && (l > 0 || split)) err = cudaEventRecord(e->ev_join[l], split ? e->d2h_stream[l] : ls);
  }
  for (int l = split ? 0 : 1; l < e->nlanes && err == cudaSuccess; ++l)
    err = cudaStreamWaitEvent(s, e->ev_join[l], 0);
  // a run that stops early never waits on its later input pieces: join the
  // copy stream explicitly (graph capture rejects unjoined work)
  if (err == cudaSuccess && last_h2d) err = cudaStreamWaitEvent(s, last_h2d, 0);
  return err;
}

static bool is_pinned(const void* p) {
  if (!p) return true;
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

static int run_impl(bi_engine* e, int first_step, int last_step, int use_graph, cudaStream_t s, const HostIO* io) {
  e->last_stream = s;
  e->last_first = first_step;
  e->last_last = last_step;
  if (io && !(is_pinned(io->in) && is_pinned(io->out))) use_graph = 0;  // pageable copies cannot be captured
  HostIO io2;
  if (io) {
    io2 = *io;
    // page-locked output of a full Eq. 7 run: the diagonal top quads are read
    // back during the last step's top-level pass (a pageable D2H would block
    // the host before the later lanes are enqueued)
    io2.split_out = io->out && is_pinned(io->out) && io->out != nullptr && e->schedule == BI_SCHEDULE_EQ7 &&
                    e->nb >= 2 && last_step == e->nsteps;
    io = &io2;
  }
  if (!use_graph) {
    BI_CUDA_TRY(enqueue_steps(e, first_step, last_step, s, 3, io));
    return 0;
  }
  GraphKey key{first_step, last_step, io ? io->in : nullptr, io ? io->out : nullptr,
               io ? io->ld_in : 0, io ? io->s_in : 0, io ? io->ld_out : 0, io ? io->s_out : 0};
  auto it = e->graphs.find(key);
  if (it == e->graphs.end()) {
    if (!e->capture_stream) BI_CUDA_TRY(cudaStreamCreateWithFlags(&e->capture_stream, cudaStreamNonBlocking));
    BI_CUDA_TRY(cudaStreamBeginCapture(e->capture_stream, cudaStreamCaptureModeThreadLocal));
    cudaError_t err = enqueue_steps(e, first_step, last_step, e->capture_stream, 3, io);
    cudaGraph_t graph = nullptr;
    cudaError_t err2 = cudaStreamEndCapture(e->capture_stream, &graph);
    if (err != cudaSuccess || err2 != cudaSuccess) {
      if (graph) cudaGraphDestroy(graph);
      set_error(std::string("graph capture failed: ") + cudaGetErrorString(err != cudaSuccess ? err : err2));
      return 3;
    }
    cudaGraphExec_t exec = nullptr;
    cudaError_t err3 = cudaGraphInstantiateWithFlags(&exec, graph, cudaGraphInstantiateFlagUseNodePriority);
    cudaGraphDestroy(graph);
    BI_CUDA_TRY(err3);
    if (e->graphs.size() >= 16) {  // bound the cache
      cudaGraphExecDestroy(e->graphs.begin()->second);
      e->graphs.erase(e->graphs.begin());
    }
    it = e->graphs.emplace(key, exec).first;
  }
  BI_CUDA_TRY(cudaGraphLaunch(it->second, s));
  return 0;
}

extern "C" int bi_engine_run(bi_engine* e, int first_step, int last_step, int use_graph, void* stream) {
  BI_REQUIRE(e && e->bound, "engine not bound");
  BI_REQUIRE(e->P == 1, "a column-sharded engine runs through bi_engine_run_ops / bi_shard_group_run");
  BI_REQUIRE(first_step >= 1 && last_step <= e->nsteps && first_step <= last_step,
             "stepid outside 1..N_s");
  return run_impl(e, first_step, last_step, use_graph, static_cast<cudaStream_t>(stream), nullptr);
}

// ---------------------------------------------------------------------------
// Pageable host buffers (a plain NumPy array through the drop-in call).
// A pageable cudaMemcpy runs at ~11 GB/s and cannot be captured; copying the
// whole input into page-locked memory first serialises a host copy, the DMA
// and the compute.  Instead the input moves in NEED ORDER, level by level
// (step 1 reads only the diagonal blocks, step 2^l first reads the level-l
// quads' B and C blocks): the host copies level l into engine-owned
// page-locked staging (all host threads), DMAs it on the copy stream, and
// the steps [2^l, 2^(l+1)) -- each range one cached CUDA graph -- wait only
// for that level.  While the device runs range l the host stages level l+1.
// A page-locked output is read back inside the last range's graph (top
// quads during the last pass); a pageable output goes through page-locked
// staging and is copied out after the stream drains.
// ---------------------------------------------------------------------------
namespace {

struct Region {
  char* dst;
  const char* src;
  int64_t dld, sld;  // bytes
  int64_t rows, bytes;
};

// Persistent host worker threads for the staging copies (spawning a thread
// per piece cost ~1-2 ms per call at cfg2 size).  run(T, f) runs f(0..T-1),
// f(0) on the caller, and returns when all are done.  One run at a time.
class CopyPool {
 public:
  void run(int T, const std::function<void(int)>& f) {
    std::lock_guard<std::mutex> one(run_mu_);
    {
      std::unique_lock<std::mutex> lk(mu_);
      while ((int)threads_.size() < T - 1) {
        const int id = (int)threads_.size();
        threads_.emplace_back([this, id] { loop(id); });
      }
      job_ = &f;
      active_ = T - 1;
      pending_ = T - 1;
      ++gen_;
    }
    cv_.notify_all();
    f(0);
    std::unique_lock<std::mutex> lk(mu_);
    done_.wait(lk, [this] { return pending_ == 0; });
    job_ = nullptr;
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto& t : threads_) t.join();
  }

 private:
  void loop(int id) {
    int seen = 0;
    for (;;) {
      const std::function<void(int)>* job = nullptr;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return gen_ != seen; });
        seen = gen_;
        if (stop_) return;
        if (id >= active_) continue;
        job = job_;
      }
      (*job)(id + 1);
      std::lock_guard<std::mutex> lk(mu_);
      if (--pending_ == 0) done_.notify_one();
    }
  }
  std::mutex run_mu_, mu_;
  std::condition_variable cv_, done_;
  std::vector<std::thread> threads_;
  const std::function<void(int)>* job_ = nullptr;
  int active_ = 0, pending_ = 0, gen_ = 0;
  bool stop_ = false;
};

static void copy_pool_run(int T, const std::function<void(int)>& f) {
  static CopyPool* pool = new CopyPool();  // process lifetime (never joined at exit)
  pool->run(T, f);
}

// dst/src 2-D regions copied by up to `threads` host threads, split by rows
static void par_copy(const std::vector<Region>& regs, int threads) {
  int64_t total = 0;
  for (const Region& r : regs) total += r.rows * r.bytes;
  if (total == 0) return;
  const int64_t per = 1 << 20;  // >= 1 MB per thread
  int T = (int)std::max<int64_t>(1, std::min<int64_t>(threads, total / per));
  if (T == 1) {
    for (const Region& r : regs)
      for (int64_t i = 0; i < r.rows; ++i) std::memcpy(r.dst + i * r.dld, r.src + i * r.sld, r.bytes);
    return;
  }
  // contiguous byte ranges of the concatenated rows, one per thread
  auto work = [&](int t) {
    const int64_t b0 = total * t / T, b1 = total * (t + 1) / T;
    int64_t pos = 0;
    for (const Region& r : regs) {
      const int64_t sz = r.rows * r.bytes;
      if (pos + sz <= b0) {
        pos += sz;
        continue;
      }
      if (pos >= b1) break;
      for (int64_t i = 0; i < r.rows; ++i) {
        const int64_t r0 = pos + i * r.bytes, r1 = r0 + r.bytes;
        const int64_t lo = std::max(r0, b0), hi = std::min(r1, b1);
        if (lo < hi) std::memcpy(r.dst + i * r.dld + (lo - r0), r.src + i * r.sld + (lo - r0), hi - lo);
      }
      pos += sz;
    }
  };
  copy_pool_run(T, work);
}

static int host_threads() {
  static const int n = [] {
    const char* v = getenv("BI_HOST_THREADS");
    int t = v ? atoi(v) : (int)std::thread::hardware_concurrency();
    return std::max(1, std::min(t, 32));
  }();
  return n;
}

}  // namespace

// input blocks first read at level lv: the diagonal blocks (lv = 0) or the
// level-lv quads' off-diagonal B and C blocks
static void level_blocks(const bi_engine* e, int lv, std::vector<std::array<int, 4>>& out) {
  out.clear();
  if (lv == 0) {
    for (int p = 0; p < e->nb; ++p) out.push_back({p, p + 1, p, p + 1});
    return;
  }
  for (int g = 0; g < (e->nb >> lv); ++g) {
    const int first = g << lv, mid = first + (1 << (lv - 1)), last = (g + 1) << lv;
    out.push_back({first, mid, mid, last});
    out.push_back({mid, last, first, mid});
  }
}

static int run_host_pipelined(bi_engine* e, const double* in, int64_t ld_in, int64_t s_in, double* out,
                              int64_t ld_out, int64_t s_out, int last_step, int use_graph, cudaStream_t s) {
  const bool in_pinned = is_pinned(in), out_pinned = is_pinned(out);
  const int64_t n = e->n;
  const int T = host_threads();
  const int64_t in_bytes = (int64_t)e->Z * n * e->ldm * 8, out_bytes = (int64_t)e->Z * n * e->ldi * 8;
  if (in && !in_pinned && e->stage_in_bytes < in_bytes) {
    if (e->stage_in) cudaFreeHost(e->stage_in);
    e->stage_in = nullptr;
    e->stage_in_bytes = 0;
    BI_CUDA_TRY(cudaHostAlloc((void**)&e->stage_in, in_bytes, cudaHostAllocPortable));
    e->stage_in_bytes = in_bytes;
    for (auto& kv : e->graphs) cudaGraphExecDestroy(kv.second);  // keyed by buffer addresses
    e->graphs.clear();
  }
  if (out && !out_pinned && e->stage_out_bytes < out_bytes) {
    if (e->stage_out) cudaFreeHost(e->stage_out);
    e->stage_out = nullptr;
    e->stage_out_bytes = 0;
    BI_CUDA_TRY(cudaHostAlloc((void**)&e->stage_out, out_bytes, cudaHostAllocPortable));
    e->stage_out_bytes = out_bytes;
  }
  // staged buffers use the device layouts ([Z][n][ldm] / [Z][n][ldi])
  const double* src = in;
  int64_t src_ld = ld_in, src_s = s_in;
  if (in && !in_pinned) {
    src = e->stage_in;
    src_ld = e->ldm;
    src_s = n * e->ldm;
  }
  double* dst = out;
  int64_t dst_ld = ld_out, dst_s = s_out;
  if (out && !out_pinned) {
    dst = e->stage_out;
    dst_ld = e->ldi;
    dst_s = n * e->ldi;
  }
  for (int lv = 0; lv <= e->k; ++lv)
    if (!e->ev_level[lv]) BI_CUDA_TRY(cudaEventCreateWithFlags(&e->ev_level[lv], cudaEventDisableTiming));
  for (int z = 0; z < e->Z; ++z)  // fresh M_inv (storage.fresh_state)
    BI_CUDA_TRY(cudaMemset2DAsync(e->Minv + (int64_t)z * e->si, e->ldi * 8, 0, n * 8, n, s));
  HostIO io{nullptr, 0, 0, nullptr, 0, 0};
  std::vector<std::array<int, 4>> blocks;
  int done = 0;  // last step enqueued
  static const bool trace = getenv("BI_PIPE_TRACE") != nullptr;
  auto now_us = [] {
    return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
  };
  const double t_start = trace ? now_us() : 0.0;
  for (int lv = 0; lv <= e->k; ++lv) {
    const double t_lv = trace ? now_us() : 0.0;
    if (in) {
      level_blocks(e, lv, blocks);
      // the level's (matrix, block) pieces in up to 4 chunks: the DMA of a
      // chunk runs while the host stages the next one
      std::vector<std::pair<int, std::array<int, 4>>> pieces;
      for (int z = 0; z < e->Z; ++z)
        for (const auto& b : blocks) pieces.push_back({z, b});
      const int nch = std::min<int>(4, (int)pieces.size());
      for (int c = 0; c < nch; ++c) {
        const size_t p0 = pieces.size() * c / nch, p1 = pieces.size() * (c + 1) / nch;
        if (!in_pinned) {  // host: user rows -> staging, same coordinates
          std::vector<Region> regs;
          for (size_t i = p0; i < p1; ++i) {
            const int z = pieces[i].first;
            const auto& b = pieces[i].second;
            const int64_t ro = e->off[b[0]], co = e->off[b[2]];
            regs.push_back({(char*)(e->stage_in + (int64_t)z * src_s + ro * src_ld + co),
                            (const char*)(in + (int64_t)z * s_in + ro * ld_in + co), src_ld * 8, ld_in * 8,
                            e->off[b[1]] - ro, (e->off[b[3]] - co) * 8});
          }
          par_copy(regs, T);
        }
        for (size_t i = p0; i < p1; ++i) {
          const int z = pieces[i].first;
          const auto& b = pieces[i].second;
          const int64_t ro = e->off[b[0]], co = e->off[b[2]];
          BI_CUDA_TRY(cudaMemcpy2DAsync(const_cast<double*>(e->M) + (int64_t)z * e->sm + ro * e->ldm + co,
                                        e->ldm * 8, src + (int64_t)z * src_s + ro * src_ld + co, src_ld * 8,
                                        (e->off[b[3]] - co) * 8, e->off[b[1]] - ro, cudaMemcpyHostToDevice,
                                        e->copy_stream));
        }
      }
      if (trace) fprintf(stderr, "[pipe] level %d host copy %.0f us (t=%.0f)\n", lv, now_us() - t_lv, now_us() - t_start);
      BI_CUDA_TRY(cudaEventRecord(e->ev_level[lv], e->copy_stream));
      BI_CUDA_TRY(cudaStreamWaitEvent(s, e->ev_level[lv], 0));
    } else if (lv < e->k) {
      continue;  // input already resident: one range
    }
    if (done >= last_step) continue;  // stop_after_step: later levels are loaded, not run
    // steps [2^lv, 2^(lv+1)) first read level lv (Eq. 7); pivot-A reads
    // everything in its single step
    int first = done + 1, last;
    if (e->schedule == BI_SCHEDULE_PIVOT_A) {
      if (in && lv < e->k) continue;
      last = 1;
    } else {
      last = lv == e->k || !in ? e->nsteps : (1 << (lv + 1)) - 1;
    }
    last = std::min(last, last_step);
    const bool final_range = last == last_step;
    io.out = final_range ? dst : nullptr;
    io.ld_out = dst_ld;
    io.s_out = dst_s;
    int rc = run_impl(e, first, last, use_graph, s, io.out ? &io : nullptr);
    if (rc) return rc;
    if (trace) fprintf(stderr, "[pipe] steps %d-%d enqueued (t=%.0f)\n", first, last, now_us() - t_start);
    done = last;
  }
  e->last_first = 1;
  e->last_last = last_step;
  if (out && !out_pinned) {  // drain, then staging -> the caller's rows
    BI_CUDA_TRY(cudaStreamSynchronize(s));
    std::vector<Region> regs;
    for (int z = 0; z < e->Z; ++z)
      regs.push_back({(char*)(out + (int64_t)z * s_out), (const char*)(dst + (int64_t)z * dst_s), ld_out * 8,
                      dst_ld * 8, n, n * 8});
    par_copy(regs, T);
  }
  return 0;
}

// Host buffers above the staging limit (cfg5: 34 GB each way): the same
// need-ordered level pipeline through a bounded page-locked ring (4 x 256 MB)
// -- the host packs pieces into a slot (all host threads), the copy stream
// DMAs the slot, and a slot is refilled once its DMA event has fired.  The
// inverse comes back through the same ring after the run (DMA of chunk i+1
// under the host copy of chunk i).
static int run_host_ring(bi_engine* e, const double* in, int64_t ld_in, int64_t s_in, double* out,
                         int64_t ld_out, int64_t s_out, int last_step, int use_graph, cudaStream_t s) {
  constexpr int R = bi_engine::kRingSlots;
  if (!e->ring_bytes) {
    const char* v = getenv("BI_RING_MB");
    e->ring_bytes = (int64_t)((v ? atof(v) : 256.0) * (1 << 20));
    e->ring_bytes = std::max<int64_t>(round_up(e->ring_bytes, 256), 256);
  }
  const int64_t RB = e->ring_bytes;
  const int64_t n = e->n;
  const int T = host_threads();
  for (int i = 0; i < R; ++i) {
    if (!e->ring[i]) BI_CUDA_TRY(cudaHostAlloc((void**)&e->ring[i], RB, cudaHostAllocPortable));
    if (!e->ring_ev[i]) BI_CUDA_TRY(cudaEventCreateWithFlags(&e->ring_ev[i], cudaEventDisableTiming));
    e->ring_busy[i] = false;
  }
  for (int lv = 0; lv <= e->k; ++lv)
    if (!e->ev_level[lv]) BI_CUDA_TRY(cudaEventCreateWithFlags(&e->ev_level[lv], cudaEventDisableTiming));
  for (int z = 0; z < e->Z; ++z)
    BI_CUDA_TRY(cudaMemset2DAsync(e->Minv + (int64_t)z * e->si, e->ldi * 8, 0, n * 8, n, s));
  const bool in_pinned = is_pinned(in), out_pinned = is_pinned(out);
  int slot = 0;
  int64_t fill = 0;
  struct Q {
    char* dev;
    int64_t dld, off, rows, bytes;
  };
  std::vector<Q> queued;
  std::vector<Region> regs;
  auto flush = [&]() -> cudaError_t {
    if (queued.empty()) return cudaSuccess;
    par_copy(regs, T);  // host rows -> the slot
    regs.clear();
    for (const Q& q : queued) {
      cudaError_t err = cudaMemcpy2DAsync(q.dev, q.dld, e->ring[slot] + q.off, q.bytes, q.bytes, q.rows,
                                          cudaMemcpyHostToDevice, e->copy_stream);
      if (err != cudaSuccess) return err;
    }
    queued.clear();
    cudaError_t err = cudaEventRecord(e->ring_ev[slot], e->copy_stream);
    e->ring_busy[slot] = true;
    slot = (slot + 1) % R;
    fill = 0;
    if (err == cudaSuccess && e->ring_busy[slot]) err = cudaEventSynchronize(e->ring_ev[slot]);  // slot free again
    e->ring_busy[slot] = false;
    return err;
  };
  auto stage = [&](const char* host, int64_t hld, int64_t rows, int64_t bytes, char* dev, int64_t dld) -> cudaError_t {
    for (int64_t r = 0; r < rows;) {
      const int64_t fit = fill >= RB ? 0 : (RB - fill) / bytes;
      if (fit <= 0) {
        cudaError_t err = flush();
        if (err != cudaSuccess) return err;
        if (RB / bytes == 0) return cudaErrorInvalidValue;  // a row larger than a slot
        continue;
      }
      const int64_t take = std::min(fit, rows - r);
      regs.push_back({e->ring[slot] + fill, host + r * hld, bytes, hld, take, bytes});
      queued.push_back({dev + r * dld, dld, fill, take, bytes});
      fill += round_up(take * bytes, 256);
      r += take;
    }
    return cudaSuccess;
  };
  std::vector<std::array<int, 4>> blocks;
  int done = 0;
  for (int lv = 0; lv <= e->k; ++lv) {
    if (in) {
      level_blocks(e, lv, blocks);
      for (int z = 0; z < e->Z; ++z)
        for (const auto& b : blocks) {
          const int64_t ro = e->off[b[0]], co = e->off[b[2]], rows = e->off[b[1]] - ro, bytes = (e->off[b[3]] - co) * 8;
          const double* h = in + (int64_t)z * s_in + ro * ld_in + co;
          double* d = const_cast<double*>(e->M) + (int64_t)z * e->sm + ro * e->ldm + co;
          if (in_pinned) {
            BI_CUDA_TRY(cudaMemcpy2DAsync(d, e->ldm * 8, h, ld_in * 8, bytes, rows, cudaMemcpyHostToDevice,
                                          e->copy_stream));
          } else {
            BI_CUDA_TRY(stage((const char*)h, ld_in * 8, rows, bytes, (char*)d, e->ldm * 8));
          }
        }
      BI_CUDA_TRY(flush());
      BI_CUDA_TRY(cudaEventRecord(e->ev_level[lv], e->copy_stream));
      BI_CUDA_TRY(cudaStreamWaitEvent(s, e->ev_level[lv], 0));
    } else if (lv < e->k) {
      continue;
    }
    if (done >= last_step) continue;
    int first = done + 1, last;
    if (e->schedule == BI_SCHEDULE_PIVOT_A) {
      if (in && lv < e->k) continue;
      last = 1;
    } else {
      last = lv == e->k || !in ? e->nsteps : (1 << (lv + 1)) - 1;
    }
    last = std::min(last, last_step);
    int rc = run_impl(e, first, last, use_graph, s, nullptr);
    if (rc) return rc;
    done = last;
  }
  e->last_first = 1;
  e->last_last = last_step;
  if (!out) return 0;
  // read-back: after the run, M_inv rows in ring-sized chunks
  BI_CUDA_TRY(cudaEventRecord(e->ev_fork, s));
  BI_CUDA_TRY(cudaStreamWaitEvent(e->copy_stream, e->ev_fork, 0));
  if (out_pinned) {
    for (int z = 0; z < e->Z; ++z)
      BI_CUDA_TRY(cudaMemcpy2DAsync(out + (int64_t)z * s_out, ld_out * 8, e->Minv + (int64_t)z * e->si, e->ldi * 8,
                                    n * 8, n, cudaMemcpyDeviceToHost, e->copy_stream));
    BI_CUDA_TRY(cudaEventRecord(e->ev_fork, e->copy_stream));
    BI_CUDA_TRY(cudaStreamWaitEvent(s, e->ev_fork, 0));
    return 0;
  }
  const int64_t rows_per = std::max<int64_t>(1, RB / (n * 8));
  struct C {
    int z;
    int64_t r0, rows;
    int slot;
  };
  std::vector<C> inflight;
  int sl = 0;
  auto drain_one = [&]() -> cudaError_t {
    const C c = inflight.front();
    inflight.erase(inflight.begin());
    cudaError_t err = cudaEventSynchronize(e->ring_ev[c.slot]);
    if (err != cudaSuccess) return err;
    std::vector<Region> rg{{(char*)(out + (int64_t)c.z * s_out + c.r0 * ld_out), e->ring[c.slot], ld_out * 8, n * 8,
                            c.rows, n * 8}};
    par_copy(rg, T);
    return cudaSuccess;
  };
  for (int z = 0; z < e->Z; ++z)
    for (int64_t r0 = 0; r0 < n; r0 += rows_per) {
      if ((int)inflight.size() == R) BI_CUDA_TRY(drain_one());
      const int64_t rows = std::min(rows_per, n - r0);
      BI_CUDA_TRY(cudaMemcpy2DAsync(e->ring[sl], n * 8, e->Minv + (int64_t)z * e->si + r0 * e->ldi, e->ldi * 8,
                                    n * 8, rows, cudaMemcpyDeviceToHost, e->copy_stream));
      BI_CUDA_TRY(cudaEventRecord(e->ring_ev[sl], e->copy_stream));
      inflight.push_back({z, r0, rows, sl});
      sl = (sl + 1) % R;
    }
  while (!inflight.empty()) BI_CUDA_TRY(drain_one());
  for (int i = 0; i < R; ++i) e->ring_busy[i] = false;
  return 0;
}

extern "C" int bi_engine_run_host(bi_engine* e, const double* host_in, int64_t ld_in, int64_t stride_in,
                                  double* host_out, int64_t ld_out, int64_t stride_out, int first_step,
                                  int last_step, int use_graph, void* stream) {
  BI_REQUIRE(e && e->bound, "engine not bound");
  BI_REQUIRE(e->P == 1, "a column-sharded engine runs through bi_engine_run_ops / bi_shard_group_run");
  BI_REQUIRE(first_step >= 1 && last_step <= e->nsteps && first_step <= last_step,
             "stepid outside 1..N_s");
  BI_REQUIRE(!host_in || (ld_in >= e->n && (e->Z == 1 || stride_in >= ld_in * e->n)),
             "host input leading dimension / stride too small");
  BI_REQUIRE(!host_out || (ld_out >= e->n && (e->Z == 1 || stride_out >= ld_out * e->n)),
             "host output leading dimension / stride too small");
  BI_REQUIRE(!host_in || first_step == 1, "host input requires first_step == 1");
  const int64_t stage_bytes = (int64_t)e->Z * e->n * std::max(e->ldm, e->ldi) * 8;
  static const int64_t stage_limit = [] {  // larger pageable buffers: unstaged pageable copies
    const char* v = getenv("BI_STAGE_LIMIT_GB");
    return (int64_t)((v ? atof(v) : 8.0) * (1 << 30));
  }();
  if (((host_in && !is_pinned(host_in)) || (host_out && !is_pinned(host_out))) && first_step == 1) {
    if (stage_bytes <= stage_limit)
      return run_host_pipelined(e, host_in, ld_in, stride_in, host_out, ld_out, stride_out, last_step, use_graph,
                                static_cast<cudaStream_t>(stream));
    return run_host_ring(e, host_in, ld_in, stride_in, host_out, ld_out, stride_out, last_step, use_graph,
                         static_cast<cudaStream_t>(stream));
  }
  HostIO io{host_in, ld_in, stride_in, host_out, ld_out, stride_out};
  return run_impl(e, first_step, last_step, use_graph, static_cast<cudaStream_t>(stream), &io);
}

extern "C" int bi_engine_run_phase(bi_engine* e, int first_step, int last_step, int mask, void* stream) {
  BI_REQUIRE(e && e->bound, "engine not bound");
  BI_REQUIRE(e->P == 1, "a column-sharded engine runs through bi_engine_run_ops / bi_shard_group_run");
  BI_REQUIRE(first_step >= 1 && last_step <= e->nsteps && first_step <= last_step, "stepid outside 1..N_s");
  BI_REQUIRE(mask >= 1 && mask <= 3, "mask must be 1 (GEMM ops), 2 (leaf inversions) or 3");
  e->last_stream = static_cast<cudaStream_t>(stream);
  const bool tl = e->timeline;  // timeline events are recorded as graph (external) nodes only
  e->timeline = false;
  cudaError_t err = enqueue_steps(e, first_step, last_step, e->last_stream, mask);
  e->timeline = tl;
  BI_CUDA_TRY(err);
  return 0;
}

extern "C" int bi_engine_timeline(bi_engine* e, float* out_ms) {
  BI_REQUIRE(e && e->bound && out_ms, "engine not bound");
  BI_REQUIRE(e->timeline, "set BI_ENGINE_TIMELINE=1 before binding");
  BI_CUDA_TRY(cudaStreamSynchronize(e->last_stream));
  for (int l = 0; l < e->nlanes; ++l)
    for (int st = 0; st <= e->nsteps; ++st) {
      float v = -1.0f;
      if (st >= e->last_first && st <= e->last_last &&
          cudaEventElapsedTime(&v, e->tl_start, e->tl_ev[(size_t)l * (e->nsteps + 1) + st]) != cudaSuccess) {
        cudaGetLastError();
        v = -1.0f;
      }
      out_ms[(size_t)l * (e->nsteps + 1) + st] = v;
    }
  return 0;
}

extern "C" int bi_engine_launches(const bi_engine* e, int first_step, int last_step, int64_t out[3]) {
  BI_REQUIRE(e && e->bound && out, "engine not bound");
  BI_REQUIRE(first_step >= 1 && last_step <= e->nsteps, "stepid outside 1..N_s");
  int64_t gemm = 0, inv = 0;
  for (int lane = 0; lane < e->nlanes; ++lane)
  for (int stepid = first_step; stepid <= last_step; ++stepid)
    for (const Op& op : e->lane_ops[lane][stepid]) {
      if (op.kind == 2 || op.kind == 3) continue;  // copy / exchange, not a kernel
      if (op.kind == 1) {
        gemm += 1;
      } else {
        const InvRec& r = e->invs[op.index];
        int64_t k = 0, gm = 0;
        inv_group_launch_counts(r.g, &k, &gm);
        inv += k - gm;
        gemm += gm;
      }
    }
  out[0] = gemm + inv;
  out[1] = gemm;
  out[2] = inv;
  return 0;
}

extern "C" int bi_engine_status(bi_engine* e, int* fail_step, int* fail_quad, int* fail_matrix) {
  BI_REQUIRE(e && e->bound, "engine not bound");
  BI_CUDA_TRY(cudaStreamSynchronize(e->last_stream));
  std::vector<int> info(e->info_ints);
  BI_CUDA_TRY(cudaMemcpy(info.data(), e->info, info.size() * 4, cudaMemcpyDeviceToHost));
  if (fail_step) *fail_step = 0;
  if (fail_quad) *fail_quad = -1;
  if (fail_matrix) *fail_matrix = -1;
  // earliest executed diag step, then matrix, then block (engine.py:313-330 order)
  for (size_t di = 0; di < e->diag_steps.size(); ++di) {
    const int stepid = e->diag_steps[di];
    if (stepid < e->last_first || stepid > e->last_last) continue;
    int best_z = -1, best_p = -1;
    for (const InvRec& r : e->invs) {
      if (r.diag_step_index != (int)di) continue;
      for (int it = 0; it < r.g.count; ++it) {
        if (info[r.info_offset + it] == 0) continue;
        const int z = r.item_matrix[it], p = r.item_block[it];
        if (best_z < 0 || z < best_z || (z == best_z && p < best_p)) {
          best_z = z;
          best_p = p;
        }
      }
    }
    if (best_z >= 0) {
      if (fail_step) *fail_step = stepid;
      if (fail_quad) *fail_quad = best_p;
      if (fail_matrix) *fail_matrix = best_z;
      set_error("singular diagonal block");
      return 1;
    }
  }
  return 0;
}

extern "C" int bi_engine_counters(const bi_engine* e, int first_step, int last_step, double out[6]) {
  BI_REQUIRE(e && out, "null argument");
  BI_REQUIRE(first_step >= 1 && last_step <= e->nsteps, "stepid outside 1..N_s");
  double mult = 0, invs = 0, red = 0, gflops = 0, lflops = 0, gbytes = 0;
  const auto& off = e->off;
  if (e->schedule == BI_SCHEDULE_PIVOT_A) {  // invertor_by_a tallies: 6 multiplies (2 accumulating) per node
    std::function<void(int, int)> node = [&](int b0, int b1) {
      if (b1 - b0 == 1) {
        invs += 1;
        lflops += 2.0 * (double)e->sizes[b0] * e->sizes[b0] * e->sizes[b0];
        return;
      }
      const int mid = (b0 + b1) / 2;
      const double p = (double)(off[mid] - off[b0]), q = (double)(off[b1] - off[mid]);
      mult += 6;
      red += 2;
      gflops += 6.0 * p * q * (p + q);
      // T_b, T_c: read A and B / C, write; D += C T_b; C = D T_c; B = T_b D; A += T_b C
      gbytes += 8.0 * ((p * p + 2 * p * q) + (p * p + 2 * p * q) + (2 * p * q + 2 * q * q) +
                       (q * q + 2 * p * q) + (q * q + 2 * p * q) + (2 * p * q + 2 * p * p));
      node(b0, mid);
      node(mid, b1);
    };
    node(0, e->nb);
  }
  for (int stepid = first_step; stepid <= last_step && e->schedule == BI_SCHEDULE_EQ7; ++stepid) {
    StepAct a;
    loopid_decode(stepid, e->nb, &a);
    if (a.kind == 0 || a.kind == 2) {
      invs += e->nb;  // engine.py:317
      for (int64_t s : e->sizes) lflops += 2.0 * (double)s * s * s;
    }
    auto quads = [&](int lv, auto fn) {
      for (int g = 0; g < (e->nb >> lv); ++g) {
        const int first = g << lv, mid = first + (1 << (lv - 1)), last = (g + 1) << lv;
        fn((double)(off[mid] - off[first]), (double)(off[last] - off[mid]));
      }
    };
    if (a.kind == 1) {
      quads(a.sid, [&](double ha, double hd) {
        mult += 2;  // engine.py:344-345
        red += 2;
        gflops += 2.0 * (ha * ha * hd + hd * hd * ha + ha * hd * ha + hd * ha * hd);
        // R, L: read A^-1 / D^-1 and B / C, write R / L; S_D, S_A: read B L + A / C R + D, write
        gbytes += 8.0 * ((ha * ha + 2 * ha * hd) + (hd * hd + 2 * ha * hd) + (2 * ha * hd + 2 * ha * ha) +
                         (2 * ha * hd + 2 * hd * hd));
      });
    } else if (a.kind == 2) {
      for (int lv = 1; lv <= a.depth; ++lv)
        quads(lv, [&](double ha, double hd) {
          mult += 2;  // engine.py:411
          gflops += 2.0 * (hd * ha * ha + ha * hd * hd);
          gbytes += 8.0 * ((2 * ha * hd + ha * ha) + (2 * ha * hd + hd * hd));  // down, up
        });
    }
  }
  out[0] = mult;
  out[1] = invs;
  out[2] = red;
  out[3] = gflops * e->Z;
  out[4] = lflops * e->Z;
  out[5] = gbytes * e->Z;
  return 0;
}

extern "C" int bi_engine_tset_square(const bi_engine* e, int level, int quad, int matrix, double** ptr,
                                     int64_t* ld, int64_t* side) {
  BI_REQUIRE(e && e->bound, "engine not bound");
  BI_REQUIRE(e->schedule == BI_SCHEDULE_EQ7, "the pivot-A schedule keeps no T-sets");
  BI_REQUIRE(level >= 1 && level <= e->k && quad >= 0 && quad < (e->nb >> level) && matrix >= 0 &&
                 matrix < e->Z,
             "tset index out of range");
  const auto& s = e->tsq[level][quad];
  *ptr = e->T + (int64_t)matrix * e->t_matrix + s.off;
  *ld = s.ld;
  *side = s.side;
  return 0;
}

extern "C" int bi_engine_destroy(bi_engine* e) {
  if (e && !e->group_comms.empty()) shard_destroy_comms(e);
  delete e;
  return 0;
}

// ===========================================================================
// Column-sharded ranks: segments of local ops between exchanges
// ===========================================================================

extern "C" int bi_engine_shard_segments(const bi_engine* e, int first_step, int last_step, int* begin, int* end,
                                        int* xchg, int cap) {
  BI_REQUIRE(e && e->bound, "engine not bound");
  BI_REQUIRE(first_step >= 1 && last_step <= e->nsteps && first_step <= last_step, "stepid outside 1..N_s");
  int n = 0, b = e->step_first_op[first_step];
  const int stop = e->step_first_op[last_step + 1];
  for (int i = b; i <= stop; ++i) {
    const bool at_x = i < stop && e->flat[i].op.kind == 3;
    if (i == stop || at_x) {
      if (n < cap) {
        begin[n] = b;
        end[n] = i;
        xchg[n] = at_x ? e->flat[i].op.index : -1;
      }
      ++n;
      b = i + 1;
    }
  }
  return n;
}

static cudaError_t enqueue_flat(bi_engine* e, int b, int en, cudaStream_t s) {
  for (int i = b; i < en; ++i) {
    const Op& op = e->flat[i].op;
    cudaError_t err = cudaSuccess;
    if (op.kind == 0) {
      PriorityScope leaf_prio(e->leaf_priority ? e->leaf_priority : g_launch_priority);
      err = launch_inv_group(e->invs[op.index].g, s);
    } else if (op.kind == 1) {
      GemmCapScope cap(e->gemm_cap);
      const GemmLaunchRec& L = e->launches[op.index];
      err = launch_gemm(e->descs.data() + L.first, e->d_descs + L.first, L.count, s);
    }
    if (err != cudaSuccess) return err;
  }
  return cudaSuccess;
}

static int run_ops_impl(bi_engine* e, int b, int en, int use_graph, cudaStream_t s) {
  e->last_stream = s;
  if (b >= en) return 0;
  e->set_policy(0);
  if (!use_graph) {
    BI_CUDA_TRY(enqueue_flat(e, b, en, s));
    return 0;
  }
  auto key = std::make_pair(b, en);
  auto it = e->seg_graphs.find(key);
  if (it == e->seg_graphs.end()) {
    if (!e->capture_stream) BI_CUDA_TRY(cudaStreamCreateWithFlags(&e->capture_stream, cudaStreamNonBlocking));
    BI_CUDA_TRY(cudaStreamBeginCapture(e->capture_stream, cudaStreamCaptureModeThreadLocal));
    cudaError_t err = enqueue_flat(e, b, en, e->capture_stream);
    cudaGraph_t graph = nullptr;
    cudaError_t err2 = cudaStreamEndCapture(e->capture_stream, &graph);
    if (err != cudaSuccess || err2 != cudaSuccess) {
      if (graph) cudaGraphDestroy(graph);
      set_error(std::string("segment capture failed: ") + cudaGetErrorString(err != cudaSuccess ? err : err2));
      return 3;
    }
    cudaGraphExec_t exec = nullptr;
    cudaError_t err3 = cudaGraphInstantiateWithFlags(&exec, graph, cudaGraphInstantiateFlagUseNodePriority);
    cudaGraphDestroy(graph);
    BI_CUDA_TRY(err3);
    it = e->seg_graphs.emplace(key, exec).first;
  }
  BI_CUDA_TRY(cudaGraphLaunch(it->second, s));
  return 0;
}

extern "C" int bi_engine_run_ops(bi_engine* e, int op_begin, int op_end, int use_graph, void* stream) {
  BI_REQUIRE(e && e->bound, "engine not bound");
  BI_REQUIRE(op_begin >= 0 && op_begin <= op_end && op_end <= (int)e->flat.size(), "op range out of bounds");
  for (int i = op_begin; i < op_end; ++i) BI_REQUIRE(e->flat[i].op.kind != 3, "op range spans an exchange");
  // the executed step range, for bi_engine_status (a run starts at op 0)
  if (op_begin == 0) {
    e->last_first = 1;
    e->last_last = 0;
  }
  if (op_end > op_begin) e->last_last = std::max(e->last_last, e->flat[op_end - 1].stepid);
  return run_ops_impl(e, op_begin, op_end, use_graph, static_cast<cudaStream_t>(stream));
}

extern "C" int bi_engine_shard_info(const bi_engine* e, int64_t out[8]) {
  BI_REQUIRE(e && out, "null argument");
  out[0] = e->P;
  out[1] = e->rank;
  out[2] = e->col0;
  out[3] = e->w;
  out[4] = e->wmax;
  out[5] = (int64_t)e->xchgs.size();
  out[6] = e->send_elems;
  out[7] = e->recv_elems;
  return 0;
}

extern "C" int bi_engine_xchg_desc(const bi_engine* e, int i, int64_t out[8]) {
  BI_REQUIRE(e && e->bound && out, "engine not bound");
  BI_REQUIRE(i >= 0 && i < (int)e->xchgs.size(), "exchange index out of range");
  const auto& x = e->xchgs[i];
  out[0] = x.g0;
  out[1] = x.gs;
  out[2] = x.rows;
  out[3] = e->wmax;
  out[4] = x.in_a;
  out[5] = x.from0;
  out[6] = x.from1;
  out[7] = x.kind * 100 + x.level;
  return 0;
}

extern "C" int bi_engine_shard_buffers(const bi_engine* e, double** sendbuf, double** recvbuf) {
  BI_REQUIRE(e && e->bound, "engine not bound");
  if (sendbuf) *sendbuf = e->sendbuf;
  if (recvbuf) *recvbuf = e->recvbuf;
  return 0;
}

// this rank's send parts -> the contiguous send area (rows x wmax, for an all-gather)
extern "C" int bi_engine_xchg_pack(bi_engine* e, int i, void* stream) {
  BI_REQUIRE(e && e->bound, "engine not bound");
  BI_REQUIRE(i >= 0 && i < (int)e->xchgs.size(), "exchange index out of range");
  BI_REQUIRE(e->send_elems > 0, "engine created without BI_SHARD_STAGING");
  const auto& x = e->xchgs[i];
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // a group of one rank has no collective: pack straight into the receive area
  double* dst = x.gs == 1 ? e->recvbuf : e->sendbuf;
  BI_CUDA_TRY(cudaMemcpy2DAsync(dst, e->wmax * 8, x.top, x.top_ld * 8, e->w * 8, x.top_rows,
                                cudaMemcpyDeviceToDevice, s));
  if (x.bot)
    BI_CUDA_TRY(cudaMemcpy2DAsync(dst + x.top_rows * e->wmax, e->wmax * 8, x.bot, x.bot_ld * 8, e->w * 8,
                                  x.bot_rows, cudaMemcpyDeviceToDevice, s));
  return 0;
}

// the group's gathered send areas ([gs][rows][wmax]) -> X (the needed members' columns side by side)
extern "C" int bi_engine_xchg_unpack(bi_engine* e, int i, void* stream) {
  BI_REQUIRE(e && e->bound, "engine not bound");
  BI_REQUIRE(i >= 0 && i < (int)e->xchgs.size(), "exchange index out of range");
  BI_REQUIRE(e->recv_elems > 0, "engine created without BI_SHARD_STAGING");
  const auto& x = e->xchgs[i];
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  for (int m = x.from0; m < x.from1; ++m) {
    const int64_t c0 = e->off[(size_t)m * e->nbp], wm = e->off[(size_t)(m + 1) * e->nbp] - c0;
    BI_CUDA_TRY(cudaMemcpy2DAsync(e->X + (c0 - x.x_col0), x.ldx * 8, e->recvbuf + (int64_t)(m - x.g0) * x.rows * e->wmax,
                                  e->wmax * 8, wm * 8, x.rows, cudaMemcpyDeviceToDevice, s));
  }
  return 0;
}

// All P ranks in this process (one engine per GPU, or several on one GPU for
// tests): one host thread enqueues every rank's segments in order; each
// exchange is peer copies of the members' send windows straight into the
// reader's X on the reader's stream, ordered by events (no host barrier, no
// staging); a rank's next segment waits until its group has copied.
extern "C" int bi_shard_group_run(bi_engine** es, int P, void* const* streams, int first_step, int last_step,
                                  int use_graph) {
  BI_REQUIRE(es && streams && P >= 1, "null argument");
  for (int r = 0; r < P; ++r) {
    BI_REQUIRE(es[r] && es[r]->bound && es[r]->P == P && es[r]->rank == r, "engines must be ranks 0..P-1 of one run");
    BI_REQUIRE(first_step >= 1 && last_step <= es[r]->nsteps && first_step <= last_step, "stepid outside 1..N_s");
  }
  int cur = 0;
  BI_CUDA_TRY(cudaGetDevice(&cur));
  std::vector<std::vector<int>> B(P), E(P), Xi(P);
  int nseg = -1;
  for (int r = 0; r < P; ++r) {
    const int n = bi_engine_shard_segments(es[r], first_step, last_step, nullptr, nullptr, nullptr, 0);
    B[r].resize(n);
    E[r].resize(n);
    Xi[r].resize(n);
    bi_engine_shard_segments(es[r], first_step, last_step, B[r].data(), E[r].data(), Xi[r].data(), n);
    BI_REQUIRE(nseg < 0 || n == nseg, "ranks disagree on the exchange schedule");
    nseg = n;
  }
  std::vector<cudaEvent_t> done(P), copied(P);
  auto cleanup = [&]() {
    for (int r = 0; r < P; ++r) {
      cudaSetDevice(es[r]->device);
      if (done[r]) cudaEventDestroy(done[r]);
      if (copied[r]) cudaEventDestroy(copied[r]);
    }
    cudaSetDevice(cur);
  };
  auto fail = [&](cudaError_t err) {
    cleanup();
    set_error(std::string("bi_shard_group_run: ") + cudaGetErrorString(err));
    return 3;
  };
  for (int r = 0; r < P; ++r) {
    es[r]->last_first = first_step;  // for bi_engine_status
    es[r]->last_last = last_step;
    cudaSetDevice(es[r]->device);
    cudaError_t err = cudaEventCreateWithFlags(&done[r], cudaEventDisableTiming);
    if (err == cudaSuccess) err = cudaEventCreateWithFlags(&copied[r], cudaEventDisableTiming);
    if (err == cudaSuccess && first_step == 1)
      err = cudaMemset2DAsync(es[r]->Minv, es[r]->ldi * 8, 0, es[r]->w * 8, es[r]->n,
                              static_cast<cudaStream_t>(streams[r]));
    if (err != cudaSuccess) return fail(err);
  }
  for (int k = 0; k < nseg; ++k) {
    for (int r = 0; r < P; ++r) {
      bi_engine* e = es[r];
      cudaStream_t s = static_cast<cudaStream_t>(streams[r]);
      cudaSetDevice(e->device);
      if (k > 0 && Xi[r][k - 1] >= 0) {  // my send windows are free once my group copied them
        const auto& px = e->xchgs[Xi[r][k - 1]];
        for (int m = px.g0; m < px.g0 + px.gs; ++m) {
          cudaError_t err = cudaStreamWaitEvent(s, copied[m], 0);
          if (err != cudaSuccess) return fail(err);
        }
      }
      int rc = run_ops_impl(e, B[r][k], E[r][k], use_graph, s);
      if (rc) {
        cleanup();
        return rc;
      }
      cudaError_t err = cudaEventRecord(done[r], s);
      if (err != cudaSuccess) return fail(err);
    }
    for (int r = 0; r < P; ++r) {
      if (Xi[r][k] < 0) continue;
      bi_engine* e = es[r];
      cudaStream_t s = static_cast<cudaStream_t>(streams[r]);
      cudaSetDevice(e->device);
      const auto& x = e->xchgs[Xi[r][k]];
      for (int m = x.from0; m < x.from1; ++m) {
        const auto& mx = es[m]->xchgs[Xi[m][k]];
        cudaError_t err = cudaStreamWaitEvent(s, done[m], 0);
        const int64_t c0 = es[m]->col0 - x.x_col0;
        if (err == cudaSuccess)
          err = cudaMemcpy2DAsync(e->X + c0, x.ldx * 8, mx.top, mx.top_ld * 8, es[m]->w * 8, mx.top_rows,
                                  cudaMemcpyDefault, s);
        if (err == cudaSuccess && mx.bot)
          err = cudaMemcpy2DAsync(e->X + mx.top_rows * x.ldx + c0, x.ldx * 8, mx.bot, mx.bot_ld * 8, es[m]->w * 8,
                                  mx.bot_rows, cudaMemcpyDefault, s);
        if (err != cudaSuccess) return fail(err);
      }
      cudaError_t err = cudaEventRecord(copied[r], s);
      if (err != cudaSuccess) return fail(err);
    }
  }
  // events may be destroyed while pending work still references them (CUDA defers the release)
  cleanup();
  return 0;
}

namespace bi {
bool shard_staging(const bi_engine* e) { return (e->shard_flags & BI_SHARD_STAGING) != 0; }
int shard_nranks(const bi_engine* e) { return e->P; }
int shard_rank(const bi_engine* e) { return e->rank; }
std::map<int, void*>& shard_group_comms(bi_engine* e) { return e->group_comms; }
int shard_zero_minv(bi_engine* e, cudaStream_t s) {
  e->last_first = 1;
  BI_CUDA_TRY(cudaMemset2DAsync(e->Minv, e->ldi * 8, 0, e->w * 8, e->n, s));
  return 0;
}
}  // namespace bi
