/*
 * blockinv_b200.h -- C ABI of the B200 (sm_100a) blockwise-inversion library
 * (libblockinv_b200.so).  The drop-in boundary for the reference `blockinv`
 * hot path (/root/reference/pkg/src/blockinv).
 *
 * Conventions
 *  - Plain C types only: pointers, 64-bit sizes, int status.  No torch types.
 *  - Every matrix pointer is a DEVICE pointer to row-major (C-order) float64
 *    with an explicit leading dimension `ld` (elements, >= cols).  The
 *    library never frees caller memory; callers size and own every buffer,
 *    including workspaces (query functions give the byte counts).
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default).
 *  - Return value: BI_OK (0) or one of the BI_E* codes; bi_last_error()
 *    returns a thread-local message for the last failure.
 *  - Singular pivots are not an error of the call: they are reported through
 *    `info` arrays / out-parameters exactly where the reference raises
 *    SingularBlock / SingularMatrix (errors.py:17-38).
 */
#ifndef BLOCKINV_B200_H
#define BLOCKINV_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  BI_OK = 0,
  BI_ESINGULAR = 1, /* a pivot block / Schur complement is singular      */
  BI_EDIM = 2,      /* shape / argument error (DimensionMismatch, ...)    */
  BI_ECUDA = 3,     /* CUDA runtime error                                 */
  BI_ENCCL = 4,     /* NCCL error / NCCL unavailable (multi-GPU transport) */
  BI_EUNSUPPORTED = 5
};

/* Library identity and the last error message of the calling thread. */
int bi_version(void);
const char* bi_last_error(void);

/* Device setup (SURVEY 8b bi_init/bi_finalize).  bi_init checks that every
 * listed device is an sm_100 part (BI_EUNSUPPORTED otherwise), sets the
 * kernels' attributes there (dynamic shared memory, cluster sizes) and
 * enables peer access between every pair of listed devices that supports it
 * (the sharded scheduler's NVLink slab exchanges).  Entry points also
 * initialise lazily, so calling it is optional; the current device is
 * preserved.  bi_finalize synchronises the listed devices and releases
 * library-owned helper streams.  The reference's counterpart is the
 * engine's worker pool (engine.py:257-270). */
int bi_init(int ndev, const int* dev_ids);
int bi_finalize(void);

/* ------------------------------------------------------------------------
 * K1: FP64 DMMA GEMM.  D = [Cin] + (alpha_sign)*A*B, strided batched.
 * Replaces core._mm_acc / multiply / schur_accumulate
 * (core.py:115-139, 142-170, 173-192) and engine.fox_block_multiply
 * (engine.py:202-249): out = (+-1)*a@b, or out += ... when accumulating.
 * Cin may be NULL (beta = 0) and may equal D (in-place accumulate, the
 * `accumulate=True` form).  A/B must not alias D (core.py:161-163).
 * ---------------------------------------------------------------------- */
int bi_gemm(int64_t m, int64_t n, int64_t k, int alpha_sign,
            const double* a, int64_t lda, int64_t stride_a,
            const double* b, int64_t ldb, int64_t stride_b,
            const double* cin, int64_t ldc, int64_t stride_c,
            double* d, int64_t ldd, int64_t stride_d,
            int batch, void* stream);
/* Grouped form (ragged batches, e.g. the non-uniform partitions of cfg3 and
 * the default partition): `count` independent GEMM problems in ONE launch,
 * each a bi_gemm argument set.  Descriptors live in host memory; with more
 * than 4 of them the table is copied into `workspace`
 * (bi_gemm_grouped_workspace_bytes(count) bytes; may be NULL up to 4). */
typedef struct bi_gemm_desc {
  int64_t m, n, k;
  int alpha_sign; /* +1 | -1 */
  const double* a; int64_t lda, stride_a;
  const double* b; int64_t ldb, stride_b;
  const double* cin; int64_t ldc, stride_c; /* cin may be NULL */
  double* d; int64_t ldd, stride_d;
  int batch;
} bi_gemm_desc;
int64_t bi_gemm_grouped_workspace_bytes(int count);
int bi_gemm_grouped(int count, const bi_gemm_desc* descs, void* workspace, int64_t workspace_bytes,
                    void* stream);
/* K1P: all-gather fused into K1 for the sharded scheduler's global levels.
 * D = [Cin] + (alpha_sign) * [A_0 | ... | A_{nseg-1}] * B, where segment s is
 * an m x k_segs[s] matrix at a_segs[s] (leading dimension lda_segs[s]) that
 * may live in a PEER GPU's memory (peer access enabled, e.g. by bi_init):
 * every k-tile is read from its owner over NVLink while earlier k-tiles are
 * multiplied, instead of all-gathering the slabs into one buffer first.
 * Replaces the exchange + multiply of the reference's Fox broadcast step
 * (engine.fox_block_multiply, engine.py:202-249) across GPUs.  1 <= nseg <= 8;
 * every segment but the last must be a multiple of 16 columns wide (k-tile
 * boundaries), so the result is bitwise equal to bi_gemm on the gathered A.
 * B, Cin and D are local; Cin may equal D. */
int bi_gemm_kseg(int64_t m, int64_t n, int alpha_sign, int nseg, const double* const* a_segs,
                 const int64_t* lda_segs, const int64_t* k_segs, const double* b, int64_t ldb,
                 const double* cin, int64_t ldc, double* d, int64_t ldd, void* stream);

/* ------------------------------------------------------------------------
 * K2/K3: batched in-place-style Gauss-Jordan inversion with partial pivoting
 * (pivot tolerance 1e-12 * n * max|block|, as gauss_jordan_oracle,
 * core.py:379-402).  Inverts `count` n x n blocks:
 *   out[i] = inverse(in[i]),  in[i] = in + i*stride_in (ld_in),
 *   out[i] = out + i*stride_out (ld_out).
 * Replaces core.invert_small (core.py:350-376), the engine's leaf inverter
 * engine._leaf_invert (engine.py:449-457) and the `invert_sub(block, out)`
 * plugin protocol (schur.py:16-18, 104-111).  info[i] = 0 on success, or
 * c+1 where c is the first pivot column with no usable pivot.
 * Blocks above order 8192 (one K3 cluster) are inverted by the pivot-A
 * recursion (recursive.py:83-123) down to leaves of at most 4096 with
 * partial pivoting inside each leaf; info is then the first failing leaf's
 * global column + its leaf info.
 * `workspace` must hold bi_inv_workspace_bytes(count, n) bytes.
 * ---------------------------------------------------------------------- */
int64_t bi_inv_workspace_bytes(int count, int64_t n);
int bi_inv_batched(int count, int64_t n,
                   const double* in, int64_t ld_in, int64_t stride_in,
                   double* out, int64_t ld_out, int64_t stride_out,
                   int* info, void* workspace, int64_t workspace_bytes,
                   void* stream);
/* Same with arbitrary blocks: in[i] / out[i] and their leading dimensions
 * are DEVICE arrays of `count` entries (the engine's pointer-table form; the
 * sharded scheduler batches every equal-order leaf of a step this way). */
int bi_inv_batched_ptrs(int count, int64_t n,
                        const double* const* in, const int64_t* ld_in,
                        double* const* out, const int64_t* ld_out,
                        int* info, void* workspace, int64_t workspace_bytes,
                        void* stream);

/* ------------------------------------------------------------------------
 * Step engine: run_inversion (engine.py:482-542) over `batch` independent
 * matrices that share one partition `sizes[nblocks]` (nblocks a power of 2,
 * partition.py:87-99).  Executes stepids [first_step, last_step] of the
 * 2*nblocks-1 step schedule (engine.py:73-162); `last_step` < N_s is the
 * `stop_after_step` form.  M_inv is written in place (zero-filled by the
 * caller before step 1, storage.py:391-411).
 *
 *   bi_engine_create   -> opaque plan; validates sizes (InvalidOrder).
 *   bi_engine_workspace_bytes -> device workspace (T-sets, leaf scratch,
 *                          descriptor tables) the caller must provide.
 *   bi_engine_bind     -> binds device buffers and uploads the schedule.
 *   bi_engine_run      -> enqueues steps on `stream` (graph-captured when
 *                          use_graph != 0); asynchronous.
 *   bi_engine_status   -> synchronizes; reports the first singular leaf as
 *                          (step, quad, matrix) like SingularBlock(step,quad)
 *                          (engine.py:320-328); returns BI_ESINGULAR then.
 *   bi_engine_counters -> OpCounters semantics of the executed steps
 *                          (engine.py:317, 344-345, 411):
 *                          out[0]=multiplies out[1]=inversions out[2]=reductions
 *                          out[3]=gemm flops (algorithmic) out[4]=leaf flops
 *                          out[5]=gemm bytes (algorithmic: each operand read
 *                          once, each output written once).
 * ---------------------------------------------------------------------- */
typedef struct bi_engine bi_engine;
int bi_engine_create(bi_engine** out, int nblocks, const int64_t* sizes, int batch);
/* Schedules.  BI_SCHEDULE_EQ7 is the reference step engine above (default;
 * step/state parity).  BI_SCHEDULE_PIVOT_A runs the 2n^3
 * pivot-A recursion of invertor_by_a (recursive.py:83-123) at block
 * granularity instead -- same partition, same K3 leaves, in place in M_inv
 * -- as one step (N_s = 1): no stop_after_step states, no T-sets, 2n^3
 * instead of (3 - 1/N_b) n^3 flops.  Singular leaves report step 1 and the
 * block index as `quad`. */
#define BI_SCHEDULE_EQ7 0
#define BI_SCHEDULE_PIVOT_A 1
int bi_engine_create_ex(bi_engine** out, int nblocks, const int64_t* sizes, int batch, int schedule);
int64_t bi_engine_workspace_bytes(const bi_engine* e);
int bi_engine_bind(bi_engine* e,
                   const double* m, int64_t ldm, int64_t stride_m,
                   double* minv, int64_t ldi, int64_t stride_i,
                   void* workspace, int64_t workspace_bytes, void* stream);
int bi_engine_run(bi_engine* e, int first_step, int last_step, int use_graph, void* stream);
/* End-to-end form with HOST buffers (the drop-in call with NumPy memory):
 * host_in[z] (ld_in, stride_in) is copied into M per matrix on a copy stream,
 * M_inv is zeroed (first_step == 1), and each inverse is copied back into
 * host_out[z] as soon as its lane finishes -- transfers overlap the other
 * matrices' compute.  Either pointer may be NULL (data already resident / no
 * read-back).  Page-locked host memory is captured into the step graph;
 * pageable memory runs the same sequence without a graph. */
int bi_engine_run_host(bi_engine* e, const double* host_in, int64_t ld_in, int64_t stride_in,
                       double* host_out, int64_t ld_out, int64_t stride_out,
                       int first_step, int last_step, int use_graph, void* stream);
int bi_engine_status(bi_engine* e, int* fail_step, int* fail_quad, int* fail_matrix);

/* ------------------------------------------------------------------------
 * Column-sharded level scheduler: the engine of rank `rank` of
 * `nranks` (a power of two dividing nblocks; batch 1, Eq. 7).  Rank r owns
 * the home range of diagonal blocks [r N_b/P, (r+1) N_b/P) and stores block
 * COLUMNS of that range of M, M_inv and every T_l (bind M / M_inv as n x w
 * slabs).  Local levels (2^l <= N_b/P) run without communication; each
 * global-level action starts with an exchange inside its rank group
 * (engine.py:336-437 split by output columns, K never split, so every P is
 * bitwise equal to P = 1):
 *   arrows   A-half ranks send [A^-1 ; C], D-half ranks [B ; D^-1]
 *            (the inverted pivot blocks and the off-diagonal operands);
 *   up/down  A-half ranks share L, D-half ranks R.
 * The replaced reference interface is the engine's fork-join over workers
 * (engine.py:257-285) and INVERTOR_WORKERS (engine.py:58-65).
 *
 *   bi_engine_shard_segments -> the op ranges between exchanges of steps
 *        [first, last]: begin/end into the flat op list, xchg = the exchange
 *        after the segment (-1 none); returns the count (call with cap 0 to size).
 *   bi_engine_run_ops        -> enqueue one segment (graph-captured).
 *   Transport A, all ranks in one process (one GPU each; tests may map
 *   several ranks to one GPU): bi_shard_group_run drives every rank from
 *   one host thread -- peer copies (NVLink, P2P enabled by bi_init) of the
 *   members' send windows into each reader's X, ordered by events.
 *   Transport B, one process per GPU: create with BI_SHARD_STAGING, then per
 *   exchange bi_engine_xchg_pack (send parts -> send area, rows x wmax),
 *   an all-gather of the send areas inside the group (NCCL) into the receive
 *   area ([gs][rows][wmax]), bi_engine_xchg_unpack (-> X).  The group
 *   [g0, g0 + gs) of bi_engine_xchg_desc is the quad's ranks for an arrows
 *   exchange and the rank's own half of them for an up/down pass (equal part
 *   heights inside a half, also with ragged block orders); gs == 1 packs
 *   straight into the receive area and needs no collective.
 * ---------------------------------------------------------------------- */
#define BI_SHARD_STAGING 1
int bi_engine_create_shard(bi_engine** out, int nblocks, const int64_t* sizes, int nranks, int rank, int flags);
int bi_engine_shard_info(const bi_engine* e, int64_t out[8]);   /* P, rank, col0, w, wmax, #xchg, send, recv elems */
int bi_engine_shard_segments(const bi_engine* e, int first_step, int last_step, int* begin, int* end, int* xchg,
                             int cap);
int bi_engine_run_ops(bi_engine* e, int op_begin, int op_end, int use_graph, void* stream);
int bi_engine_xchg_desc(const bi_engine* e, int i, int64_t out[8]); /* g0, gs, rows, wmax, in_a, from0, from1, kind*100+level */
int bi_engine_shard_buffers(const bi_engine* e, double** sendbuf, double** recvbuf);
int bi_engine_xchg_pack(bi_engine* e, int i, void* stream);
int bi_engine_xchg_unpack(bi_engine* e, int i, void* stream);
int bi_shard_group_run(bi_engine** engines, int nranks, void* const* streams, int first_step, int last_step,
                       int use_graph);
/* Transport C, one process per GPU, NCCL inside the library (libnccl.so.2 is
 * dlopen'ed; a process that already loaded NCCL shares it):
 *   rank 0: bi_nccl_unique_id(id) -> every rank (out of band, e.g. a
 *   torch.distributed broadcast) -> bi_nccl_comm_init(P, id, rank, &world)
 *   on its GPU -> bi_engine_shard_set_comm(e, world) (collective: one
 *   ncclCommSplit per power-of-two group size) -> bi_engine_run_nccl(e, 1,
 *   N_s, use_graph, stream): every segment and every exchange (pack ->
 *   ncclAllGather -> unpack) enqueued by this one call, stream-ordered.
 * BI_ENCCL reports NCCL failures or a missing / too old libnccl. */
int bi_nccl_available(void);
int bi_nccl_unique_id(unsigned char* id /* 128 bytes */);
int bi_nccl_comm_init(int nranks, const unsigned char* id, int rank, void** comm);
int bi_nccl_comm_destroy(void* comm);
int bi_engine_shard_set_comm(bi_engine* e, void* world_comm);
int bi_engine_run_nccl(bi_engine* e, int first_step, int last_step, int use_graph, void* stream);
/* Enqueue only one class of ops of steps [first, last] (no graph): mask 1 =
 * the engine's K1 GEMM launches, 2 = the leaf inversions (K3 incl. their
 * trailing-update GEMMs), 3 = both.  For per-kernel timing in bench.py. */
int bi_engine_run_phase(bi_engine* e, int first_step, int last_step, int mask, void* stream);
/* Kernel launches of steps [first, last]: out[0] total, out[1] K1 (engine
 * GEMMs + leaf trailing updates), out[2] other K3 kernels. */
int bi_engine_launches(const bi_engine* e, int first_step, int last_step, int64_t out[3]);
int bi_engine_counters(const bi_engine* e, int first_step, int last_step, double out[6]);
/* Profiling aid: with BI_ENGINE_TIMELINE=1 in the environment at bind time,
 * every lane records a timing event after each step (graph runs included).
 * After a run, out_ms[lane * (N_s + 1) + stepid] = ms from the run's start to
 * the end of that step on that lane (-1 for steps outside the last run). */
int bi_engine_timeline(bi_engine* e, float* out_ms);
/* T-set access for step-state parity: pointer + ld of the level-`level`
 * provisional square of quad `quad` of matrix `matrix` (S_D at A's
 * position, R at B's, L at C's, S_A at D's; storage.py:166-262). */
int bi_engine_tset_square(const bi_engine* e, int level, int quad, int matrix,
                          double** ptr, int64_t* ld, int64_t* side);
int bi_engine_destroy(bi_engine* e);

/* ------------------------------------------------------------------------
 * Single-level 2x2 pivot formulas on one square matrix m (order n, split p).
 * pivot = 'A' : invert_via_a (schur.py:114-139, Eq. 2)
 * pivot = 'D' : invert_via_d (schur.py:142-164, Eq. 3; the singular-A11 path)
 * pivot = 'X' : invert_via_ad (schur.py:219-259, Eq. 7)
 * counter-diagonal layout (rows split at p, columns at n - p; schur.py:92-101):
 * pivot = 'B' : invert_via_b (schur.py:167-190)
 * pivot = 'C' : invert_via_c (schur.py:193-216)
 * pivot = 'Y' : invert_via_bc (schur.py:262-297)
 * Sub-inversions use K3.  On a singular pivot returns BI_ESINGULAR with
 * *fail_block = 'A','D','B','C' or 'a','d','b','c' (SchurA/D/B/C) -- the
 * labels of schur._sub_inverse (schur.py:104-111).  out must not alias m.
 * ---------------------------------------------------------------------- */
int64_t bi_schur2x2_workspace_bytes(int64_t n, int64_t p);
int bi_schur2x2(int pivot, int64_t n, int64_t p,
                const double* m, int64_t ldm, double* out, int64_t ldo,
                void* workspace, int64_t workspace_bytes,
                int* fail_block, void* stream);

/* ------------------------------------------------------------------------
 * invertor_inplace_by_a (recursive.py:273-333): x <- x^-1 in place by the
 * pivot-A recursion (Eq. 2) with K3 leaves of order <= leaf_order.
 * On failure *fail_path receives the recursion path as a string of 'A'/'S'
 * (A / SchurA) of at most 63 characters.
 * ---------------------------------------------------------------------- */
int64_t bi_inplace_by_a_workspace_bytes(int64_t n, int64_t leaf_order);
int bi_inplace_by_a(int64_t n, double* x, int64_t ldx, int64_t leaf_order,
                    void* workspace, int64_t workspace_bytes,
                    char* fail_path, void* stream);

/* ------------------------------------------------------------------------
 * K4: residual norms for verification (core.residual_norm, core.py:405-414,
 * in the Frobenius form of the north star).  Writes, for `batch` pairs,
 * out[2*i] = ||A_i X_i - I||_F^2 and out[2*i+1] = max |A_i X_i - I| (device
 * pointer, 2*batch doubles).  workspace: bi_residual_workspace_bytes.
 * ---------------------------------------------------------------------- */
int64_t bi_residual_workspace_bytes(int64_t n, int batch);
int bi_residual(int64_t n, int batch,
                const double* a, int64_t lda, int64_t stride_a,
                const double* x, int64_t ldx, int64_t stride_x,
                double* out, void* workspace, int64_t workspace_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* BLOCKINV_B200_H */
