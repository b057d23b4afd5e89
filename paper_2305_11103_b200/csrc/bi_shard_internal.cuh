// Accessors the NCCL transport (bi_nccl.cu) needs from the engine (bi_engine.cu).
#pragma once
#include <cuda_runtime.h>

#include <map>

#include "../../include/blockinv_b200.h"

namespace bi {
bool shard_staging(const bi_engine* e);
int shard_nranks(const bi_engine* e);
int shard_rank(const bi_engine* e);
std::map<int, void*>& shard_group_comms(bi_engine* e);  // group size -> ncclComm_t
int shard_zero_minv(bi_engine* e, cudaStream_t s);
void shard_destroy_comms(bi_engine* e);  // bi_nccl.cu: the engine's group communicators
}  // namespace bi
