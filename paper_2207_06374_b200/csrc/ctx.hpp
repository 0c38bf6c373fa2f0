// The C ABI's context object (include/trstmi_b200.h: trstmi_ctx): one device,
// its stream and work counter, the lazily created large-frame engine, and the
// optional cross-rank communicator of the multi-GPU trial scheduler
// (csrc/sharding.cu).  Shared by the translation units that implement the ABI.
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>

#include <string>

#include "bde_engine.hpp"
#include "large_engine.hpp"

struct trstmi_ctx {
  int device = 0;
  int sm_count = 0;
  cudaStream_t stream = nullptr;
  int* counter = nullptr;
  trstmi_large::Engine* large = nullptr;  // large-frame engine for the sharded single frame (lazy)
  trstmi_bde_host::Engine* bde = nullptr; // batched large-frame engine (lazy)
  int large_workers = 8;                  // concurrent large-path trials (streams)
  int shard_world = 1;                    // single-frame row-block sharding (trstmi_set_shard)
  // multi-GPU trial scheduler (trstmi_comm_init): one process per GPU
  ncclComm_t comm = nullptr;
  int world = 1, rank = 0;
  std::string err;
};
