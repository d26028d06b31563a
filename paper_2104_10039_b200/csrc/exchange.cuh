// exchange.cuh — the per-iteration exchange of the 1-D destination
// partition: every rank owns a 32-aligned, edge-balanced
// destination range and a full replica of the message (property) vector.
// After each iteration the owned slices of msg_next are all-gathered
// (grouped ncclBroadcast per root = AllGatherV over NVLink/NVSwitch) and the
// iteration counters are all-reduced, so every rank takes the same early-exit
// and EngineError decisions (engine.hpp:226-240).
#pragma once

#include <nccl.h>

#include <memory>

#include "graph.cuh"

namespace ggb {
struct LocalGroup;  // in-process transport (exchange.cu)
}

struct gg_exchange {
    int rank = 0, nranks = 1;
    ncclComm_t comm = nullptr;               // NCCL transport (one process per GPU)
    std::shared_ptr<ggb::LocalGroup> local;  // or: ranks as threads of one process
};

namespace ggb {

// libnccl.so.2 is dlopen'ed on first multi-GPU use (the single-GPU path has
// no NCCL dependency and never clashes with the NCCL torch already loaded).
struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};
const NcclApi& nccl();

// All-gather of each rank's slice of a global array. slots = true: the
// array is in message-slot order and only the slots that are ever gathered
// (out-degree > 0, a prefix of each rank's slot range) travel.
void exchange_slices(DevGraph& g, void* global_buf, size_t elem_size, bool slots = false);
void exchange_counters(DevGraph& g, void* ctr);
// sum of `local` over ranks below this one (allgather of one u64 per rank)
uint64_t exchange_exclusive_base(DevGraph& g, uint64_t local);
// sum of `local` over all ranks
uint64_t exchange_sum(DevGraph& g, uint64_t local);
// element-wise sum over ranks of a device u32[count] array, in place
// (setup only: graph validation)
void exchange_allreduce_u32(DevGraph& g, uint32_t* buf, uint64_t count);

}  // namespace ggb
