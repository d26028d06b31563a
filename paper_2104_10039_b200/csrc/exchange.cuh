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
    bool fused = true;                       // vertex kernel stores into peer replicas
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

// Fused exchange. The vertex kernel that computes the new messages also
// stores each gathered slot's message into every rank's replica (peer
// memory), so no separate all-gather pass runs; with one message buffer per
// rank the iteration then needs one barrier between the gathers and the
// vertex kernel (no rank may overwrite a replica another rank still reads).
// (kMaxPeers, common.cuh: one NVSwitch node)
// Collective over the ranks: true when every rank's `msg` (bytes) is
// addressable from this rank's device (g.peer_msg filled), false when some
// rank cannot map its peers (the caller all-gathers with exchange_slices).
// Cached for the same buffer. NCCL transport: `msg` must come from
// exchange_msg_buffer (CUDA IPC needs a cudaMalloc allocation).
bool exchange_register_peers(DevGraph& g, void* msg, size_t bytes);
// The message buffer of a run: IPC-exportable for the NCCL transport, the
// workspace's otherwise.
void* exchange_msg_buffer(DevGraph& g, size_t bytes);
// Stream-ordered barrier: nothing enqueued after it on any rank starts
// before everything enqueued before it on every rank has completed.
void exchange_barrier(DevGraph& g);
// closes the IPC mappings of g (graph teardown)
void exchange_release_peers(DevGraph& g);
void exchange_counters(DevGraph& g, void* ctr);
// sum of `local` over ranks below this one (allgather of one u64 per rank)
uint64_t exchange_exclusive_base(DevGraph& g, uint64_t local);
// sum of `local` over all ranks
uint64_t exchange_sum(DevGraph& g, uint64_t local);
// element-wise sum over ranks of a device u32[count] array, in place
// (setup only: graph validation)
void exchange_allreduce_u32(DevGraph& g, uint32_t* buf, uint64_t count);

}  // namespace ggb
