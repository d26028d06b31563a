// graph.cuh — HBM-resident pull CSC (gg::Graph, graph.hpp:29-49) and the
// per-graph device workspace.
//
// HBM layout per rank (local = owned destination range [v_begin, v_end)),
// see DESIGN.md §3:
//   off      u64[nloc+1]        local in-edge offsets (rebased to 0)
//   vid_of_p u32[nloc]          POSITION order of the local vertices: the R
//                               vertices with in-edges ("rows", vertex order)
//                               first, then the in-degree-0 ones. Per-vertex run
//                               state (property, status, accumulators, the
//                               sparsified offsets) is stored by position, so
//                               the vertex epilogue walks the rows densely and
//                               skips the in-degree-0 tail once none is active.
//   slot_p, deg_p               message slot / out-degree by position
//   src      u32[pad+e_loc+..]  in-edge sources as MESSAGE SLOT ids, at padded
//                               positions pad + local edge (pad = global pos mod 512)
//   w        W[...]             none | u32 | f32 | f64, padded likewise
//   outdeg   u32[n]             out-degree of every (global) vertex
//   slot_of / vtx_of_slot       hot-first message slot map (global)
//   full     ListMeta           run -> non-empty-vertex map of the full list
// Run workspace (Workspace, grow-only, reused across runs): bitmap (1 bit per
// local edge, EdgeFlags graph.hpp:54-72), sparsified s_off/s_src/s_w + its
// ListMeta, msg[2], prop, status[2], acc_out/hv/tv/carry, counters.
#pragma once

#include <functional>
#include <map>
#include <string>
#include <vector>

#include "common.cuh"

struct gg_exchange;

namespace ggb {

struct DevBuffer {
    void* ptr = nullptr;
    size_t bytes = 0;
};

// Device allocations go through the stream-ordered pool of the device
// (cudaMallocAsync), whose release threshold is raised at graph creation:
// freed memory stays cached, so re-creating a graph of the same size (the
// end-to-end path) does not pay cudaMalloc / cudaFree of tens of GB.
inline void* dev_alloc(size_t bytes, cudaStream_t st) {
    void* p = nullptr;
    GGB_CUDA(cudaMallocAsync(&p, bytes ? bytes : 16, st));
    return p;
}
inline void dev_free(void* p, cudaStream_t st) {
    if (p) cudaFreeAsync(p, st);
}

// Grow-only named workspace: runs reuse device memory, so no allocation
// happens inside a timed run after the first one.
struct Workspace {
    std::map<std::string, DevBuffer> bufs;
    cudaStream_t stream = nullptr;
    void* get(const std::string& name, size_t bytes) {
        DevBuffer& b = bufs[name];
        if (b.bytes < bytes || !b.ptr) {
            if (b.ptr) dev_free(b.ptr, stream);
            b.ptr = dev_alloc(bytes, stream);
            b.bytes = bytes ? bytes : 16;
        }
        return b.ptr;
    }
    template <class T>
    T* get(const std::string& name, size_t count) {
        return static_cast<T*>(get(name, count * sizeof(T)));
    }
    void release() {
        for (auto& kv : bufs) dev_free(kv.second.ptr, stream);
        bufs.clear();
    }
};

// Edge-centric layout of one list (full or sparsified CSC): padded
// positions P = pad + local edge index, runs of 16 and tasks of 512 padded
// positions, run_i[r] = the non-empty vertex containing the first valid
// position of run r (see kernels.cuh).
// The edge kernel walks only the list's NON-EMPTY vertices (nz_vid / nz_start,
// a doubly-compressed view), so long stretches of empty vertices cost nothing.
// Full list: nz_vid[i] = the local vertex of row i (rows are its non-empty
// vertices, so row = nz index). Sparsified list: nz_vid[i] = the ROW of its
// i-th non-empty vertex (the layout runs in row space).
struct ListMeta {
    uint64_t pad = 0;      // padded position of local edge 0 (global position mod 512)
    uint64_t e = 0;        // local edges
    uint64_t nruns = 0;    // ntasks * 32 (every run index of a task is addressable)
    uint64_t ntasks = 0;
    uint64_t nz = 0;       // non-empty vertices (full list; the sparsified list keeps it on the device)
    uint32_t* run_i = nullptr;     // [nruns+1] index into nz_* of the vertex at the run's first
                                   // position; run_i[nruns] = nz - 1
    uint32_t* nz_vid = nullptr;    // [nz] local vertex id
    uint64_t* nz_start = nullptr;  // [nz+1] local edge offset (nz_start[nz] = e)
    uint64_t e_end() const { return pad + e; }
};

struct DevGraph {
    int device = 0;
    int rank = 0, nranks = 1;
    gg_exchange* exchange = nullptr;
    uint64_t n = 0, e_global = 0;
    uint64_t v_begin = 0, v_end = 0, nloc = 0;
    uint64_t e_base = 0, e_loc = 0;        // global id of first local edge, local count
    std::vector<uint64_t> bounds;          // vertex bounds of every rank (nranks+1)
    std::vector<uint64_t> ebounds;         // edge bounds of every rank
    uint64_t* off = nullptr;
    uint32_t* src = nullptr;   // padded: local edge i at src[full.pad + i]
    void* w = nullptr;         // padded likewise
    gg_weight_kind wkind = GG_W_NONE;
    uint32_t* outdeg = nullptr;
    // Message-slot layout: messages are stored hot-first (descending
    // out-degree within each rank's range) so the gathers' hot set packs
    // into L2; src arrays hold slot ids. slot_of[v] / vtx_of_slot[s], global.
    uint32_t* slot_of = nullptr;
    uint32_t* vtx_of_slot = nullptr;
    // Several ranks: the message slots a gather can read (out-degree > 0) of
    // each rank's vertices, as two slot ranges per rank {b0, e0, b1, e1}:
    // its hot tier-0 slots and the out-degree > 0 prefix of its tier-1 slots
    // (compute_slots); hot_slots = the tier-0 total, a GLOBAL prefix of the
    // slot order, so every rank's gathers can single it out (L1/L2 classes).
    std::vector<uint64_t> gather_ranges;
    uint64_t hot_slots = 0;
    // Fused exchange (exchange_register_peers): every rank's message buffer
    // as addressed from this rank's device (peer memory over NVLink /
    // NVSwitch, or the same device for the in-process transport), so the
    // vertex kernel stores each new message into every replica. Empty: the
    // messages are all-gathered after the vertex kernel (exchange_slices).
    std::vector<void*> peer_msg;
    const void* peer_msg_for = nullptr;  // own buffer the peers were registered for
    size_t peer_msg_bytes = 0;
    std::vector<void*> ipc_opened;       // peer buffers opened through CUDA IPC
    void* ipc_msg = nullptr;             // own message buffer, cudaMalloc'd (IPC-exportable)
    size_t ipc_msg_bytes = 0;
    ListMeta full;
    // position order (graph.cuh header): rows = full.nz non-empty vertices
    uint64_t nrows = 0;
    uint32_t* vid_of_p = nullptr;  // [nloc + 1] local vertex of position p (full.nz_vid = rows)
    uint32_t* slot_p = nullptr;    // [nloc + 1] message slot of position p
    uint32_t* deg_p = nullptr;     // [nloc + 1] out-degree of position p
    // gg_dev_graph_create_for_run: the bitmap / compacted sources of
    // sparsify(sigma, seed) are already in the workspace for the next run
    bool pre_sparse = false;
    double pre_sigma = 0.0;
    uint64_t pre_seed = 0;
    cudaStream_t stream = nullptr;
    int num_sms = 148;
    Workspace ws;
    // double[n] projection of the last run's final properties, computed on
    // demand in the workspace (valid until the next run); set by every run
    std::function<const double*()> project_last;
    void* h_ctr = nullptr;            // pinned host mirror of the iteration counters
    cudaEvent_t ev[8] = {};           // timing events, created on first use
    std::vector<cudaEvent_t> bev;     // timing events of batched iterations
    void* host_counters(size_t bytes) {
        if (!h_ctr) GGB_CUDA(cudaHostAlloc(&h_ctr, bytes, cudaHostAllocDefault));
        return h_ctr;
    }
    cudaEvent_t event(int i) {
        if (!ev[i]) GGB_CUDA(cudaEventCreate(&ev[i]));
        return ev[i];
    }
    cudaEvent_t batch_event(size_t i) {
        while (bev.size() <= i) {
            cudaEvent_t e;
            GGB_CUDA(cudaEventCreate(&e));
            bev.push_back(e);
        }
        return bev[i];
    }
    ~DevGraph();
};

size_t weight_size(gg_weight_kind k);
// A graph's sparsified sources are stored in sp_slot order (common.cuh) iff
// it carries no weights: a graph-level rule, so the upload-overlapped
// sparsification, every rebuild and the approximate gather agree without
// knowing the program. Measured (profiles/r2_summary.md, session 5): the
// coalesced source loads pay on the unweighted configs (c5 gathers -3.2 %,
// c3 +1 % GTEPS); on weighted graphs the dearer compaction stores outweigh
// them (c4 -2.5 %, c2 -0.4 %).
inline bool sp_quads(const DevGraph& g) { return weight_size(g.wkind) == 0; }
// graph creation steps shared by the C-ABI constructors (capi.cu)
void setup_common(DevGraph& g, const gg_part_opts* opts);
void finish_graph(DevGraph& g, const uint64_t* host_off_full);

// A full CSC generated on device (rmat.cu).
struct RmatCsc {
    uint64_t n = 0, e = 0;
    uint64_t* off = nullptr;
    uint32_t* src = nullptr;
    void* w = nullptr;
    uint32_t* outdeg = nullptr;
};
RmatCsc rmat_generate(const gg_rmat_params& p, cudaStream_t st);
// graph.cpp:249-257 symmetrized() of a resident single-rank graph, as a full
// CSC in HBM on `st`'s device (symmetrize.cu)
RmatCsc symmetrize_device(const DevGraph& g, cudaStream_t st);
// a DevGraph (after setup_common) from a full device CSC (capi.cu)
void adopt_csc(DevGraph& g, RmatCsc r, gg_weight_kind wk);
void bp_priors_device(uint64_t n, uint64_t seed, float* out, cudaStream_t st);

// Hot-first message slots (slot_of / vtx_of_slot) and the rewrite of the
// full list's sources from vertex ids to slot ids.
void assign_slots(DevGraph& g);
// the two halves of assign_slots, for the pipelined upload: slot_of /
// vtx_of_slot (stream-ordered, no sync) and the in-place source relabel
void compute_slots(DevGraph& g);
// (bad != nullptr: range-check the sources, flagging any >= n into *bad)
void relabel_sources(DevGraph& g, uint32_t* src, uint64_t count, unsigned int* bad = nullptr);
// flag decreasing local offsets into *bad (Graph::validate, graph.cpp:83-86)
void check_offsets(DevGraph& g, unsigned int* bad);
// Copy the full list's sources back to host as vertex ids.
void export_sources(const DevGraph& g, uint32_t* host_out);
// Size `meta` for (pad, e) and build its run -> vertex map from `off`.
void build_runs(DevGraph& g, const uint64_t* off, uint64_t pad, uint64_t e,
                const std::string& tag, ListMeta& meta);
// The full list's layout plus the position order (vid_of_p, slot_p, deg_p;
// needs slot_of and outdeg); every graph constructor ends with it.
void build_full(DevGraph& g);
// engine.cpp:63-75 as the integer test mix64(key ^ e) < T (keep_all: sigma >= 1)
struct SparsifySpec {
    uint64_t T = 0, key = 0;
    int keep_all = 0;
};
SparsifySpec sparsify_spec(double sigma, uint64_t seed, bool all_ones);
// flags -> sparsified CSC (s_off, padded s_src/s_w) + its run map. Returns
// the kept (local) edge count. With `hash`, the flags are first computed
// into `bitmap` (the initial sparsify, engine.hpp:154-161).
uint64_t rebuild_sparse(DevGraph& g, uint32_t* bitmap, uint64_t* s_off, uint32_t* s_src,
                        void* s_w, ListMeta& meta, cudaEvent_t ev0, cudaEvent_t ev1,
                        int* launches, const SparsifySpec* hash = nullptr);
// Initial sparsification overlapped with the upload (one rank, unweighted):
// chunks of edges [e_lo, e_hi) as their sources land, then the run's layout.
uint64_t presparse_tile_edges();
void presparse_chunk(DevGraph& g, const SparsifySpec& h, uint64_t e_lo, uint64_t e_hi);
uint64_t presparse_finish(DevGraph& g, uint64_t* s_off, ListMeta& meta);
// padded-position base of the sparsified list of this rank (exclusive scan
// of kept counts over ranks, modulo the task size); 0 on one GPU.
uint64_t sparse_pad(DevGraph& g, uint64_t kept_local);
// engine.cpp:63-75 sparsify into a bitmap over local edges (global ids hashed).
void sparsify_bitmap(DevGraph& g, uint32_t* bitmap, double sigma, uint64_t seed, bool all_ones);
// Deferred superstep bad-vertex scan.
void launch_superstep_invalid(DevGraph& g, const uint8_t* st, const uint64_t* s_off, void* ctr);
int occupancy_grid(const void* kernel, int block, size_t smem, int num_sms);

}  // namespace ggb

struct gg_dev_graph {
    ggb::DevGraph g;
};
