// ProcessGroup for the B200 build.  Three transports behind one interface:
//   * peer mode (the B200-native default for one process per GPU): every rank's communication buffers live
//     in a symmetric set of allocations (same sizes, same order on every rank), mapped into every peer over
//     NVLink / NVSwitch with CUDA IPC (or directly, for ranks in the same process).  The Ulysses reshard
//     kernels then move the data themselves: K1 stores each packed row straight into the destination rank's
//     receive buffer, K2 loads each row straight from the source rank's attention output, so the all-to-all
//     IS the pack / unpack kernel.  Ordering comes from a device-side barrier (release / acquire flags at
//     system scope) before and after each exchange; a barrier that waits longer than the group's timeout
//     raises the group's error flag -> ProtocolError (errors.hpp:30-34) instead of hanging.
//     all_reduce = reduce-scatter + all-gather over peer loads, summing in ascending rank order: the SPEC's
//     fixed-order sum, bitwise reproducible.
//   * NCCL mode (the library baseline): all_to_all = grouped ncclSend/ncclRecv between staging buffers and
//     the pack / unpack kernels, all_reduce = ncclAllReduce.  Async errors and a host-side deadline ->
//     ncclCommAbort + ProtocolError.
//   * loopback mode: P virtual ranks on one device driven by one host thread (the SPEC's in-process SPMD,
//     SPEC.md:183).  The reshard kernels use the same fused direct-store / direct-load form as peer mode,
//     with the peers' buffers being the other virtual ranks' buffers.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdint>
#include <map>
#include <string>
#include <vector>

#include "../../include/sptrain_b200.h"
#include "launch.h"

struct spt_comm {
    enum Mode { kLoopback = 0, kNccl = 1, kPeer = 2 };
    Mode mode = kLoopback;
    int nranks = 1;
    int rank = 0;  // NCCL / peer mode: this process's (or thread's) rank
    int device = 0;
    bool loopback = false;  // == (mode == kLoopback)
    ncclComm_t nccl = nullptr;
    int64_t timeout_ns = 300ll * 1000 * 1000 * 1000;  // barrier / host watchdog deadline

    struct Stat {
        int64_t calls = 0;
        int64_t bytes_sent = 0;  // outbound bytes per rank (to peers != self)
    };
    std::map<std::string, Stat> stats;

    // ---- peer mode state
    spt_allgather_fn exchange = nullptr;
    void* exchange_user = nullptr;
    struct SymAlloc {
        void* local = nullptr;
        size_t bytes = 0;
        std::vector<void*> peer;  // [nranks] base address of every rank's copy, as mapped here
        std::vector<char> opened;  // [nranks] 1: opened with cudaIpcOpenMemHandle (close on free)
        bool live = true;
    };
    std::vector<SymAlloc> sym;  // creation order: identical on every rank
    size_t sym_connected = 0;   // allocations [0, sym_connected) are mapped on this rank
    uint64_t* flags = nullptr;  // symmetric [kMaxSP]: arrival epoch of each peer at the latest barrier
    uint64_t* epoch = nullptr;  // local device counter of barriers entered (graph-replay safe)
    int32_t* err_host = nullptr;  // pinned, mapped: 1 = a barrier timed out
    int32_t* err_dev = nullptr;   // device alias of err_host

    int local_ranks() const { return loopback ? nranks : 1; }
    int global_rank(int local) const { return loopback ? local : rank; }
    bool peer() const { return mode == kPeer; }

    // recv[j] on rank i = send[i] from rank j; `send`/`recv` hold one base pointer per LOCAL rank,
    // each [nranks][bytes_per_peer].  Peer mode: send must be a symmetric allocation (pulled by the peers).
    void all_to_all(const char* tag, const std::vector<const void*>& send, const std::vector<void*>& recv,
                    size_t bytes_per_peer, cudaStream_t st);
    // In-place sum across ranks.  Loopback: buffers are shared by construction (no-op).  Peer mode: buf must be
    // (inside) a symmetric allocation.
    void all_reduce(const char* tag, void* buf, size_t count, ncclDataType_t dt, cudaStream_t st);
    // out [nranks * count] = concat of every rank's `in` in rank order (local rank 0's pointers).
    void all_gather(const char* tag, const void* in, void* out, size_t bytes, cudaStream_t st);
    // Record a collective that the fused reshard kernels performed (CommStats).
    void note(const char* tag, int64_t bytes_sent) {
        auto& s = stats[tag];
        s.calls += 1;
        s.bytes_sent += bytes_sent;
    }
    // Throws ProtocolError when a barrier timed out or NCCL reported an asynchronous error.
    void check_async();
    // Wait for `st` to drain with the group's deadline (NCCL: abort the communicator on expiry).
    void wait_stream(cudaStream_t st);
    std::string stats_json() const;

    // ---- peer mode
    void* sym_alloc(size_t bytes);  // zero-filled device allocation, same on every rank
    void sym_free(void* p);
    void connect();  // map every allocation made since the last connect (calls `exchange`)
    void* peer_ptr(int r, const void* local) const;  // rank r's copy of the symmetric address `local`
    void barrier(cudaStream_t st);
};

namespace spt {

// seq_to_head with the all-to-all fused into K1 (payload layout :351).  `launch(r, tab)` runs
// local rank r's pack into the row table `tab`; outs[r] is local rank r's receive buffer [P * s_loc][row].
//   loopback: rank r's rows go straight into every virtual rank's receive buffer (tab.p[j] = outs[j]);
//   peer:     straight into every peer's receive buffer over NVLink, between two barriers;
//   NCCL:     into the contiguous staging buffer `send`, then grouped ncclSend / ncclRecv into outs[0].
template <class F>
void fused_seq_to_head(spt_comm* cm, const char* tag, const std::vector<void*>& outs, void* send, int64_t s_loc,
                       int64_t row_bytes, cudaStream_t st, F&& launch) {
    const int P = cm->nranks;
    const int64_t peer_bytes = s_loc * row_bytes;
    RowTab t{};
    if (cm->mode == spt_comm::kLoopback) {
        for (int r = 0; r < P; ++r) {
            for (int j = 0; j < P; ++j) t.p[j] = outs[j];
            t.row_off = (int64_t)r * s_loc;
            launch(r, t);
        }
        cm->note(tag, peer_bytes * (P - 1));
    } else if (cm->mode == spt_comm::kPeer) {
        for (int j = 0; j < P; ++j) t.p[j] = cm->peer_ptr(j, outs[0]);
        t.row_off = (int64_t)cm->rank * s_loc;
        cm->barrier(st);  // every peer is done reading its receive buffer's previous contents
        launch(0, t);
        cm->barrier(st);  // every peer's rows have landed here
        cm->note(tag, peer_bytes * (P - 1));
    } else {
        launch(0, contiguous_rows(send, P, s_loc, row_bytes));
        cm->all_to_all(tag, {send}, {outs[0]}, (size_t)peer_bytes, st);
    }
}

// head_to_seq with the all-to-all fused into K2: `launch(r, tab)` runs local rank r's unpack
// reading source rank j's rows from tab.p[j]; srcs[r] is local rank r's head-sharded buffer [P * s_loc][row].
//   loopback / peer: loads straight from the sources (peers: over NVLink, between two barriers);
//   NCCL: ncclSend / ncclRecv of srcs[0] into the staging buffer `recv`, then the unpack from it.
template <class F>
void fused_head_to_seq(spt_comm* cm, const char* tag, const std::vector<void*>& srcs, void* recv, int64_t s_loc,
                       int64_t row_bytes, cudaStream_t st, F&& launch) {
    const int P = cm->nranks;
    const int64_t peer_bytes = s_loc * row_bytes;
    RowTab t{};
    if (cm->mode == spt_comm::kLoopback) {
        for (int r = 0; r < P; ++r) {
            for (int j = 0; j < P; ++j) t.p[j] = srcs[j];
            t.row_off = (int64_t)r * s_loc;
            launch(r, t);
        }
        cm->note(tag, peer_bytes * (P - 1));
    } else if (cm->mode == spt_comm::kPeer) {
        for (int j = 0; j < P; ++j) t.p[j] = cm->peer_ptr(j, srcs[0]);
        t.row_off = (int64_t)cm->rank * s_loc;
        cm->barrier(st);  // every peer's source rows are written
        launch(0, t);
        cm->barrier(st);  // every peer has read this rank's rows
        cm->note(tag, peer_bytes * (P - 1));
    } else {
        cm->all_to_all(tag, {srcs[0]}, {recv}, (size_t)peer_bytes, st);
        launch(0, contiguous_rows(recv, P, s_loc, row_bytes));
    }
}

}  // namespace spt
