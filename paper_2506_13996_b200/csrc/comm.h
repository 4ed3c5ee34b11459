// ProcessGroup for the B200 build.
//   * NCCL mode: one process per GPU; all_to_all = grouped ncclSend/ncclRecv over NVLink/NVSwitch,
//     all_reduce = ncclAllReduce (NVLS-capable).  Async errors -> ProtocolError.
//   * loopback mode: P virtual ranks on one device driven by one host thread — the SPEC's
//     in-process SPMD with device-to-device copies; used to run SP=P on one GPU.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdint>
#include <map>
#include <string>
#include <vector>

#include "../../include/sptrain_b200.h"

struct spt_comm {
    int nranks = 1;
    int rank = 0;  // NCCL mode: this process's rank
    int device = 0;
    bool loopback = false;
    ncclComm_t nccl = nullptr;

    struct Stat {
        int64_t calls = 0;
        int64_t bytes_sent = 0;  // outbound bytes per rank (to peers != self)
    };
    std::map<std::string, Stat> stats;

    int local_ranks() const { return loopback ? nranks : 1; }
    int global_rank(int local) const { return loopback ? local : rank; }

    // recv[j] on rank i = send[i] from rank j; `send`/`recv` hold one base pointer per LOCAL rank,
    // each [nranks][bytes_per_peer].
    void all_to_all(const char* tag, const std::vector<const void*>& send, const std::vector<void*>& recv,
                    size_t bytes_per_peer, cudaStream_t st);
    // In-place sum across ranks.  Loopback: buffers are shared by construction (no-op).
    void all_reduce(const char* tag, void* buf, size_t count, ncclDataType_t dt, cudaStream_t st);
    // out [nranks * count] = concat of every rank's `in` in rank order (local rank 0's pointers).
    void all_gather(const char* tag, const void* in, void* out, size_t bytes, cudaStream_t st);
    void check_async();
    std::string stats_json() const;
};
