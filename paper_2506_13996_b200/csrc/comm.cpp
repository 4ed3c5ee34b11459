#include "comm.h"

#include <cstring>
#include <sstream>

#include "common.h"

namespace spt {
#define SPT_NCCL(call)                                                                                       \
    do {                                                                                                     \
        ncclResult_t r_ = (call);                                                                            \
        if (r_ != ncclSuccess) SPT_THROW(SPT_ERR_COLLECTIVE, std::string(#call " failed: ") + ncclGetErrorString(r_)); \
    } while (0)
}  // namespace spt

using namespace spt;

void spt_comm::all_to_all(const char* tag, const std::vector<const void*>& send, const std::vector<void*>& recv,
                          size_t bytes_per_peer, cudaStream_t st) {
    auto& s = stats[tag];
    s.calls += 1;
    s.bytes_sent += (int64_t)bytes_per_peer * (nranks - 1);
    if (loopback) {
        for (int i = 0; i < nranks; ++i)
            for (int j = 0; j < nranks; ++j)
                SPT_CUDA(cudaMemcpyAsync((char*)recv[j] + (size_t)i * bytes_per_peer,
                                         (const char*)send[i] + (size_t)j * bytes_per_peer, bytes_per_peer,
                                         cudaMemcpyDeviceToDevice, st));
        return;
    }
    SPT_NCCL(ncclGroupStart());
    for (int j = 0; j < nranks; ++j) {
        SPT_NCCL(ncclSend((const char*)send[0] + (size_t)j * bytes_per_peer, bytes_per_peer, ncclChar, j, nccl, st));
        SPT_NCCL(ncclRecv((char*)recv[0] + (size_t)j * bytes_per_peer, bytes_per_peer, ncclChar, j, nccl, st));
    }
    SPT_NCCL(ncclGroupEnd());
}

void spt_comm::all_reduce(const char* tag, void* buf, size_t count, ncclDataType_t dt, cudaStream_t st) {
    auto& s = stats[tag];
    s.calls += 1;
    size_t es = dt == ncclFloat32 ? 4 : dt == ncclFloat64 || dt == ncclInt64 ? 8 : dt == ncclBfloat16 ? 2 : 4;
    s.bytes_sent += (int64_t)(count * es * 2 * (nranks - 1) / std::max(1, nranks));
    if (loopback || nranks == 1) return;
    SPT_NCCL(ncclAllReduce(buf, buf, count, dt, ncclSum, nccl, st));
}

void spt_comm::all_gather(const char* tag, const void* in, void* out, size_t bytes, cudaStream_t st) {
    auto& s = stats[tag];
    s.calls += 1;
    s.bytes_sent += (int64_t)bytes * (nranks - 1);
    if (loopback || nranks == 1) {
        if (out != in) SPT_CUDA(cudaMemcpyAsync(out, in, bytes * (loopback ? nranks : 1), cudaMemcpyDeviceToDevice, st));
        return;
    }
    SPT_NCCL(ncclAllGather(in, out, bytes, ncclChar, nccl, st));
}

void spt_comm::check_async() {
    if (loopback || !nccl) return;
    ncclResult_t ar;
    SPT_NCCL(ncclCommGetAsyncError(nccl, &ar));
    if (ar != ncclSuccess && ar != ncclInProgress)
        SPT_THROW(SPT_ERR_PROTOCOL, std::string("NCCL async error: ") + ncclGetErrorString(ar));
}

std::string spt_comm::stats_json() const {
    std::ostringstream os;
    os << "{\"world_size\":" << nranks << ",\"loopback\":" << (loopback ? "true" : "false") << ",\"collectives\":{";
    bool first = true;
    for (auto& kv : stats) {
        os << (first ? "" : ",") << "\"" << kv.first << "\":{\"calls\":" << kv.second.calls
           << ",\"bytes_sent_per_rank\":" << kv.second.bytes_sent << "}";
        first = false;
    }
    os << "}}";
    return os.str();
}

extern "C" {

spt_status spt_comm_unique_id(uint8_t out_id[128]) {
    return capi_guard([&] {
        ncclUniqueId id;
        SPT_NCCL(ncclGetUniqueId(&id));
        static_assert(sizeof(id) == 128, "ncclUniqueId size");
        std::memcpy(out_id, &id, 128);
    });
}

spt_status spt_comm_init_rank(const uint8_t id[128], int32_t nranks, int32_t rank, int32_t device, spt_comm** out) {
    return capi_guard([&] {
        SPT_CHECK(nranks >= 1 && rank >= 0 && rank < nranks, SPT_ERR_CONFIG, "bad rank/world size");
        SPT_CUDA(cudaSetDevice(device));
        auto* c = new spt_comm();
        c->nranks = nranks;
        c->rank = rank;
        c->device = device;
        if (nranks > 1) {
            ncclUniqueId uid;
            std::memcpy(&uid, id, 128);
            ncclResult_t r = ncclCommInitRank(&c->nccl, nranks, uid, rank);
            if (r != ncclSuccess) {
                delete c;
                SPT_THROW(SPT_ERR_COLLECTIVE, std::string("ncclCommInitRank failed: ") + ncclGetErrorString(r));
            }
        }
        *out = c;
    });
}

spt_status spt_comm_init_loopback(int32_t nranks, int32_t device, spt_comm** out) {
    return capi_guard([&] {
        SPT_CHECK(nranks >= 1, SPT_ERR_CONFIG, "bad world size");
        SPT_CUDA(cudaSetDevice(device));
        auto* c = new spt_comm();
        c->nranks = nranks;
        c->rank = 0;
        c->device = device;
        c->loopback = true;
        *out = c;
    });
}

spt_status spt_comm_destroy(spt_comm* comm) {
    return capi_guard([&] {
        if (!comm) return;
        if (comm->nccl) ncclCommDestroy(comm->nccl);
        delete comm;
    });
}

spt_status spt_comm_stats_json(spt_comm* comm, char* buf, size_t cap) {
    return capi_guard([&] {
        std::string s = comm->stats_json();
        SPT_CHECK(s.size() + 1 <= cap, SPT_ERR_SHAPE, "buffer too small");
        std::memcpy(buf, s.c_str(), s.size() + 1);
    });
}

}  // extern "C"
