#include "comm.h"

#include <dlfcn.h>

#include <cstring>
#include <mutex>
#include <sstream>

#include "common.h"

namespace spt {
// NCCL is resolved lazily with dlopen when the first NCCL communicator is created, so loading this
// library never pins an NCCL build into the process: if PyTorch already loaded its NCCL, dlopen
// returns that same library; otherwise the system libnccl.so.2 is used.
struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*);
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
    ncclResult_t (*CommDestroy)(ncclComm_t);
    ncclResult_t (*GroupStart)();
    ncclResult_t (*GroupEnd)();
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
    ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*);
    const char* (*GetErrorString)(ncclResult_t);
};

static const NcclApi& nccl_api() {
    static NcclApi api{};
    static std::once_flag once;
    static std::string err;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            err = std::string("cannot dlopen libnccl.so.2: ") + dlerror();
            return;
        }
        auto sym = [&](const char* n) {
            void* p = dlsym(h, n);
            if (!p && err.empty()) err = std::string("libnccl.so.2 lacks ") + n;
            return p;
        };
        api.GetUniqueId = (decltype(api.GetUniqueId))sym("ncclGetUniqueId");
        api.CommInitRank = (decltype(api.CommInitRank))sym("ncclCommInitRank");
        api.CommDestroy = (decltype(api.CommDestroy))sym("ncclCommDestroy");
        api.GroupStart = (decltype(api.GroupStart))sym("ncclGroupStart");
        api.GroupEnd = (decltype(api.GroupEnd))sym("ncclGroupEnd");
        api.Send = (decltype(api.Send))sym("ncclSend");
        api.Recv = (decltype(api.Recv))sym("ncclRecv");
        api.AllReduce = (decltype(api.AllReduce))sym("ncclAllReduce");
        api.AllGather = (decltype(api.AllGather))sym("ncclAllGather");
        api.CommGetAsyncError = (decltype(api.CommGetAsyncError))sym("ncclCommGetAsyncError");
        api.GetErrorString = (decltype(api.GetErrorString))sym("ncclGetErrorString");
    });
    SPT_CHECK(err.empty(), SPT_ERR_COLLECTIVE, err);
    return api;
}

#define SPT_NCCL(call)                                                                                             \
    do {                                                                                                           \
        ncclResult_t r_ = nccl_api().call;                                                                         \
        if (r_ != ncclSuccess)                                                                                     \
            SPT_THROW(SPT_ERR_COLLECTIVE, std::string("nccl" #call " failed: ") + nccl_api().GetErrorString(r_)); \
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
    SPT_NCCL(GroupStart());
    for (int j = 0; j < nranks; ++j) {
        SPT_NCCL(Send((const char*)send[0] + (size_t)j * bytes_per_peer, bytes_per_peer, ncclChar, j, nccl, st));
        SPT_NCCL(Recv((char*)recv[0] + (size_t)j * bytes_per_peer, bytes_per_peer, ncclChar, j, nccl, st));
    }
    SPT_NCCL(GroupEnd());
}

void spt_comm::all_reduce(const char* tag, void* buf, size_t count, ncclDataType_t dt, cudaStream_t st) {
    auto& s = stats[tag];
    s.calls += 1;
    size_t es = dt == ncclFloat32 ? 4 : dt == ncclFloat64 || dt == ncclInt64 ? 8 : dt == ncclBfloat16 ? 2 : 4;
    s.bytes_sent += (int64_t)(count * es * 2 * (nranks - 1) / std::max(1, nranks));
    if (loopback || nranks == 1) return;
    SPT_NCCL(AllReduce(buf, buf, count, dt, ncclSum, nccl, st));
}

void spt_comm::all_gather(const char* tag, const void* in, void* out, size_t bytes, cudaStream_t st) {
    auto& s = stats[tag];
    s.calls += 1;
    s.bytes_sent += (int64_t)bytes * (nranks - 1);
    if (loopback || nranks == 1) {
        if (out != in) SPT_CUDA(cudaMemcpyAsync(out, in, bytes * (loopback ? nranks : 1), cudaMemcpyDeviceToDevice, st));
        return;
    }
    SPT_NCCL(AllGather(in, out, bytes, ncclChar, nccl, st));
}

void spt_comm::check_async() {
    if (loopback || !nccl) return;
    ncclResult_t ar;
    SPT_NCCL(CommGetAsyncError(nccl, &ar));
    if (ar != ncclSuccess && ar != ncclInProgress)
        SPT_THROW(SPT_ERR_PROTOCOL, std::string("NCCL async error: ") + nccl_api().GetErrorString(ar));
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
        SPT_NCCL(GetUniqueId(&id));
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
            ncclResult_t r = nccl_api().CommInitRank(&c->nccl, nranks, uid, rank);
            if (r != ncclSuccess) {
                delete c;
                SPT_THROW(SPT_ERR_COLLECTIVE, std::string("ncclCommInitRank failed: ") + nccl_api().GetErrorString(r));
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
        if (comm->nccl) nccl_api().CommDestroy(comm->nccl);
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
