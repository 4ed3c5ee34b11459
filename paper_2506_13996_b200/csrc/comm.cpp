#include "comm.h"

#include <dlfcn.h>
#include <unistd.h>

#include <chrono>
#include <thread>

#include <cstring>
#include <mutex>
#include <sstream>

#include "common.h"
#include "launch.h"

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
    ncclResult_t (*CommAbort)(ncclComm_t);
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
        api.CommAbort = (decltype(api.CommAbort))sym("ncclCommAbort");
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

// peer.cu
void peer_barrier(void* const* flag_bufs, int rank, int P, uint64_t* epoch, int64_t timeout_ns, int32_t* err,
                  cudaStream_t st);
int64_t peer_chunk_elems(int64_t count, int P);
void peer_reduce_chunk(void* const* bufs, int P, int rank, int64_t count, int elem_kind, cudaStream_t st);
void peer_gather_chunks(void* const* bufs, int P, int rank, int64_t chunk_bytes, int64_t total_bytes, cudaStream_t st);
void peer_pull(void* const* src, int P, int64_t src_off, int64_t bytes, void* dst, cudaStream_t st);

static size_t dt_bytes(ncclDataType_t dt) {
    return dt == ncclFloat64 || dt == ncclInt64 ? 8 : dt == ncclBfloat16 ? 2 : 4;
}

// One allocation's identity as exchanged between ranks (spt_allgather_fn payload)
struct PeerHandle {
    cudaIpcMemHandle_t ipc;
    int32_t pid;
    int32_t device;
    uint64_t bytes;
    uint64_t ptr;
};
}  // namespace spt

using namespace spt;

// ------------------------------------------------------------------ peer mode: symmetric allocations
void* spt_comm::sym_alloc(size_t bytes) {
    SPT_CHECK(mode == kPeer, SPT_ERR_INTERNAL, "sym_alloc outside peer mode");
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, std::max<size_t>(bytes, 256));
    if (e != cudaSuccess)
        SPT_THROW(SPT_ERR_OOM, "cudaMalloc(" + std::to_string(bytes) + ") failed: " + cudaGetErrorString(e));
    SPT_CUDA(cudaMemset(p, 0, std::max<size_t>(bytes, 256)));
    SymAlloc a;
    a.local = p;
    a.bytes = std::max<size_t>(bytes, 256);
    a.peer.assign(nranks, nullptr);
    a.opened.assign(nranks, 0);
    a.peer[rank] = p;
    sym.push_back(std::move(a));
    return p;
}

void spt_comm::sym_free(void* p) {
    for (auto& a : sym) {
        if (a.local != p || !a.live) continue;
        for (int r = 0; r < nranks; ++r)
            if (a.opened[r]) cudaIpcCloseMemHandle(a.peer[r]);
        cudaFree(a.local);
        a.live = false;
        a.local = nullptr;
        a.peer.assign(nranks, nullptr);
        a.opened.assign(nranks, 0);
        return;
    }
}

// Exchange the identities of the allocations made since the last connect and map the peers' copies.  Every
// rank must have made the same allocations in the same order (CollectiveError otherwise, errors.hpp:24-28).
void spt_comm::connect() {
    if (mode != kPeer || sym_connected == sym.size()) return;
    SPT_CHECK(exchange != nullptr, SPT_ERR_CONFIG, "peer group has no exchange callback");
    const size_t k = sym.size() - sym_connected;
    const size_t per = sizeof(uint64_t) + k * sizeof(PeerHandle);
    std::vector<char> mine(per, 0), all(per * nranks, 0);
    *reinterpret_cast<uint64_t*>(mine.data()) = k;
    for (size_t i = 0; i < k; ++i) {
        auto& a = sym[sym_connected + i];
        PeerHandle h{};
        if (a.live) SPT_CUDA(cudaIpcGetMemHandle(&h.ipc, a.local));
        h.pid = (int32_t)getpid();
        h.device = device;
        h.bytes = a.live ? a.bytes : 0;
        h.ptr = (uint64_t)(uintptr_t)a.local;
        std::memcpy(mine.data() + sizeof(uint64_t) + i * sizeof(PeerHandle), &h, sizeof(h));
    }
    const int32_t rc = exchange(mine.data(), all.data(), per, exchange_user);
    SPT_CHECK(rc == 0, SPT_ERR_COLLECTIVE, "peer handle exchange failed (callback returned " + std::to_string(rc) + ")");
    for (int r = 0; r < nranks; ++r) {
        const char* blk = all.data() + (size_t)r * per;
        SPT_CHECK(*reinterpret_cast<const uint64_t*>(blk) == k, SPT_ERR_COLLECTIVE,
                  "peer group: rank " + std::to_string(r) + " made a different number of symmetric allocations");
        if (r == rank) continue;
        for (size_t i = 0; i < k; ++i) {
            PeerHandle h;
            std::memcpy(&h, blk + sizeof(uint64_t) + i * sizeof(PeerHandle), sizeof(h));
            auto& a = sym[sym_connected + i];
            SPT_CHECK(h.bytes == (a.live ? a.bytes : 0), SPT_ERR_COLLECTIVE,
                      "peer group: symmetric allocation " + std::to_string(sym_connected + i) + " differs in size on rank " +
                          std::to_string(r));
            if (!a.live) continue;
            if (h.pid == (int32_t)getpid()) {  // a rank on another thread of this process: plain pointer
                if (h.device != device) {
                    const cudaError_t e = cudaDeviceEnablePeerAccess(h.device, 0);
                    if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
                    else SPT_CUDA(e);
                }
                a.peer[r] = (void*)(uintptr_t)h.ptr;
            } else {
                void* p = nullptr;
                SPT_CUDA(cudaIpcOpenMemHandle(&p, h.ipc, cudaIpcMemLazyEnablePeerAccess));
                a.peer[r] = p;
                a.opened[r] = 1;
            }
        }
    }
    sym_connected = sym.size();
}

void* spt_comm::peer_ptr(int r, const void* local) const {
    const char* l = static_cast<const char*>(local);
    for (size_t i = 0; i < sym_connected; ++i) {
        const auto& a = sym[i];
        const char* b = static_cast<const char*>(a.local);
        if (a.live && l >= b && l < b + a.bytes) return static_cast<char*>(a.peer[r]) + (l - b);
    }
    SPT_THROW(SPT_ERR_CONFIG, "peer group: pointer is not inside a connected symmetric allocation");
}

void spt_comm::barrier(cudaStream_t st) {
    SPT_CHECK(mode == kPeer, SPT_ERR_INTERNAL, "barrier outside peer mode");
    std::vector<void*> f(nranks);
    for (int r = 0; r < nranks; ++r) f[r] = peer_ptr(r, flags);
    peer_barrier(f.data(), rank, nranks, epoch, timeout_ns, err_dev, st);
}

// ------------------------------------------------------------------ collectives
void spt_comm::all_to_all(const char* tag, const std::vector<const void*>& send, const std::vector<void*>& recv,
                          size_t bytes_per_peer, cudaStream_t st) {
    note(tag, (int64_t)bytes_per_peer * (nranks - 1));
    if (mode == kLoopback) {
        for (int i = 0; i < nranks; ++i)
            for (int j = 0; j < nranks; ++j)
                SPT_CUDA(cudaMemcpyAsync((char*)recv[j] + (size_t)i * bytes_per_peer,
                                         (const char*)send[i] + (size_t)j * bytes_per_peer, bytes_per_peer,
                                         cudaMemcpyDeviceToDevice, st));
        return;
    }
    if (mode == kPeer) {  // recv[j] = peer j's send[rank]: one pull kernel between two barriers
        std::vector<void*> src(nranks);
        for (int r = 0; r < nranks; ++r) src[r] = peer_ptr(r, send[0]);
        barrier(st);
        peer_pull(src.data(), nranks, (int64_t)rank * bytes_per_peer, bytes_per_peer, recv[0], st);
        barrier(st);
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
    const size_t es = dt_bytes(dt);
    note(tag, (int64_t)(count * es * 2 * (nranks - 1) / std::max(1, nranks)));
    if (mode == kLoopback) return;
    if (mode == kPeer) {
        if (nranks == 1) return;
        const int kind = dt == ncclFloat32 ? 0 : dt == ncclFloat64 ? 1 : dt == ncclInt64 ? 2 : -1;
        SPT_CHECK(kind >= 0, SPT_ERR_CONFIG, "peer all_reduce: fp32, fp64 or int64 only");
        std::vector<void*> b(nranks);
        for (int r = 0; r < nranks; ++r) b[r] = peer_ptr(r, buf);
        barrier(st);  // every rank's contribution is complete
        peer_reduce_chunk(b.data(), nranks, rank, (int64_t)count, kind, st);
        barrier(st);  // every chunk is reduced
        peer_gather_chunks(b.data(), nranks, rank, peer_chunk_elems((int64_t)count, nranks) * (int64_t)es,
                           (int64_t)(count * es), st);
        barrier(st);  // nobody reads this rank's buffer any more
        return;
    }
    SPT_NCCL(AllReduce(buf, buf, count, dt, ncclSum, nccl, st));
}

void spt_comm::all_gather(const char* tag, const void* in, void* out, size_t bytes, cudaStream_t st) {
    note(tag, (int64_t)bytes * (nranks - 1));
    if (mode == kLoopback) {
        if (out != in) SPT_CUDA(cudaMemcpyAsync(out, in, bytes * nranks, cudaMemcpyDeviceToDevice, st));
        return;
    }
    if (mode == kPeer) {
        std::vector<void*> src(nranks);
        for (int r = 0; r < nranks; ++r) src[r] = peer_ptr(r, in);
        barrier(st);
        peer_pull(src.data(), nranks, 0, (int64_t)bytes, out, st);
        barrier(st);
        return;
    }
    SPT_NCCL(AllGather(in, out, bytes, ncclChar, nccl, st));
}

void spt_comm::check_async() {
    if (mode == kPeer) {
        SPT_CHECK(*(volatile int32_t*)err_host == 0, SPT_ERR_PROTOCOL,
                  "peer group rank " + std::to_string(rank) + ": a barrier waited longer than " +
                      std::to_string(timeout_ns / 1000000) + " ms (dead, stalled or diverged peer)");
        return;
    }
    if (mode != kNccl || !nccl) return;
    ncclResult_t ar;
    SPT_NCCL(CommGetAsyncError(nccl, &ar));
    if (ar != ncclSuccess && ar != ncclInProgress)
        SPT_THROW(SPT_ERR_PROTOCOL, std::string("NCCL async error: ") + nccl_api().GetErrorString(ar));
}

// Host watchdog: poll the stream instead of blocking in cudaStreamSynchronize, so a collective that never
// completes (a peer died before entering it) turns into ProtocolError after the group's deadline.
void spt_comm::wait_stream(cudaStream_t st) {
    const auto t0 = std::chrono::steady_clock::now();
    for (int it = 0;; ++it) {
        const cudaError_t q = cudaStreamQuery(st);
        if (q == cudaSuccess) break;
        if (q != cudaErrorNotReady) SPT_CUDA(q);
        if (mode != kLoopback) check_async();
        const int64_t waited =
            std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0).count();
        if (mode != kLoopback && waited > timeout_ns + 2000000000ll) {
            if (mode == kNccl && nccl) {
                nccl_api().CommAbort(nccl);  // unblocks the stuck NCCL kernels; the communicator is unusable
                nccl = nullptr;
            }
            SPT_THROW(SPT_ERR_PROTOCOL, "rank " + std::to_string(rank) + ": step did not complete within " +
                                            std::to_string(timeout_ns / 1000000) + " ms (collective stalled)");
        }
        if (it > 100) std::this_thread::sleep_for(std::chrono::microseconds(200));
    }
    if (mode != kLoopback) check_async();
}

std::string spt_comm::stats_json() const {
    std::ostringstream os;
    const char* m = mode == kPeer ? "peer" : mode == kNccl ? "nccl" : "loopback";
    os << "{\"world_size\":" << nranks << ",\"transport\":\"" << m << "\",\"loopback\":" << (loopback ? "true" : "false")
       << ",\"collectives\":{";
    bool first = true;
    for (auto& kv : stats) {
        os << (first ? "" : ",") << "\"" << kv.first << "\":{\"calls\":" << kv.second.calls
           << ",\"bytes_sent_per_rank\":" << kv.second.bytes_sent << "}";
        first = false;
    }
    os << "}}";
    return os.str();
}

static spt_comm* new_comm(int32_t nranks, int32_t rank, int32_t device, spt_comm::Mode mode) {
    SPT_CHECK(nranks >= 1 && nranks <= kMaxSP && rank >= 0 && rank < nranks, SPT_ERR_CONFIG,
              "bad rank/world size (1 <= world <= " + std::to_string(kMaxSP) + ")");
    SPT_CUDA(cudaSetDevice(device));
    auto* c = new spt_comm();
    c->nranks = nranks;
    c->rank = rank;
    c->device = device;
    c->mode = mode;
    c->loopback = mode == spt_comm::kLoopback;
    return c;
}

static void destroy_comm(spt_comm* c) {
    if (!c) return;
    if (c->nccl) nccl_api().CommDestroy(c->nccl);
    for (auto& a : c->sym)
        if (a.live) c->sym_free(a.local);
    if (c->epoch) cudaFree(c->epoch);
    if (c->err_host) cudaFreeHost(c->err_host);
    delete c;
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

// NCCL group: the communicator is created for every world size, including 1, so a single-rank group still
// runs the real ncclAllReduce / ncclAllGather (a 1-rank all_to_all is never issued: P = 1 has no reshard).
spt_status spt_comm_init_rank(const uint8_t id[128], int32_t nranks, int32_t rank, int32_t device, spt_comm** out) {
    return capi_guard([&] {
        spt_comm* c = new_comm(nranks, rank, device, spt_comm::kNccl);
        ncclUniqueId uid;
        std::memcpy(&uid, id, 128);
        ncclResult_t r = ncclSuccess;
        try {
            r = nccl_api().CommInitRank(&c->nccl, nranks, uid, rank);
        } catch (...) {
            delete c;
            throw;
        }
        if (r != ncclSuccess) {
            delete c;
            SPT_THROW(SPT_ERR_COLLECTIVE, std::string("ncclCommInitRank failed: ") + nccl_api().GetErrorString(r));
        }
        *out = c;
    });
}

spt_status spt_comm_init_loopback(int32_t nranks, int32_t device, spt_comm** out) {
    return capi_guard([&] { *out = new_comm(nranks, 0, device, spt_comm::kLoopback); });
}

spt_status spt_comm_init_peer(int32_t nranks, int32_t rank, int32_t device, spt_allgather_fn exchange, void* user,
                              spt_comm** out) {
    return capi_guard([&] {
        SPT_CHECK(exchange != nullptr || nranks == 1, SPT_ERR_CONFIG, "peer group needs an exchange callback");
        spt_comm* c = new_comm(nranks, rank, device, spt_comm::kPeer);
        try {
            c->exchange = exchange;
            c->exchange_user = user;
            SPT_CUDA(cudaMalloc(&c->epoch, sizeof(uint64_t)));
            SPT_CUDA(cudaMemset(c->epoch, 0, sizeof(uint64_t)));
            SPT_CUDA(cudaHostAlloc(&c->err_host, sizeof(int32_t), cudaHostAllocMapped | cudaHostAllocPortable));
            *c->err_host = 0;
            SPT_CUDA(cudaHostGetDevicePointer((void**)&c->err_dev, c->err_host, 0));
            c->flags = (uint64_t*)c->sym_alloc(kMaxSP * sizeof(uint64_t));
            if (nranks > 1) c->connect();
            else c->sym_connected = c->sym.size();
        } catch (...) {
            destroy_comm(c);
            throw;
        }
        *out = c;
    });
}

spt_status spt_comm_set_timeout_ms(spt_comm* comm, int64_t ms) {
    return capi_guard([&] {
        SPT_CHECK(comm && ms > 0, SPT_ERR_CONFIG, "timeout must be > 0 ms");
        comm->timeout_ns = ms * 1000000;
    });
}

spt_status spt_comm_check(spt_comm* comm) {
    return capi_guard([&] { comm->check_async(); });
}

spt_status spt_comm_world(spt_comm* comm, int32_t* nranks, int32_t* rank, int32_t* transport) {
    return capi_guard([&] {
        if (nranks) *nranks = comm->nranks;
        if (rank) *rank = comm->rank;
        if (transport) *transport = (int32_t)comm->mode;
    });
}

spt_status spt_comm_alloc(spt_comm* comm, size_t bytes, void** out) {
    return capi_guard([&] {
        if (comm->mode == spt_comm::kPeer) {
            *out = comm->sym_alloc(bytes);
            return;
        }
        SPT_CUDA(cudaMalloc(out, std::max<size_t>(bytes, 256)));
        SPT_CUDA(cudaMemset(*out, 0, std::max<size_t>(bytes, 256)));
    });
}

spt_status spt_comm_free(spt_comm* comm, void* p) {
    return capi_guard([&] {
        if (comm->mode == spt_comm::kPeer) comm->sym_free(p);
        else cudaFree(p);
    });
}

spt_status spt_comm_connect(spt_comm* comm) {
    return capi_guard([&] {
        if (comm->nranks > 1) comm->connect();
        else comm->sym_connected = comm->sym.size();
    });
}

spt_status spt_comm_barrier(spt_comm* comm, void* stream) {
    return capi_guard([&] {
        if (comm->mode == spt_comm::kPeer && comm->nranks > 1) comm->barrier((cudaStream_t)stream);
        else if (comm->mode == spt_comm::kNccl && comm->nranks > 1) {
            // a zero-payload all-reduce is NCCL's cheapest rendezvous
            static thread_local float* dummy = nullptr;
            if (!dummy) SPT_CUDA(cudaMalloc(&dummy, 4));
            SPT_NCCL(AllReduce(dummy, dummy, 1, ncclFloat32, ncclSum, comm->nccl, (cudaStream_t)stream));
        }
    });
}

spt_status spt_comm_wait(spt_comm* comm, void* stream) {
    return capi_guard([&] { comm->wait_stream((cudaStream_t)stream); });
}

spt_status spt_comm_destroy(spt_comm* comm) {
    return capi_guard([&] { destroy_comm(comm); });
}

spt_status spt_comm_stats_json(spt_comm* comm, char* buf, size_t cap) {
    return capi_guard([&] {
        std::string s = comm->stats_json();
        SPT_CHECK(s.size() + 1 <= cap, SPT_ERR_SHAPE, "buffer too small");
        std::memcpy(buf, s.c_str(), s.size() + 1);
    });
}

// SPEC.md:155-163 all_reduce_sum, in place.  bufs: one pointer per LOCAL rank (loopback: every virtual rank's
// buffer, summed in rank order and written back to all of them; NCCL / peer: bufs[0]; peer mode needs a
// spt_comm_alloc'ed buffer).
static void all_reduce_capi(spt_comm* comm, void* const* bufs, int64_t n, ncclDataType_t dt, cudaStream_t st);
spt_status spt_all_reduce_f32(spt_comm* comm, void* const* bufs, int64_t n, void* stream) {
    return capi_guard([&] { all_reduce_capi(comm, bufs, n, ncclFloat32, (cudaStream_t)stream); });
}
spt_status spt_all_reduce_f64(spt_comm* comm, void* const* bufs, int64_t n, void* stream) {
    return capi_guard([&] { all_reduce_capi(comm, bufs, n, ncclFloat64, (cudaStream_t)stream); });
}
spt_status spt_all_reduce_i64(spt_comm* comm, void* const* bufs, int64_t n, void* stream) {
    return capi_guard([&] { all_reduce_capi(comm, bufs, n, ncclInt64, (cudaStream_t)stream); });
}

// SPEC.md:145-153 all_to_all: recv[j] on rank i = send[i] from rank j (bytes_per_peer each).
spt_status spt_all_to_all(spt_comm* comm, const void* const* send, void* const* recv, size_t bytes_per_peer,
                          void* stream) {
    return capi_guard([&] {
        const int L = comm->local_ranks();
        std::vector<const void*> s(send, send + L);
        std::vector<void*> r(recv, recv + L);
        comm->all_to_all("all_to_all", s, r, bytes_per_peer, (cudaStream_t)stream);
    });
}

}  // extern "C"

static void all_reduce_capi(spt_comm* comm, void* const* bufs, int64_t n, ncclDataType_t dt, cudaStream_t st) {
    if (comm->mode != spt_comm::kLoopback) {
        comm->all_reduce("all_reduce", bufs[0], (size_t)n, dt, st);
        return;
    }
    comm->note("all_reduce", (int64_t)(n * dt_bytes(dt) * 2 * (comm->nranks - 1) / comm->nranks));
    if (comm->nranks == 1) return;
    const int kind = dt == ncclFloat32 ? 0 : dt == ncclFloat64 ? 1 : 2;
    // the virtual ranks' buffers play the peers: the same reduce-scatter / all-gather kernels, one rank at a time
    std::vector<void*> b(bufs, bufs + comm->nranks);
    for (int r = 0; r < comm->nranks; ++r) peer_reduce_chunk(b.data(), comm->nranks, r, n, kind, st);
    for (int r = 0; r < comm->nranks; ++r)
        peer_gather_chunks(b.data(), comm->nranks, r, peer_chunk_elems(n, comm->nranks) * (int64_t)dt_bytes(dt),
                           n * (int64_t)dt_bytes(dt), st);
}
