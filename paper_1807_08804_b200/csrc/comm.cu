// comm.cu -- NCCL and in-process backends of the row-sharded join's collectives.
#include <dlfcn.h>

#include <algorithm>
#include <string>

#include "comm.h"

namespace gps {

// ---------------------------------------------------------------- NCCL
namespace {
typedef int ncclResult_t;
typedef void* ncclComm_t;
enum { ncclUint64 = 5, ncclUint8 = 1 };
struct NcclApi {
    ncclResult_t (*AllGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    bool ok = false;
    std::string why;
};

NcclApi& nccl() {
    static NcclApi api;
    static bool tried = false;
    if (!tried) {
        tried = true;
        // RTLD_NOLOAD first: reuse the libnccl torch already loaded, else load the soname
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            api.why = "libnccl.so.2 not found";
            return api;
        }
        api.AllGather = (decltype(api.AllGather))dlsym(h, "ncclAllGather");
        api.Send = (decltype(api.Send))dlsym(h, "ncclSend");
        api.Recv = (decltype(api.Recv))dlsym(h, "ncclRecv");
        api.GroupStart = (decltype(api.GroupStart))dlsym(h, "ncclGroupStart");
        api.GroupEnd = (decltype(api.GroupEnd))dlsym(h, "ncclGroupEnd");
        api.GetErrorString = (decltype(api.GetErrorString))dlsym(h, "ncclGetErrorString");
        api.ok = api.AllGather && api.Send && api.Recv && api.GroupStart && api.GroupEnd;
        if (!api.ok) api.why = "libnccl.so.2 lacks a required symbol";
    }
    return api;
}

void nccl_ck(ncclResult_t r, const char* what) {
    if (r != 0) {
        const char* s = nccl().GetErrorString ? nccl().GetErrorString(r) : "?";
        fail(GPS_ENCCL, std::string(what) + ": " + s);
    }
}

struct NcclComm : Comm {
    ncclComm_t comm;
    void allgather_u64(const uint64_t* d_send, uint64_t* d_recv, size_t count, cudaStream_t s) override {
        nccl_ck(nccl().AllGather(d_send, d_recv, count, ncclUint64, comm, s), "ncclAllGather");
    }
    void exchange(const std::vector<P2POp>& ops, cudaStream_t s) override {
        nccl_ck(nccl().GroupStart(), "ncclGroupStart");
        for (const P2POp& o : ops) {
            if (o.send_bytes) nccl_ck(nccl().Send(o.send, o.send_bytes, ncclUint8, o.peer, comm, s), "ncclSend");
            if (o.recv_bytes) nccl_ck(nccl().Recv(o.recv, o.recv_bytes, ncclUint8, o.peer, comm, s), "ncclRecv");
        }
        nccl_ck(nccl().GroupEnd(), "ncclGroupEnd");
    }
};
}  // namespace

Comm* make_nccl_comm(void* c, int rank, int world) {
    if (!nccl().ok) fail(GPS_ENCCL, nccl().why);
    NcclComm* x = new NcclComm();
    x->comm = c;
    x->rank = rank;
    x->world = world;
    return x;
}

// ------------------------------------------------------- shard arithmetic
ShardPlan shard_plan(int world, int rank, const uint64_t* Pall, float thr) {
    ShardPlan sp;
    uint64_t S = 0, mx = 0;
    for (int t = 0; t < world; t++) {
        if (t < rank) S += Pall[t];
        sp.total += Pall[t];
        mx = std::max(mx, Pall[t]);
    }
    const double mean = (double)sp.total / world;
    sp.rebalance = sp.total > 0 && (double)mx > (double)thr * mean;
    sp.local_targets.resize(world + 1);
    const uint64_t q = sp.total / world, rem = sp.total % world;
    for (int t = 0; t <= world; t++) {
        // global start of rank t's share = pairs_range(total, t, world).lo (t = world: total)
        const uint64_t T = t == world ? sp.total : q * t + ((uint64_t)t < rem ? (uint64_t)t : rem);
        // rows are assigned by their GLOBAL first pair g = S + poff[i] (T_t <= g < T_{t+1}, the
        // last rank also takes g = total), so every rank cuts consistently; a share starting past
        // this rank's pairs maps to pairs + 1 (no local row reaches it)
        sp.local_targets[t] = T <= S ? 0 : std::min<uint64_t>(T - S, Pall[rank] + 1);
    }
    return sp;
}

ShardRecv shard_recv(int world, int rank, const uint64_t* send) {
    ShardRecv r;
    r.at.resize(world);
    for (int src = 0; src < world; src++) {
        r.at[src] = r.total;
        r.total += send[(size_t)src * world + rank];
    }
    return r;
}

// ----------------------------------------------------------- in-process
void LocalHub::barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const uint64_t g = gen;
    if (++arrived == world) {
        arrived = 0;
        gen++;
        cv.notify_all();
    } else {
        cv.wait(lk, [&] { return gen != g; });
    }
}

namespace {
struct LocalComm : Comm {
    LocalHub* hub;
    void allgather_u64(const uint64_t* d_send, uint64_t* d_recv, size_t count, cudaStream_t s) override {
        GPS_CK(cudaStreamSynchronize(s));
        hub->ptrs[rank] = d_send;
        hub->barrier();
        for (int r = 0; r < world; r++)
            GPS_CK(cudaMemcpyAsync(d_recv + (size_t)r * count, hub->ptrs[r], sizeof(uint64_t) * count,
                                   cudaMemcpyDeviceToDevice, s));
        GPS_CK(cudaStreamSynchronize(s));
        hub->barrier();   // peers may reuse their send buffer only after every rank copied it
    }
    void exchange(const std::vector<P2POp>& ops, cudaStream_t s) override {
        GPS_CK(cudaStreamSynchronize(s));
        hub->ops[rank] = ops;
        hub->barrier();
        for (const P2POp& o : ops) {
            if (!o.recv_bytes) continue;
            const P2POp* mirror = nullptr;
            for (const P2POp& p : hub->ops[o.peer])
                if (p.peer == rank) mirror = &p;
            if (!mirror || mirror->send_bytes != o.recv_bytes) fail(GPS_ENCCL, "local exchange size mismatch");
            GPS_CK(cudaMemcpyAsync(o.recv, mirror->send, o.recv_bytes, cudaMemcpyDeviceToDevice, s));
        }
        GPS_CK(cudaStreamSynchronize(s));
        hub->barrier();
    }
};
}  // namespace

Comm* make_local_comm(LocalHub* hub, int rank) {
    LocalComm* x = new LocalComm();
    x->hub = hub;
    x->rank = rank;
    x->world = hub->world;
    return x;
}

}  // namespace gps
