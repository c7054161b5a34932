// comm.h -- collectives of the row-sharded join: a per-step
// all-gather of one u64 per rank (pair / row counts) and grouped point-to-point
// exchange of partial-embedding rows for rebalancing.  Two backends:
//   NcclComm   -- the ncclComm_t torch created (ProcessGroupNCCL._comm_ptr()),
//                 libnccl.so.2 resolved with dlopen (the copy torch loaded);
//   LocalComm  -- in-process ranks (threads) sharing one device, used to test
//                 the sharding and rebalancing logic on a single GPU.
#pragma once
#include <stdint.h>

#include <condition_variable>
#include <mutex>
#include <vector>

#include "internal.cuh"

namespace gps {

struct P2POp {
    int peer;
    const void* send;    // device pointer (may be null when send_bytes == 0)
    size_t send_bytes;
    void* recv;          // device pointer
    size_t recv_bytes;
};

struct Comm {
    int rank = 0, world = 1;
    virtual ~Comm() = default;
    // d_recv[world * count] <- every rank's d_send[count] (rank-major), stream-ordered on s
    virtual void allgather_u64(const uint64_t* d_send, uint64_t* d_recv, size_t count, cudaStream_t s) = 0;
    // grouped send/recv (each op pairs with the peer's mirror op)
    virtual void exchange(const std::vector<P2POp>& ops, cudaStream_t s) = 0;
};

Comm* make_nccl_comm(void* nccl_comm, int rank, int world);

// Host arithmetic of the row-sharded join; pure functions of the
// all-gathered counts, identical on every rank.
struct ShardPlan {
    bool rebalance = false;                 // max/mean pairs per rank > threshold
    uint64_t total = 0;                     // global pairs of the step
    std::vector<uint64_t> local_targets;    // [world+1]: rank t takes the local rows i with
                                            // local_targets[t] <= poff[i] < local_targets[t+1]
                                            // (clamped to [0, local pairs + 1])
};
// pairs_all[t] = rank t's local pairs; rank order is the global order.
ShardPlan shard_plan(int world, int rank, const uint64_t* pairs_all, float threshold);
struct ShardRecv {
    std::vector<uint64_t> at;               // [world]: row offset of source t's block in the receive buffer
    uint64_t total = 0;                     // rows received (own block included)
};
// send[src * world + dst] = rows src sends to dst (all-gathered matrix).
ShardRecv shard_recv(int world, int rank, const uint64_t* send);

// Shared state of in-process ranks.
struct LocalHub {
    int world;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    uint64_t gen = 0;
    std::vector<const void*> ptrs;     // per-rank published device pointers
    std::vector<std::vector<P2POp>> ops;
    explicit LocalHub(int w) : world(w), ptrs(w), ops(w) {}
    void barrier();
};
Comm* make_local_comm(LocalHub* hub, int rank);

}  // namespace gps

struct gps_local_comm {
    gps::LocalHub hub;
    explicit gps_local_comm(int w) : hub(w) {}
};
