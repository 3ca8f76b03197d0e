// loopback.cuh -- an in-process stand-in for the NCCL calls of the
// partitioned path (partition.cuh), for N host threads ("ranks") of ONE
// process that share a device.  NCCL refuses two ranks on one GPU, and the
// boxes this library is tested on have one GPU; with this transport bound
// behind the same NcclApi function table, the complete per-rank code path of
// a multi-GPU run -- slice loading, bounds all-gather, the exchange modes,
// termination, owned-slice / gathered output, the overflow certificate --
// executes exactly as with NCCL, only the bytes move by device copies instead
// of NVLink.  Included by falcon.cu through partition.cuh.
//
// Semantics kept from NCCL: every call is issued on a stream and a rank's
// calls are matched with the other ranks' calls in issue order (collectives
// by position, send/recv per peer pair); ncclGroupStart/End batch calls so
// grouped sends and receives cannot deadlock.  Executing a group is
// host-synchronous here (the streams are synchronised, the ranks meet at a
// barrier, each rank copies what it receives, the ranks meet again) -- a
// stronger ordering than NCCL's, so any program correct under NCCL is
// correct here.  A barrier that waits longer than 120 s fails the call
// (ncclSystemError) instead of hanging.
#pragma once
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <vector>

namespace {

constexpr char LB_MAGIC[8] = {'F', 'L', 'C', 'N', 'L', 'O', 'O', 'P'};

struct LbOp {
    enum Kind { SEND, RECV, REDUCE, ALLREDUCE, BCAST, ALLGATHER } kind;
    const void *send;
    void *recv;
    size_t count;
    ncclDataType_t dt;
    ncclRedOp_t op;
    int peer;   // SEND/RECV: the other rank; REDUCE/BCAST: the root
    cudaStream_t stream;
};

struct LbWorld {
    int nranks = 0, refs = 0;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    uint64_t gen = 0;
    std::vector<std::vector<LbOp>> posted;
    explicit LbWorld(int n) : nranks(n), refs(n), posted((size_t)n) {}
    // false on timeout (a rank never arrived: mismatched collective sequence)
    bool barrier() {
        std::unique_lock<std::mutex> lk(mu);
        const uint64_t g = gen;
        if (++arrived == nranks) {
            arrived = 0;
            gen++;
            cv.notify_all();
            return true;
        }
        return cv.wait_for(lk, std::chrono::seconds(120), [&] { return gen != g; });
    }
};

struct LbComm {
    LbWorld *w;
    int rank;
};

thread_local int tl_lb_depth = 0;
thread_local LbComm *tl_lb_comm = nullptr;
thread_local std::vector<LbOp> tl_lb_ops;
thread_local LbComm *tl_lb_last = nullptr;   // this thread's communicator (an empty group still meets the others)
thread_local std::vector<std::pair<void *, size_t>> tl_lb_tmp;   // per-rank staging buffers, reused

// The i-th staging buffer of this rank's current group (grown, never freed:
// a cudaFree per call would synchronise the device every superstep).
void *lb_tmp(size_t i, size_t bytes) {
    if (tl_lb_tmp.size() <= i) tl_lb_tmp.resize(i + 1, {nullptr, 0});
    auto &b = tl_lb_tmp[i];
    if (b.second < bytes) {
        if (b.first) cudaFree(b.first);
        b.first = nullptr;
        b.second = 0;
        if (cudaMalloc(&b.first, bytes) != cudaSuccess) return nullptr;
        b.second = bytes;
    }
    return b.first;
}

size_t lb_size(ncclDataType_t dt) {
    switch (dt) {
    case ncclInt8: case ncclUint8: return 1;
    case ncclFloat16: case ncclBfloat16: return 2;
    case ncclInt32: case ncclUint32: case ncclFloat32: return 4;
    default: return 8;
    }
}

struct LbSrcs { const void *p[64]; };

template <typename T>
__global__ void k_lb_reduce(LbSrcs s, int P, size_t count, int op, T *out) {
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
        T acc = static_cast<const T *>(s.p[0])[i];
        for (int r = 1; r < P; r++) {
            const T x = static_cast<const T *>(s.p[r])[i];
            acc = op == ncclMin ? (x < acc ? x : acc) : op == ncclMax ? (x > acc ? x : acc) : (T)(acc + x);
        }
        out[i] = acc;
    }
}

cudaError_t lb_reduce(const std::vector<const void *> &srcs, size_t count, ncclDataType_t dt, ncclRedOp_t op,
                      void *out, cudaStream_t s) {
    LbSrcs t{};
    for (size_t r = 0; r < srcs.size(); r++) t.p[r] = srcs[r];
    const int P = (int)srcs.size();
    const unsigned grid = (unsigned)std::min<size_t>(4096, (count + 255) / 256 + 1);
    switch (dt) {
    case ncclInt32: k_lb_reduce<int32_t><<<grid, 256, 0, s>>>(t, P, count, op, (int32_t *)out); break;
    case ncclUint32: k_lb_reduce<uint32_t><<<grid, 256, 0, s>>>(t, P, count, op, (uint32_t *)out); break;
    case ncclInt64: k_lb_reduce<long long><<<grid, 256, 0, s>>>(t, P, count, op, (long long *)out); break;
    case ncclUint64:
        k_lb_reduce<unsigned long long><<<grid, 256, 0, s>>>(t, P, count, op, (unsigned long long *)out);
        break;
    case ncclUint8: k_lb_reduce<uint8_t><<<grid, 256, 0, s>>>(t, P, count, op, (uint8_t *)out); break;
    case ncclInt8: k_lb_reduce<int8_t><<<grid, 256, 0, s>>>(t, P, count, op, (int8_t *)out); break;
    default: return cudaErrorInvalidValue;
    }
    cudaError_t e = cudaGetLastError();
    return e != cudaSuccess ? e : cudaStreamSynchronize(s);
}

// Execute one group of this rank's calls together with the other ranks' groups.
ncclResult_t lb_execute(LbComm *c, std::vector<LbOp> &ops) {
    LbWorld *w = c->w;
    const int me = c->rank;
    for (auto &o : ops)
        if (cudaStreamSynchronize(o.stream) != cudaSuccess) return ncclUnhandledCudaError;
    {
        std::lock_guard<std::mutex> lk(w->mu);
        w->posted[(size_t)me] = ops;
    }
    if (!w->barrier()) return ncclSystemError;
    // phase A: read the other ranks' buffers into private destinations
    struct Pend { void *tmp; void *recv; size_t bytes; cudaStream_t s; };
    std::vector<Pend> pend;
    ncclResult_t rc = ncclSuccess;
    std::vector<int> sends_seen((size_t)w->nranks, 0);   // k-th recv from p <-> k-th send p -> me
    int coll = 0;
    auto coll_op = [&](int r, int k) -> const LbOp * {   // rank r's k-th collective of this group
        int i = 0;
        for (auto &o : w->posted[(size_t)r]) {
            if (o.kind == LbOp::SEND || o.kind == LbOp::RECV) continue;
            if (i++ == k) return &o;
        }
        return nullptr;
    };
    for (auto &o : ops) {
        const size_t bytes = o.count * lb_size(o.dt);
        if (o.kind == LbOp::SEND) continue;
        if (o.kind == LbOp::RECV) {
            int k = sends_seen[(size_t)o.peer]++, i = 0;
            const LbOp *match = nullptr;
            for (auto &x : w->posted[(size_t)o.peer])
                if (x.kind == LbOp::SEND && x.peer == me && i++ == k) { match = &x; break; }
            if (!match || match->count * lb_size(match->dt) != bytes) { rc = ncclInvalidUsage; break; }
            if (bytes && cudaMemcpyAsync(o.recv, match->send, bytes, cudaMemcpyDefault, o.stream) != cudaSuccess)
                rc = ncclUnhandledCudaError;
            continue;
        }
        const int k = coll++;
        std::vector<const LbOp *> all((size_t)w->nranks);
        for (int r = 0; r < w->nranks; r++) {
            all[(size_t)r] = coll_op(r, k);
            if (!all[(size_t)r] || all[(size_t)r]->kind != o.kind || all[(size_t)r]->count != o.count) {
                rc = ncclInvalidUsage;
            }
        }
        if (rc != ncclSuccess) break;
        if (o.kind == LbOp::BCAST) {
            if (bytes && o.recv != all[(size_t)o.peer]->send &&
                cudaMemcpyAsync(o.recv, all[(size_t)o.peer]->send, bytes, cudaMemcpyDefault, o.stream) != cudaSuccess)
                rc = ncclUnhandledCudaError;
        } else if (o.kind == LbOp::ALLGATHER) {
            for (int r = 0; r < w->nranks && rc == ncclSuccess; r++) {
                void *dst = static_cast<char *>(o.recv) + (size_t)r * bytes;
                // my own contribution is written in phase B (send may alias recv)
                if (r == me) continue;
                if (bytes && cudaMemcpyAsync(dst, all[(size_t)r]->send, bytes, cudaMemcpyDefault, o.stream) != cudaSuccess)
                    rc = ncclUnhandledCudaError;
            }
            if (rc == ncclSuccess && bytes) {
                void *tmp = lb_tmp(pend.size(), bytes);
                if (!tmp || cudaMemcpyAsync(tmp, o.send, bytes, cudaMemcpyDefault, o.stream) != cudaSuccess)
                    rc = ncclUnhandledCudaError;
                pend.push_back({tmp, static_cast<char *>(o.recv) + (size_t)me * bytes, bytes, o.stream});
            }
        } else if (o.kind == LbOp::ALLREDUCE || (o.kind == LbOp::REDUCE && o.peer == me)) {
            std::vector<const void *> srcs;
            for (auto *x : all) srcs.push_back(x->send);
            void *tmp = bytes ? lb_tmp(pend.size(), bytes) : nullptr;
            if (bytes && (!tmp || lb_reduce(srcs, o.count, o.dt, o.op, tmp, o.stream) != cudaSuccess))
                rc = ncclUnhandledCudaError;
            pend.push_back({tmp, o.recv, bytes, o.stream});
        }
    }
    for (auto &o : ops) cudaStreamSynchronize(o.stream);
    if (!w->barrier()) return ncclSystemError;   // every read of a peer buffer is complete
    // phase B: write this rank's own destinations
    for (auto &p : pend) {
        if (p.bytes && cudaMemcpyAsync(p.recv, p.tmp, p.bytes, cudaMemcpyDefault, p.s) != cudaSuccess)
            rc = ncclUnhandledCudaError;
        cudaStreamSynchronize(p.s);
    }
    if (!w->barrier()) return ncclSystemError;   // posted[] may be reused by the next group
    return rc;
}

ncclResult_t lb_post(ncclComm_t comm, LbOp op) {
    LbComm *c = reinterpret_cast<LbComm *>(comm);
    tl_lb_last = c;
    if (tl_lb_depth > 0) {
        if (tl_lb_comm && tl_lb_comm != c) return ncclInvalidUsage;   // one communicator per group
        tl_lb_comm = c;
        tl_lb_ops.push_back(op);
        return ncclSuccess;
    }
    std::vector<LbOp> one{op};
    return lb_execute(c, one);
}

ncclResult_t lb_GetUniqueId(ncclUniqueId *) { return ncclInvalidUsage; }   // ids come from falcon_comm_loopback_id
ncclResult_t lb_CommInitRank(ncclComm_t *comm, int nranks, ncclUniqueId id, int rank) {
    if (memcmp(id.internal, LB_MAGIC, 8) != 0) return ncclInvalidArgument;
    LbWorld *w = nullptr;
    memcpy(&w, id.internal + 8, sizeof w);
    if (!w || w->nranks != nranks || rank < 0 || rank >= nranks) return ncclInvalidArgument;
    *comm = reinterpret_cast<ncclComm_t>(new LbComm{w, rank});
    return ncclSuccess;
}
ncclResult_t lb_CommDestroy(ncclComm_t comm) {
    LbComm *c = reinterpret_cast<LbComm *>(comm);
    bool last = false;
    {
        std::lock_guard<std::mutex> lk(c->w->mu);
        last = --c->w->refs == 0;
    }
    if (last) delete c->w;
    delete c;
    return ncclSuccess;
}
ncclResult_t lb_Reduce(const void *s, void *r, size_t n, ncclDataType_t dt, ncclRedOp_t op, int root, ncclComm_t c,
                       cudaStream_t st) {
    return lb_post(c, {LbOp::REDUCE, s, r, n, dt, op, root, st});
}
ncclResult_t lb_AllReduce(const void *s, void *r, size_t n, ncclDataType_t dt, ncclRedOp_t op, ncclComm_t c,
                          cudaStream_t st) {
    return lb_post(c, {LbOp::ALLREDUCE, s, r, n, dt, op, 0, st});
}
ncclResult_t lb_Broadcast(const void *s, void *r, size_t n, ncclDataType_t dt, int root, ncclComm_t c,
                          cudaStream_t st) {
    return lb_post(c, {LbOp::BCAST, s, r, n, dt, ncclSum, root, st});
}
ncclResult_t lb_Send(const void *s, size_t n, ncclDataType_t dt, int peer, ncclComm_t c, cudaStream_t st) {
    return lb_post(c, {LbOp::SEND, s, nullptr, n, dt, ncclSum, peer, st});
}
ncclResult_t lb_Recv(void *r, size_t n, ncclDataType_t dt, int peer, ncclComm_t c, cudaStream_t st) {
    return lb_post(c, {LbOp::RECV, nullptr, r, n, dt, ncclSum, peer, st});
}
ncclResult_t lb_AllGather(const void *s, void *r, size_t n, ncclDataType_t dt, ncclComm_t c, cudaStream_t st) {
    return lb_post(c, {LbOp::ALLGATHER, s, r, n, dt, ncclSum, 0, st});
}
ncclResult_t lb_GroupStart() {
    tl_lb_depth++;
    return ncclSuccess;
}
ncclResult_t lb_GroupEnd() {
    if (tl_lb_depth <= 0) return ncclInvalidUsage;
    if (--tl_lb_depth > 0) return ncclSuccess;
    std::vector<LbOp> ops;
    ops.swap(tl_lb_ops);
    LbComm *c = tl_lb_comm ? tl_lb_comm : tl_lb_last;
    tl_lb_comm = nullptr;
    return c ? lb_execute(c, ops) : ncclSuccess;
}
const char *lb_GetErrorString(ncclResult_t r) {
    switch (r) {
    case ncclSuccess: return "success";
    case ncclUnhandledCudaError: return "loopback: CUDA error";
    case ncclSystemError: return "loopback: a rank did not arrive within 120 s (mismatched calls?)";
    case ncclInvalidArgument: return "loopback: invalid argument";
    case ncclInvalidUsage: return "loopback: calls do not match across ranks";
    default: return "loopback: error";
    }
}

}  // namespace
