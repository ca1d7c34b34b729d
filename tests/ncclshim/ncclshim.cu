// tests/ncclshim/ncclshim.cu -- TEST INFRASTRUCTURE: a stand-in libnccl for running
// the library's NCCL transport (paper_2502_05279_b200/csrc/dist.cu) with P > 1
// ranks when only ONE GPU is available.  Real NCCL refuses two ranks on one
// device; this shim implements the five entry points dist.cu dlopens --
// ncclGroupStart/End, ncclSend/Recv, ncclAllReduce (sum of doubles) and
// ncclGetErrorString -- between P processes on the same GPU with CUDA IPC:
//
//   * every rank owns one device staging buffer (IPC-exported) split into P
//     regions; the messages it sends to peer q in one group are copied, in
//     posting order, into region q, and the group's sequence number and byte
//     count are published in a shared host page (an mmap'ed file);
//   * the receiver waits for that sequence number, copies its messages in
//     posting order out of the peer's region (IPC-opened) and publishes that it
//     consumed them; a sender waits for the consumption before reusing a region.
//
// Semantics are NCCL's for what dist.cu relies on: point-to-point messages
// between a pair are matched in posting order within a group, a group
// completes as a whole, and the data dependencies follow the stream order
// (the shim synchronises the stream at ncclGroupEnd, so it is blocking where
// NCCL is asynchronous -- a functional stand-in, not a performance model).
// The all-reduce sums the ranks' values in rank order (deterministic).
//
// Created by shimCommInit(path, rank, nranks, capacity_bytes) from the test
// (tests/test_gpu_dist_shim.py); the returned pointer is passed to dist.cu as the
// ncclComm_t.  Uses nccl.h only for the types, so the signatures are exactly
// NCCL's.
#include <cuda_runtime.h>
#include <fcntl.h>
#include <nccl.h>
#include <sched.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>
#include <sys/mman.h>
#include <unistd.h>

#include <vector>

namespace {

constexpr int MAXR = 16;

struct Shared {  // the mmap'ed page every rank sees
    volatile int joined;
    cudaIpcMemHandle_t stage[MAXR];
    volatile long long pub_seq[MAXR][MAXR];   // [sender][receiver]: last group published
    volatile long long pub_bytes[MAXR][MAXR];
    volatile long long cons_seq[MAXR][MAXR];  // [sender][receiver]: last group consumed by receiver
    volatile long long red_seq[MAXR];
    volatile double red_val[MAXR][64];
};

struct Op {
    bool send;
    void *buf;
    size_t bytes;
    int peer;
    cudaStream_t s;
};

struct Comm {
    int rank = 0, nranks = 1;
    size_t cap = 0;  // bytes per region
    Shared *sh = nullptr;
    char *stage = nullptr;            // own staging buffer (P regions)
    char *peer_stage[MAXR] = {};      // IPC-opened peers' buffers
    long long seq[MAXR] = {};         // groups sent to each peer
    long long rseq[MAXR] = {};        // groups received from each peer
    long long red = 0;
    int depth = 0;
    std::vector<Op> ops;
};

Comm *g_last = nullptr;

void spin() { sched_yield(); }

ncclResult_t flush(Comm *c)
{
    if (c->ops.empty())
        return ncclSuccess;
    for (const Op &o : c->ops)
        if (cudaStreamSynchronize(o.s) != cudaSuccess)
            return ncclUnhandledCudaError;
    const int P = c->nranks, me = c->rank;
    // sends: per peer, concatenate in posting order into region [peer] of my staging buffer
    std::vector<size_t> off(P, 0);
    std::vector<bool> has(P, false);
    for (const Op &o : c->ops)
        if (o.send)
            has[o.peer] = true;
    for (int q = 0; q < P; q++)
        if (has[q])
            while (c->sh->cons_seq[me][q] != c->seq[q])  // region free (the peer consumed the last group)
                spin();
    for (const Op &o : c->ops) {
        if (!o.send)
            continue;
        if (off[o.peer] + o.bytes > c->cap)
            return ncclInternalError;
        // cudaMemcpy D2D does not wait for completion: copy on the op's stream, then sync
        if (cudaMemcpyAsync(c->stage + (size_t)o.peer * c->cap + off[o.peer], o.buf, o.bytes,
                            cudaMemcpyDeviceToDevice, o.s) != cudaSuccess ||
            cudaStreamSynchronize(o.s) != cudaSuccess)
            return ncclUnhandledCudaError;
        off[o.peer] += o.bytes;
    }
    for (int q = 0; q < P; q++)
        if (has[q]) {
            c->sh->pub_bytes[me][q] = (long long)off[q];
            __sync_synchronize();
            c->sh->pub_seq[me][q] = ++c->seq[q];
        }
    // receives: per peer, in posting order out of region [me] of the peer's staging buffer
    std::vector<size_t> roff(P, 0);
    std::vector<bool> rhas(P, false);
    for (const Op &o : c->ops)
        if (!o.send)
            rhas[o.peer] = true;
    for (int q = 0; q < P; q++)
        if (rhas[q])
            while (c->sh->pub_seq[q][me] != c->rseq[q] + 1)
                spin();
    __sync_synchronize();
    for (const Op &o : c->ops) {
        if (o.send)
            continue;
        if (roff[o.peer] + o.bytes > (size_t)c->sh->pub_bytes[o.peer][me])
            return ncclInvalidUsage;  // more bytes posted than the peer sent
        if (cudaMemcpyAsync(o.buf, c->peer_stage[o.peer] + (size_t)me * c->cap + roff[o.peer], o.bytes,
                            cudaMemcpyDeviceToDevice, o.s) != cudaSuccess ||
            cudaStreamSynchronize(o.s) != cudaSuccess)  // the peer may reuse its region once we publish
            return ncclUnhandledCudaError;
        roff[o.peer] += o.bytes;
    }
    for (int q = 0; q < P; q++)
        if (rhas[q]) {
            if (roff[q] != (size_t)c->sh->pub_bytes[q][me])
                return ncclInvalidUsage;  // posted receives do not match the peer's sends
            __sync_synchronize();
            c->sh->cons_seq[q][me] = ++c->rseq[q];
        }
    c->ops.clear();
    return ncclSuccess;
}

}  // namespace

extern "C" {

// Test-side constructor: path = a fresh file name shared by the P processes.
void *shimCommInit(const char *path, int rank, int nranks, long long cap_bytes)
{
    if (nranks < 1 || nranks > MAXR || rank < 0 || rank >= nranks)
        return nullptr;
    int fd = open(path, O_RDWR | O_CREAT, 0600);
    if (fd < 0)
        return nullptr;
    if (ftruncate(fd, sizeof(Shared)) != 0) {
        close(fd);
        return nullptr;
    }
    void *m = mmap(nullptr, sizeof(Shared), PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
    if (m == MAP_FAILED)
        return nullptr;
    Comm *c = new Comm();
    c->rank = rank;
    c->nranks = nranks;
    c->cap = (size_t)cap_bytes;
    c->sh = (Shared *)m;
    if (cudaMalloc(&c->stage, c->cap * nranks) != cudaSuccess)
        return nullptr;
    cudaIpcMemHandle_t hd;
    if (cudaIpcGetMemHandle(&hd, c->stage) != cudaSuccess)
        return nullptr;
    memcpy((void *)&c->sh->stage[rank], &hd, sizeof(hd));
    __sync_synchronize();
    __sync_fetch_and_add(&c->sh->joined, 1);
    while (c->sh->joined < nranks)
        spin();
    __sync_synchronize();
    for (int q = 0; q < nranks; q++) {
        if (q == rank)
            continue;
        cudaIpcMemHandle_t ph;
        memcpy(&ph, (const void *)&c->sh->stage[q], sizeof(ph));
        if (cudaIpcOpenMemHandle((void **)&c->peer_stage[q], ph, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess)
            return nullptr;
    }
    g_last = c;
    return c;
}

ncclResult_t ncclGroupStart()
{
    if (g_last)
        g_last->depth++;
    return ncclSuccess;
}

ncclResult_t ncclGroupEnd()
{
    Comm *c = g_last;
    if (!c || c->depth <= 0)
        return ncclInvalidUsage;
    if (--c->depth > 0)
        return ncclSuccess;
    return flush(c);
}

static size_t tsize(ncclDataType_t t) { return t == ncclDouble ? 8 : (t == ncclFloat || t == ncclInt32) ? 4 : 1; }

ncclResult_t ncclSend(const void *buf, size_t count, ncclDataType_t t, int peer, ncclComm_t comm, cudaStream_t s)
{
    Comm *c = (Comm *)comm;
    if (!c || peer < 0 || peer >= c->nranks || peer == c->rank)
        return ncclInvalidArgument;
    c->ops.push_back({true, const_cast<void *>(buf), count * tsize(t), peer, s});
    return c->depth > 0 ? ncclSuccess : flush(c);
}

ncclResult_t ncclRecv(void *buf, size_t count, ncclDataType_t t, int peer, ncclComm_t comm, cudaStream_t s)
{
    Comm *c = (Comm *)comm;
    if (!c || peer < 0 || peer >= c->nranks || peer == c->rank)
        return ncclInvalidArgument;
    c->ops.push_back({false, buf, count * tsize(t), peer, s});
    return c->depth > 0 ? ncclSuccess : flush(c);
}

ncclResult_t ncclAllReduce(const void *sendbuff, void *recvbuff, size_t count, ncclDataType_t t, ncclRedOp_t op,
                           ncclComm_t comm, cudaStream_t s)
{
    Comm *c = (Comm *)comm;
    if (!c || t != ncclDouble || op != ncclSum || count > 64)
        return ncclInvalidArgument;
    double v[64], out[64];
    if (cudaMemcpyAsync(v, sendbuff, count * 8, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
        return ncclUnhandledCudaError;
    const long long k = ++c->red;
    // every rank must have read the previous reduction's values before mine are overwritten
    for (int q = 0; q < c->nranks; q++)
        while (c->sh->red_seq[q] < 2 * (k - 1))
            spin();
    for (size_t i = 0; i < count; i++)
        c->sh->red_val[c->rank][i] = v[i];
    __sync_synchronize();
    c->sh->red_seq[c->rank] = 2 * k - 1;  // published
    for (int q = 0; q < c->nranks; q++)
        while (c->sh->red_seq[q] < 2 * k - 1)
            spin();
    __sync_synchronize();
    for (size_t i = 0; i < count; i++) {
        double acc = 0.0;
        for (int q = 0; q < c->nranks; q++)  // rank order: deterministic
            acc += c->sh->red_val[q][i];
        out[i] = acc;
    }
    __sync_synchronize();
    c->sh->red_seq[c->rank] = 2 * k;  // read everyone's values
    for (int q = 0; q < c->nranks; q++)
        while (c->sh->red_seq[q] < 2 * k)
            spin();
    if (cudaMemcpyAsync(recvbuff, out, count * 8, cudaMemcpyHostToDevice, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
        return ncclUnhandledCudaError;
    return ncclSuccess;
}

const char *ncclGetErrorString(ncclResult_t r)
{
    switch (r) {
    case ncclSuccess: return "ncclshim: success";
    case ncclUnhandledCudaError: return "ncclshim: CUDA error";
    case ncclInvalidArgument: return "ncclshim: invalid argument";
    case ncclInvalidUsage: return "ncclshim: invalid usage (unmatched send/recv or group)";
    case ncclInternalError: return "ncclshim: staging capacity exceeded";
    default: return "ncclshim: error";
    }
}

}  // extern "C"
