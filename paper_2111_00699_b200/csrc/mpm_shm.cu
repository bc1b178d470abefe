// Host rendezvous of the ranks of one node over a shared-memory segment.
//
// The reference's workers are threads that meet at a SpinBarrier and read each other's Python
// objects (multiworker.py:27-107).  With one process per GPU, the device-paced pipeline
// (peer.py) needs the host side only on collective steps (frame starts, rebuild steps): a
// barrier and a few integers per rank.  A library collective for that costs a kernel launch, a
// device round trip and a stream sync per call (~100 us each, five to seven per collective
// step); all ranks of a B200 box share a host, so the same exchange is two cache-line writes
// and a sense-reversing barrier in shared memory (~microseconds).
//
// Segment layout (the caller maps it, zero-filled, at least mpm_shm_bytes(n_ranks) long):
//   [0]   int32 arrived, int32 sense           (one 64-byte line)
//   [64 + 128 r]  int32 local_sense of rank r, then MPM_SHM_MAX_VALUES int64 values
#include <sched.h>
#include <time.h>

#include "mpm_common.cuh"

namespace {

struct ShmHeader {
    int32_t arrived;
    int32_t sense;
    int32_t pad[14];
};
struct ShmRank {
    int32_t local_sense;
    int32_t pad;
    int64_t values[MPM_SHM_MAX_VALUES];
};
static_assert(sizeof(ShmHeader) == 64 && sizeof(ShmRank) == 128, "segment layout");

double now_ms()
{
    timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return ts.tv_sec * 1e3 + ts.tv_nsec * 1e-6;
}

// sense-reversing central barrier; returns false on timeout
bool shm_barrier(ShmHeader *h, ShmRank *me, int n_ranks, int timeout_ms)
{
    const int32_t my = !me->local_sense;
    me->local_sense = my;
    if (__atomic_add_fetch(&h->arrived, 1, __ATOMIC_SEQ_CST) == n_ranks) {
        __atomic_store_n(&h->arrived, 0, __ATOMIC_SEQ_CST);
        __atomic_store_n(&h->sense, my, __ATOMIC_SEQ_CST);
        return true;
    }
    const double t0 = now_ms();
    for (unsigned spin = 0; __atomic_load_n(&h->sense, __ATOMIC_SEQ_CST) != my; ++spin) {
        if ((spin & 1023) == 1023) {
            if (now_ms() - t0 > timeout_ms) return false;
            sched_yield();
        }
    }
    return true;
}

}  // namespace

extern "C" {

int64_t mpm_shm_bytes(int32_t n_ranks) { return (int64_t)sizeof(ShmHeader) + (int64_t)sizeof(ShmRank) * n_ranks; }

int mpm_shm_allgather_i64(void *base, int32_t n_ranks, int32_t rank, const int64_t *values, int32_t n_values,
                          int64_t *out, int32_t timeout_ms)
{
    if (!base || n_ranks < 1 || rank < 0 || rank >= n_ranks || n_values < 0 || n_values > MPM_SHM_MAX_VALUES ||
        (n_values && (!values || !out)))
        return MPM_ERR_REJECTED_INPUT;
    ShmHeader *h = (ShmHeader *)base;
    ShmRank *ranks = (ShmRank *)((char *)base + sizeof(ShmHeader));
    ShmRank *me = ranks + rank;
    for (int k = 0; k < n_values; ++k) me->values[k] = values[k];
    if (!shm_barrier(h, me, n_ranks, timeout_ms)) return MPM_ERR_BARRIER_TIMEOUT;   // every slot written
    for (int q = 0; q < n_ranks; ++q)
        for (int k = 0; k < n_values; ++k) out[(size_t)q * n_values + k] = ranks[q].values[k];
    if (!shm_barrier(h, me, n_ranks, timeout_ms)) return MPM_ERR_BARRIER_TIMEOUT;   // every slot read
    return MPM_OK;
}

}  // extern "C"
