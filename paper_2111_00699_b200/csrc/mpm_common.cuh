// Shared device helpers of the B200 MLS-MPM core (sm_100a).
// Reference paths are relative to /root/reference/pkg/src/mpmbench/.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/mpm_b200.h"

#define MPM_SM_COUNT 148

// particle channels (particles.py:24-31)
#define CH_POS 0
#define CH_VEL 3
#define CH_C 6
#define CH_MASS 15
#define CH_DEF 16
#define CH_PLASTIC 25

#define MPM_EMPTY_KEY ((long long)-1)
#define MPM_HASH_MULT 0x9E3779B97F4A7C15ull
#define MPM_INT_MAX 0x7fffffff

namespace mpm {

// ---- error plumbing ---------------------------------------------------------------
void set_last_error(const char *what, cudaError_t e);
int check_launch(const char *what, int n_kernels);   // also counts the kernels just launched

// ---- Morton coding (grid.py:41-70), 21 bits per axis, x lowest ---------------------
__host__ __device__ __forceinline__ unsigned long long part1by2(unsigned long long x)
{
    x &= 0x1FFFFFull;
    x = (x | (x << 32)) & 0x1F00000000FFFFull;
    x = (x | (x << 16)) & 0x1F0000FF0000FFull;
    x = (x | (x << 8)) & 0x100F00F00F00F00Full;
    x = (x | (x << 4)) & 0x10C30C30C30C30C3ull;
    x = (x | (x << 2)) & 0x1249249249249249ull;
    return x;
}
__host__ __device__ __forceinline__ unsigned long long compact1by2(unsigned long long x)
{
    x &= 0x1249249249249249ull;
    x = (x ^ (x >> 2)) & 0x10C30C30C30C30C3ull;
    x = (x ^ (x >> 4)) & 0x100F00F00F00F00Full;
    x = (x ^ (x >> 8)) & 0x1F0000FF0000FFull;
    x = (x ^ (x >> 16)) & 0x1F00000000FFFFull;
    x = (x ^ (x >> 32)) & 0x1FFFFFull;
    return x;
}
__host__ __device__ __forceinline__ long long encode_cell(long long x, long long y, long long z)
{
    return (long long)(part1by2((unsigned long long)x) | (part1by2((unsigned long long)y) << 1) |
                       (part1by2((unsigned long long)z) << 2));
}

// multiply-shift hash of grid.py:130-133 (arithmetic shift of the wrapped signed product)
__device__ __forceinline__ int hash_slot(long long key, int shift, int mask)
{
    long long prod = (long long)((unsigned long long)key * MPM_HASH_MULT);
    return (int)((prod >> shift) & (long long)mask);
}
__host__ __device__ __forceinline__ int hash_shift_for(int cap)
{
    // grid.py: shift = 64 - log2(cap)
    int bits = 0;
    while ((1 << bits) < cap) ++bits;
    return 64 - bits;
}

// node slot inside a 4^3 block: Morton of the low two bits per axis (pipeline.py:144-147)
__device__ __forceinline__ int node_slot(int cx, int cy, int cz)
{
    return (cx & 1) | ((cy & 1) << 1) | ((cz & 1) << 2) | ((cx & 2) << 2) | ((cy & 2) << 3) |
           ((cz & 2) << 4);
}

// Guard of speculative launches (mpm_guard in the header): the device word holds the first
// step whose gather found a particle outside its free zone (INT_MAX while none).  A kernel
// of step s returns without touching memory when that word is < s, so the host may enqueue
// step s+1 before it has read step s's flag; the kernel that raises the flag (step s itself)
// and the rest of step s still run to completion.
struct DevGuard {
    int *word;
    int step;
    int n_peers;
    int *peer_words[MPM_MAX_PEERS];
};
// raise the guard: this rank's word and, with peer-mapped memory, every peer's (system scope)
// A word that peers update over NVLink (atomicMin_system) is updated with system scope by its
// owner too: atomics of different scopes on one address are not atomic with respect to each other
// (a lost minimum would leave the word above the true first bad step).
__device__ __forceinline__ void guard_raise(const DevGuard &g)
{
    if (!g.word) return;
    if (g.n_peers > 0) {
        atomicMin_system(g.word, g.step);
        for (int p = 0; p < g.n_peers; ++p) atomicMin_system(g.peer_words[p], g.step);
    } else {
        atomicMin(g.word, g.step);
    }
}
__device__ __forceinline__ bool guarded_out(const DevGuard &g)
{
    if (g.word == nullptr) return false;
    int v;
    if (g.n_peers > 0) asm volatile("ld.relaxed.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(g.word) : "memory");
    else v = *((volatile const int *)g.word);
    return v < g.step;
}
inline DevGuard make_guard(const mpm_guard *g)
{
    DevGuard d;
    d.word = g ? g->first_bad_step : nullptr;
    d.step = g ? g->step : 0;
    d.n_peers = g ? g->n_peer_words : 0;
    if (d.n_peers < 0 || d.n_peers > MPM_MAX_PEERS) d.n_peers = 0;
    for (int p = 0; p < MPM_MAX_PEERS; ++p) d.peer_words[p] = (g && p < d.n_peers) ? g->peer_words[p] : nullptr;
    return d;
}

// ---- programmatic dependent launch (sm_90+) -------------------------------------------
// The steady-state step is a chain transfer -> grid update -> transfer -> ... on one stream.  A
// kernel launched with the programmatic-serialization attribute may have its CTAs resident
// while the tail of the previous kernel drains; they block in pdl_wait() until that kernel has
// completed and its writes are visible, so the launch latency between dependent kernels
// (2-4 us each, two per step) is off the critical path.  Every kernel of the chain calls
// pdl_wait() before it touches memory (the guard word included) and pdl_launch_dependents()
// right after it.  Kernels launched the ordinary way are unaffected (full serialisation).
#ifndef MPM_PDL
#define MPM_PDL 1
#endif
__device__ __forceinline__ void pdl_wait()
{
#if MPM_PDL
    asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}
__device__ __forceinline__ void pdl_launch_dependents()
{
#if MPM_PDL
    asm volatile("griddepcontrol.launch_dependents;");
#endif
}
// Set while a kernel chain is being captured into a CUDA graph (mpm_rebuild): the nodes of a graph are
// launched the plain way (a programmatic edge behind a memset / memcpy node is not capturable, and
// inside a graph the launch latency the attribute hides is not there).
extern thread_local bool g_plain_launch;
unsigned long long launch_counter_add(unsigned long long n);

template <typename... KArgs, typename... Args>
inline void launch_chained(void (*kernel)(KArgs...), int grid, int block, cudaStream_t stream, Args &&...args)
{
#if MPM_PDL
    if (g_plain_launch) {
        kernel<<<grid, block, 0, stream>>>(static_cast<KArgs>(args)...);
        return;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3((unsigned)block);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
#else
    kernel<<<grid, block, 0, stream>>>(static_cast<KArgs>(args)...);
#endif
}

// exclusive scan of int32 (three kernels, no library): out may alias in; total (device) optional
// n_dev (optional): the length lives on the device, n = min(n, *n_dev * mul + add); grids are sized by n
void exclusive_scan_i32(const int32_t *in, int32_t *out, int32_t n, int32_t *block_sums,
                        int32_t *total, cudaStream_t stream, const int32_t *n_dev = nullptr, int mul = 1,
                        int add = 0);
// scratch entries needed by exclusive_scan_i32 for n elements
inline int32_t scan_scratch_len(int64_t n) { return (int32_t)((n + 1023) / 1024 + 1); }

}  // namespace mpm
