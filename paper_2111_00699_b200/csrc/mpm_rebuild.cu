// Rebuild-mapping on the device: particle codes, block hash with first-occurrence
// numbering, 27-dilation, stable counting sort, lane-group packing.
//
// The reference builds these structures with SEQUENTIAL loops whose visiting order defines
// the result (grid.py:136-157, 282-322; particles.py:66-80, 152-173).  The kernels here
// are parallel but reproduce that order exactly:
//   * "index = order of first occurrence" is computed as
//         atomicMin(first[slot], sequence number)  ->  flag(sequence number == first)
//         ->  exclusive scan of the flags  ->  index = scan[first]
//   * the counting sort takes unordered tickets inside a (block, cell) bin and then ranks
//     the members of each bin by input index, which is what a stable sort would produce.
// Reference paths are relative to /root/reference/pkg/src/mpmbench/.
#include "mpm_common.cuh"

namespace mpm {

// ===================================================================================
// exclusive scan (int32): reduce / scan block sums / apply
// ===================================================================================
constexpr int SCAN_THREADS = 256;
constexpr int SCAN_ITEMS = 4;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;

__device__ __forceinline__ int warp_inclusive_scan(int v, int lane)
{
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        int t = __shfl_up_sync(0xffffffffu, v, d);
        if (lane >= d) v += t;
    }
    return v;
}

// exclusive scan of one value per thread across the CTA; returns the exclusive prefix, *total = CTA sum
__device__ __forceinline__ int block_exclusive_scan(int v, int *total)
{
    __shared__ int warp_sums[33];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nwarps = (blockDim.x + 31) >> 5;
    const int inc = warp_inclusive_scan(v, lane);
    if (lane == 31) warp_sums[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        const int w = lane < nwarps ? warp_sums[lane] : 0;
        const int winc = warp_inclusive_scan(w, lane);
        warp_sums[lane] = winc - w;
        if (lane == 31) warp_sums[32] = winc;
    }
    __syncthreads();
    const int excl = warp_sums[warp] + inc - v;
    *total = warp_sums[32];
    __syncthreads();   // warp_sums is reused by the next call
    return excl;
}

// Length of a scan whose size lives on the device: n = min(bound, *n_dev * mul + add) (n_dev NULL:
// the bound itself).  Grids are sized from the bound, which the host knows; the rebuild never waits
// for a count in the middle of its kernel chain.
struct ScanLen {
    const int *n_dev;
    int mul, add, bound;
};
__device__ __forceinline__ int scan_len(const ScanLen &L)
{
    if (!L.n_dev) return L.bound;
    const long long n = (long long)(*L.n_dev) * L.mul + L.add;
    return (int)(n < (long long)L.bound ? (n < 0 ? 0 : n) : L.bound);
}

__global__ void __launch_bounds__(SCAN_THREADS) scan_reduce_kernel(const int *in, ScanLen L, int *block_sums)
{
    pdl_wait();
    pdl_launch_dependents();
    const int n = scan_len(L);
    const int base = blockIdx.x * SCAN_TILE + threadIdx.x * SCAN_ITEMS;
    int s = 0;
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; ++k)
        if (base + k < n) s += in[base + k];
    int total;
    block_exclusive_scan(s, &total);
    if (threadIdx.x == 0) block_sums[blockIdx.x] = total;
}

__global__ void __launch_bounds__(1024) scan_blocksums_kernel(int *block_sums, int nb, int *total_out)
{
    pdl_wait();
    pdl_launch_dependents();
    __shared__ int carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int start = 0; start < nb; start += 1024) {
        int i = start + threadIdx.x;
        int v = i < nb ? block_sums[i] : 0;
        int total;
        int excl = block_exclusive_scan(v, &total);
        int c = carry;
        if (i < nb) block_sums[i] = excl + c;
        __syncthreads();
        if (threadIdx.x == 0) carry = c + total;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        block_sums[nb] = carry;
        if (total_out) *total_out = carry;
    }
}

__global__ void __launch_bounds__(SCAN_THREADS) scan_apply_kernel(const int *in, int *out, ScanLen L,
                                                                  const int *block_sums)
{
    pdl_wait();
    pdl_launch_dependents();
    const int n = scan_len(L);
    const int base = blockIdx.x * SCAN_TILE + threadIdx.x * SCAN_ITEMS;
    int v[SCAN_ITEMS];
    int s = 0;
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; ++k) {
        v[k] = (base + k < n) ? in[base + k] : 0;
        s += v[k];
    }
    int total;
    int excl = block_exclusive_scan(s, &total) + block_sums[blockIdx.x];
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; ++k) {
        if (base + k < n) out[base + k] = excl;
        excl += v[k];
    }
}

void exclusive_scan_i32(const int32_t *in, int32_t *out, int32_t n, int32_t *block_sums,
                        int32_t *total, cudaStream_t stream, const int32_t *n_dev, int mul, int add)
{
    if (n <= 0) {
        if (total) cudaMemsetAsync(total, 0, sizeof(int32_t), stream);
        return;
    }
    const ScanLen L = {n_dev, mul, add, n};
    const int nb = (n + SCAN_TILE - 1) / SCAN_TILE;
    launch_chained(scan_reduce_kernel, nb, SCAN_THREADS, stream, in, L, block_sums);
    launch_chained(scan_blocksums_kernel, 1, 1024, stream, block_sums, nb, total);
    launch_chained(scan_apply_kernel, nb, SCAN_THREADS, stream, in, out, L, block_sums);
}

// ===================================================================================
// live-lane compaction (particles.py:177-188, 336-358)
// ===================================================================================
__global__ void __launch_bounds__(256) live_count_kernel(const uint16_t *__restrict__ lane_meta,
                                                         const int *__restrict__ group_len,
                                                         int n_groups, const int *__restrict__ n_groups_dev,
                                                         int drop_q, int *__restrict__ group_live)
{
    pdl_wait();
    pdl_launch_dependents();
    const int g = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (g >= n_groups) return;
    // the count on the device (n_groups is then the launch bound): groups beyond it hold nothing
    const int len = (n_groups_dev && g >= *n_groups_dev) ? 0 : group_len[g];
    bool live = lane < len;
    if (live && drop_q) live = !(lane_meta[g * 32 + lane] & MPM_LANE_QUARANTINED);
    unsigned m = __ballot_sync(0xffffffffu, live);
    if (lane == 0) group_live[g] = __popc(m);
}

__global__ void __launch_bounds__(256) live_write_kernel(const uint16_t *__restrict__ lane_meta,
                                                         const int *__restrict__ group_len,
                                                         int n_groups, const int *__restrict__ n_groups_dev,
                                                         int drop_q, const int *__restrict__ group_base,
                                                         int *__restrict__ src_slot)
{
    pdl_wait();
    pdl_launch_dependents();
    const int g = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (g >= n_groups) return;
    const int len = (n_groups_dev && g >= *n_groups_dev) ? 0 : group_len[g];
    bool live = lane < len;
    if (live && drop_q) live = !(lane_meta[g * 32 + lane] & MPM_LANE_QUARANTINED);
    unsigned m = __ballot_sync(0xffffffffu, live);
    if (live) src_slot[group_base[g] + __popc(m & ((1u << lane) - 1u))] = g * 32 + lane;
}

// ===================================================================================
// particle codes (particles.py:52-58, grid.py:92-107): float64, DIVISION by dx
// ===================================================================================
__device__ __forceinline__ float load_channel(const float *__restrict__ data, int nch, int slot, int ch)
{
    return data[((size_t)(slot >> 5) * nch + ch) * 32 + (slot & 31)];
}

__global__ void __launch_bounds__(256) particle_codes_kernel(
    const float *__restrict__ data, int nch, const int *__restrict__ src_slot,
    const int *__restrict__ n_live_dev, const float *__restrict__ staged, int n_staged, int n_upper,
    double dx, long long *__restrict__ codes, int *__restrict__ bad_index)
{
    pdl_wait();
    pdl_launch_dependents();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int n_live = n_live_dev ? *n_live_dev : 0;
    const int n = n_live + n_staged;
    if (i >= n_upper) return;
    if (i >= n) { codes[i] = 0; return; }
    float p[3];
    if (i < n_live) {
        const int slot = src_slot[i];
#pragma unroll
        for (int a = 0; a < 3; ++a) p[a] = load_channel(data, nch, slot, CH_POS + a);
    } else {
        const float *s = staged + (size_t)(i - n_live) * nch;
#pragma unroll
        for (int a = 0; a < 3; ++a) p[a] = s[CH_POS + a];
    }
    long long c[3];
    bool bad = false;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        double q = __dsub_rn(__ddiv_rn((double)p[a], dx), 0.5);
        double fl = floor(q);
        // non-finite positions fall outside the encodable range like any other stray particle
        long long cell = (fl >= -4.0e18 && fl <= 4.0e18) ? (long long)fl + MPM_CELL_BIAS : -1;
        if (cell < 0 || cell >= (1 << 21)) { bad = true; cell = 0; }
        c[a] = cell;
    }
    if (bad) atomicMin(bad_index, i);
    codes[i] = encode_cell(c[0], c[1], c[2]);
}

// ===================================================================================
// hash insert in first-occurrence order (grid.py:136-157)
// ===================================================================================
__global__ void hash_clear_kernel(long long *hkeys, int *hvals, int *hfirst, int cap)
{
    pdl_wait();
    pdl_launch_dependents();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < cap) {
        hkeys[i] = MPM_EMPTY_KEY;
        hvals[i] = -1;
        hfirst[i] = MPM_INT_MAX;
    }
}

// returns the slot of `code` after inserting it if absent, or -1 on overflow
__device__ __forceinline__ int hash_insert(long long *hkeys, int shift, int mask, long long code)
{
    int slot = hash_slot(code, shift, mask);
    for (int probes = 0; probes <= mask; ++probes) {
        long long prev = hkeys[slot];
        if (prev == code) return slot;
        if (prev == MPM_EMPTY_KEY) {
            prev = (long long)atomicCAS((unsigned long long *)&hkeys[slot],
                                        (unsigned long long)MPM_EMPTY_KEY, (unsigned long long)code);
            if (prev == MPM_EMPTY_KEY || prev == code) return slot;
        }
        slot = (slot + 1) & mask;
    }
    return -1;
}

__device__ __forceinline__ int hash_find(const long long *hkeys, int shift, int mask, long long code)
{
    int slot = hash_slot(code, shift, mask);
    for (int probes = 0; probes <= mask; ++probes) {
        long long k = hkeys[slot];
        if (k == code) return slot;
        if (k == MPM_EMPTY_KEY) return -1;
        slot = (slot + 1) & mask;
    }
    return -1;
}

__global__ void __launch_bounds__(256) block_insert_kernel(const long long *__restrict__ codes,
                                                           const int *__restrict__ n_dev, int n_upper,
                                                           long long *hkeys, int *hfirst, int shift,
                                                           int mask, int *__restrict__ pslot,
                                                           int *overflow)
{
    pdl_wait();
    pdl_launch_dependents();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_upper) return;
    if (i >= *n_dev) { pslot[i] = -1; return; }
    const long long bcode = codes[i] >> 6;
    const int slot = hash_insert(hkeys, shift, mask, bcode);
    pslot[i] = slot;
    if (slot < 0) { *overflow = 1; return; }
    atomicMin(&hfirst[slot], i);
}

__global__ void __launch_bounds__(256) first_flag_kernel(const int *__restrict__ pslot,
                                                         const int *__restrict__ hfirst,
                                                         const int *__restrict__ hvals, int n_upper,
                                                         const int *__restrict__ n_dev, int n_mul,
                                                         int only_unassigned, int *__restrict__ flag)
{
    pdl_wait();
    pdl_launch_dependents();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_upper) return;
    if (n_dev && i >= *n_dev * n_mul) { flag[i] = 0; return; }   // beyond the live entries: pslot is stale
    const int slot = pslot[i];
    int f = 0;
    if (slot >= 0 && hfirst[slot] == i && (!only_unassigned || hvals[slot] < 0)) f = 1;
    flag[i] = f;
}

__global__ void __launch_bounds__(256) block_assign_kernel(const long long *__restrict__ codes,
                                                           const int *__restrict__ pslot,
                                                           const int *__restrict__ hfirst,
                                                           const int *__restrict__ rank, int n_upper,
                                                           int *hvals, long long *__restrict__ gcodes)
{
    pdl_wait();
    pdl_launch_dependents();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_upper) return;
    const int slot = pslot[i];
    if (slot >= 0 && hfirst[slot] == i) {
        const int r = rank[i];
        hvals[slot] = r;
        gcodes[r] = codes[i] >> 6;
    }
}

__global__ void __launch_bounds__(256) gidx_kernel(const int *__restrict__ pslot,
                                                   const int *__restrict__ hvals, int n_upper,
                                                   int *__restrict__ gidx)
{
    pdl_wait();
    pdl_launch_dependents();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_upper) return;
    const int slot = pslot[i];
    gidx[i] = slot >= 0 ? hvals[slot] : -1;
}

// ===================================================================================
// 27-dilation (grid.py:282-322)
// ===================================================================================
__global__ void __launch_bounds__(256) dilate_insert_kernel(const long long *__restrict__ gcodes,
                                                            const int *__restrict__ n_g_dev, long long *hkeys,
                                                            const int *__restrict__ hvals, int *hfirst,
                                                            int shift, int mask, int *__restrict__ qslot,
                                                            int *bad_block, int *overflow)
{
    pdl_wait();
    pdl_launch_dependents();
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    const int n_g = *n_g_dev;
    if (q >= n_g * 27) return;
    const int g = q / 27, s = q - g * 27;
    const int dz = s / 9 - 1, dy = (s / 3) % 3 - 1, dxx = s % 3 - 1;
    const unsigned long long code = (unsigned long long)gcodes[g];
    const long long nx = (long long)compact1by2(code) + dxx;
    const long long ny = (long long)compact1by2(code >> 1) + dy;
    const long long nz = (long long)compact1by2(code >> 2) + dz;
    if (nx < 0 || ny < 0 || nz < 0 || nx >= (1 << 19) || ny >= (1 << 19) || nz >= (1 << 19)) {
        atomicMin(bad_block, g);
        qslot[q] = -1;
        return;
    }
    const long long ncode = encode_cell(nx, ny, nz);
    const int slot = hash_insert(hkeys, shift, mask, ncode);
    qslot[q] = slot;
    if (slot < 0) { *overflow = 1; return; }
    if (hvals[slot] < 0) atomicMin(&hfirst[slot], q);   // gblock slots keep their index
}

// also copies the gblock codes to the head of the table (grid.py:362-371: gblocks occupy [0, n_g))
__global__ void __launch_bounds__(256) dilate_assign_kernel(const int *__restrict__ qslot,
                                                            const int *__restrict__ flag,
                                                            const int *__restrict__ rank,
                                                            const int *__restrict__ n_g_dev, int pblock_cap,
                                                            const long long *__restrict__ hkeys,
                                                            const long long *__restrict__ gcodes,
                                                            int *hvals, long long *__restrict__ codes,
                                                            int *overflow)
{
    pdl_wait();
    pdl_launch_dependents();
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    const int n_g = *n_g_dev;
    if (q < n_g && q < pblock_cap) codes[q] = gcodes[q];
    if (q >= n_g * 27) return;
    if (!flag[q]) return;
    const int slot = qslot[q];
    const int idx = n_g + rank[q];
    if (idx >= pblock_cap) { *overflow = 2; return; }
    hvals[slot] = idx;
    codes[idx] = hkeys[slot];
}

__global__ void __launch_bounds__(256) dilate_link_kernel(const int *__restrict__ qslot,
                                                          const int *__restrict__ hvals,
                                                          const int *__restrict__ n_g_dev,
                                                          int *__restrict__ neighbor)
{
    pdl_wait();
    pdl_launch_dependents();
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= *n_g_dev * 27) return;
    const int slot = qslot[q];
    neighbor[q] = slot >= 0 ? hvals[slot] : -1;
}

__global__ void __launch_bounds__(256) block_origin_kernel(const long long *__restrict__ codes,
                                                           const int *__restrict__ count_dev,
                                                           int pblock_cap, int4 *__restrict__ origin)
{
    pdl_wait();
    pdl_launch_dependents();
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= pblock_cap || b >= *count_dev) return;
    const unsigned long long code = (unsigned long long)codes[b];
    origin[b] = make_int4(4 * (int)compact1by2(code), 4 * (int)compact1by2(code >> 1),
                          4 * (int)compact1by2(code >> 2), 0);
}

// Scalars of one rebuild (device words S[16], mpm_rebuild): 0 n_live, 1 n_total, 2 bad particle,
// 3 n_gblocks, 4 hash overflow, 5 pblock count, 6 bad block, 7 n_groups, 8 abort mask,
// 9..12 the counts an aborted rebuild needs room for (gblocks, table entries, groups, nodes).
__global__ void rebuild_init_kernel(int *S, int *large_list, int *guard_word)
{
    pdl_wait();
    pdl_launch_dependents();
    const int i = threadIdx.x;
    if (i < 16) S[i] = (i == 2 || i == 6) ? MPM_INT_MAX : 0;
    if (i == 16 && large_list) large_list[0] = 0;
    if (i == 17 && guard_word) *guard_word = MPM_INT_MAX;
}

// A count that outgrew the caller's buffers (or a particle / block outside the domain) aborts the
// rebuild WITHOUT a host round trip: the counts the later kernels read are zeroed, so every one of
// them -- and the rest of the rebuild step issued behind them -- is a no-op, and the guard of the
// steps enqueued behind the rebuild is lowered below every step (-1: the chain does not depend on the
// step number, so it can be replayed as a CUDA graph).  The host finds the abort mask
// and the sizes needed when it reads the scalars (mpm_rebuild_wait), grows the buffers and calls again.
__device__ __forceinline__ void rebuild_abort(int *S, int why, int *guard_word, int guard_step)
{
    (void)guard_step;
    S[8] |= why;
    S[1] = 0; S[3] = 0; S[5] = 0; S[7] = 0;
    if (guard_word) atomicMin(guard_word, -1);
}
__global__ void rebuild_check_blocks_kernel(int *S, int gblocks_bound, int hash_cap, int table_cap,
                                            int *guard_word, int guard_step)
{
    pdl_wait();
    pdl_launch_dependents();
    const int n_g = S[3];
    int why = 0;
    if (S[2] != MPM_INT_MAX) why |= 8;                                   // particle outside the domain
    if (S[4] || 8ll * n_g > hash_cap) why |= 1;                          // hash table too small
    if (n_g > gblocks_bound) { why |= 2; S[9] = n_g; }
    if (27ll * n_g > table_cap) { why |= 2; S[10] = 27 * n_g; }          // worst case of the dilation
    if (why) rebuild_abort(S, why, guard_word, guard_step);
}
__global__ void rebuild_check_groups_kernel(int *S, int groups_cap, int nodes_cap, int *guard_word, int guard_step,
                                            int *n_groups_out)
{
    pdl_wait();
    pdl_launch_dependents();
    // the new store's group count, kept on the device for the NEXT rebuild (it is then the old store)
    if (n_groups_out) *n_groups_out = (S[8] || S[7] > groups_cap) ? 0 : S[7];
    if (S[8]) return;
    int why = 0;
    if (S[6] != MPM_INT_MAX) why |= 16;                                  // block on the domain boundary
    if (S[4] == 1) why |= 1;                                             // the halo did not fit the hash table
    if (S[7] > groups_cap) { why |= 4; S[11] = S[7]; }
    if (S[5] > nodes_cap) { why |= 4; S[12] = S[5]; }
    if (why) {
        const int count = S[5], n_groups = S[7], n_g = S[3], n = S[1];
        rebuild_abort(S, why, guard_word, guard_step);
        S[13] = n; S[14] = n_g; S[15] = count; (void)n_groups;
    }
}

// zero the first *count rows (64 float4 nodes each) of a nodal buffer: the reset of vel at a rebuild
__global__ void __launch_bounds__(256) zero_rows_kernel(float4 *rows, const int *__restrict__ count_dev, int bound)
{
    pdl_wait();
    pdl_launch_dependents();
    const int b = blockIdx.x * 4 + (threadIdx.x >> 6);
    if (b >= bound || b >= *count_dev) return;
    rows[(size_t)b * 64 + (threadIdx.x & 63)] = make_float4(0.f, 0.f, 0.f, 0.f);
}

__global__ void add_dev_kernel(int *dst, const int *a, const int *b)
{
    pdl_wait();
    pdl_launch_dependents();
    *dst = *a + *b;
}

__global__ void add_scalar_kernel(int *dst, const int *a, int b)
{
    pdl_wait();
    pdl_launch_dependents();
    *dst = *a + b;
}

// ===================================================================================
// stable counting sort + lane groups (particles.py:66-80, 152-173)
// ===================================================================================
__global__ void __launch_bounds__(256) hist_kernel(const long long *__restrict__ codes,
                                                   const int *__restrict__ gidx,
                                                   const int *__restrict__ n_dev, int n_upper,
                                                   int *bins, int *__restrict__ ticket)
{
    pdl_wait();
    pdl_launch_dependents();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_upper || i >= *n_dev) return;
    const int key = (gidx[i] << 6) | (int)(codes[i] & 63);
    ticket[i] = atomicAdd(&bins[key], 1);
}

__global__ void __launch_bounds__(256) place_kernel(const long long *__restrict__ codes,
                                                    const int *__restrict__ gidx,
                                                    const int *__restrict__ n_dev, int n_upper,
                                                    const int *__restrict__ bin_start,
                                                    const int *__restrict__ ticket,
                                                    int *__restrict__ tmp_perm)
{
    pdl_wait();
    pdl_launch_dependents();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_upper || i >= *n_dev) return;
    const int key = (gidx[i] << 6) | (int)(codes[i] & 63);
    tmp_perm[bin_start[key] + ticket[i]] = i;
}

// rank the members of each bin by input index: the order a stable sort yields.  A bin holds the
// particles of one cell (8-27 normally): every member counts the members with a smaller index.
// That loop is quadratic in the bin size, so bins above MPM_LARGE_BIN members (particles piled
// into one cell) are only listed here and ranked by large_bin_rank_kernel, whose
// cost is linear in the bin size.
#ifndef MPM_LARGE_BIN
#define MPM_LARGE_BIN 1024
#endif
__global__ void __launch_bounds__(256) stable_rank_kernel(const long long *__restrict__ codes,
                                                          const int *__restrict__ gidx,
                                                          const int *__restrict__ n_dev, int n_upper,
                                                          const int *__restrict__ bin_start,
                                                          const int *__restrict__ tmp_perm,
                                                          int *__restrict__ perm, int *large_list)
{
    pdl_wait();
    pdl_launch_dependents();
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n_upper || j >= *n_dev) return;
    const int i = tmp_perm[j];
    const int key = (gidx[i] << 6) | (int)(codes[i] & 63);
    const int s = bin_start[key], e = bin_start[key + 1];
    if (e - s > MPM_LARGE_BIN) {
        // large_list[0] = number of large bins, then their keys (at most n / MPM_LARGE_BIN of them)
        if (j == s) large_list[1 + atomicAdd(&large_list[0], 1)] = key;
        return;
    }
    int rank = 0;
    for (int t = s; t < e; ++t) rank += tmp_perm[t] < i;
    perm[s + rank] = i;
}

// Stable order of a LARGE bin without comparing its members with each other: the members are a
// subset of the input indices [0, n), so their sorted order is the order of the set bits of a
// bitmap over the input.  One CTA per large bin: clear n/32 words, set one bit per member,
// exclusive scan of the word popcounts, emit.  O(n/32 + members) per large bin, and there are at
// most n / MPM_LARGE_BIN such bins.  `scratch` holds 2 * words per CTA (bitmap, prefix).
constexpr int LARGE_BIN_CTAS = 8;
__global__ void __launch_bounds__(1024) large_bin_rank_kernel(const int *__restrict__ bin_start,
                                                              const int *__restrict__ tmp_perm,
                                                              int *__restrict__ perm,
                                                              const int *__restrict__ large_list,
                                                              unsigned *scratch, int words)
{
    pdl_wait();
    pdl_launch_dependents();
    const int n_large = large_list[0];
    if (n_large == 0) return;
    __shared__ int carry;
    unsigned *bits = scratch + (size_t)blockIdx.x * 2 * words;
    int *pre = (int *)(bits + words);
    const int tid = threadIdx.x;
    for (int k = blockIdx.x; k < n_large; k += gridDim.x) {
        const int key = large_list[1 + k];
        const int s = bin_start[key], e = bin_start[key + 1];
        for (int w = tid; w < words; w += 1024) bits[w] = 0u;
        if (tid == 0) carry = 0;
        __syncthreads();
        for (int t = s + tid; t < e; t += 1024) {
            const int i = tmp_perm[t];
            atomicOr(&bits[i >> 5], 1u << (i & 31));
        }
        __syncthreads();
        for (int base = 0; base < words; base += 1024) {
            const int w = base + tid;
            const int v = w < words ? __popc(bits[w]) : 0;
            int total;
            const int excl = block_exclusive_scan(v, &total);
            const int c = carry;
            if (w < words) pre[w] = excl + c;
            __syncthreads();
            if (tid == 0) carry = c + total;
            __syncthreads();
        }
        for (int w = tid; w < words; w += 1024) {
            unsigned m = bits[w];
            int r = s + pre[w];
            while (m) {
                perm[r++] = w * 32 + (__ffs(m) - 1);
                m &= m - 1;
            }
        }
        __syncthreads();
    }
}

__global__ void __launch_bounds__(256) block_groups_kernel(const int *__restrict__ bin_start,
                                                           const int *__restrict__ n_g_dev,
                                                           int *__restrict__ ngroups)
{
    pdl_wait();
    pdl_launch_dependents();
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    const int n_g = *n_g_dev;
    if (b == n_g) ngroups[b] = 0;      // n_g + 1 entries so that the scan leaves ngroups[n_g] = n_groups
    if (b >= n_g) return;
    const int c = bin_start[(b + 1) * 64] - bin_start[b * 64];
    ngroups[b] = (c + 31) >> 5;
}

// ===================================================================================
// scatter into the new AoSoA store (particles.py:192-199, 235-261, 453)
// ===================================================================================
__device__ __forceinline__ int clamp09(long long v) { return v < 0 ? 0 : (v > 9 ? 9 : (int)v); }

// NCH is a template parameter so that the channel loop unrolls: the NCH loads of a lane (one per
// 128-byte channel row of its source group) are all in flight before the first store, instead of
// one dependent load-store pair at a time (the kernel is latency-bound, not DRAM-bound: its DRAM
// traffic is already the algorithmic 2 x NCH x 4 bytes per particle).
template <int NCH>
__global__ void __launch_bounds__(256) scatter_sorted_kernel(
    const float *__restrict__ old_data, const long long *__restrict__ old_ids,
    const int *__restrict__ src_slot, const int *__restrict__ n_live_dev,
    const float *__restrict__ staged, const long long *__restrict__ staged_ids,
    const int *__restrict__ perm, const int *__restrict__ bin_start,
    const int *__restrict__ block_group_first, const int *__restrict__ n_g_dev,
    const int4 *__restrict__ table_origin,
    double inv_dx, float *__restrict__ new_data, long long *__restrict__ new_ids,
    uint16_t *__restrict__ new_meta, int *__restrict__ group_len, int *__restrict__ group_block,
    int *__restrict__ group_start, const int *__restrict__ n_groups_dev, int n_groups_bound)
{
    pdl_wait();
    pdl_launch_dependents();
    const int g = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (g >= n_groups_bound || g >= *n_groups_dev) return;
    const int n_g = *n_g_dev;
    // block of this group: last b with block_group_first[b] <= g
    int lo = 0, hi = n_g;   // invariant: bgf[lo] <= g < bgf[hi]
    while (hi - lo > 1) {
        int mid = (lo + hi) >> 1;
        if (block_group_first[mid] <= g) lo = mid; else hi = mid;
    }
    const int b = lo;
    const int bstart = bin_start[b * 64], bend = bin_start[(b + 1) * 64];
    const int first = bstart + (g - block_group_first[b]) * 32;
    const int len = min(32, bend - first);
    if (lane == 0) {
        group_len[g] = len;
        group_block[g] = b;
        group_start[g] = first;
    }
    float *dst = new_data + (size_t)g * NCH * 32 + lane;
    float v[NCH];
    long long id = 0;
    uint16_t key = 0;
    if (lane >= len) {
#pragma unroll
        for (int c = 0; c < NCH; ++c) v[c] = 0.0f;
    } else {
        const int i = perm[first + lane];
        const int n_live = n_live_dev ? *n_live_dev : 0;
        if (i < n_live) {
            const int slot = src_slot[i];
            const float *src = old_data + (size_t)(slot >> 5) * NCH * 32 + (slot & 31);
#pragma unroll
            for (int c = 0; c < NCH; ++c) v[c] = src[c * 32];
            id = old_ids[slot];
        } else {
            const float *src = staged + (size_t)(i - n_live) * NCH;
#pragma unroll
            for (int c = 0; c < NCH; ++c) v[c] = src[c];
            id = staged_ids[i - n_live];
        }
        // lane key: float64 floor(p * inv_dx - 0.5) + bias - (origin - 4), clamped (particles.py:235-261)
        const int4 org = table_origin[b];
        const int kx = clamp09((long long)floor(__dsub_rn(__dmul_rn((double)v[CH_POS + 0], inv_dx), 0.5)) + MPM_CELL_BIAS - (org.x - 4));
        const int ky = clamp09((long long)floor(__dsub_rn(__dmul_rn((double)v[CH_POS + 1], inv_dx), 0.5)) + MPM_CELL_BIAS - (org.y - 4));
        const int kz = clamp09((long long)floor(__dsub_rn(__dmul_rn((double)v[CH_POS + 2], inv_dx), 0.5)) + MPM_CELL_BIAS - (org.z - 4));
        key = (uint16_t)(kx + 10 * (ky + 10 * kz));
    }
#pragma unroll
    for (int c = 0; c < NCH; ++c) dst[c * 32] = v[c];
    new_ids[g * 32 + lane] = id;
    new_meta[g * 32 + lane] = key;
}

// ===================================================================================
// readback helpers
// ===================================================================================
// flat[group_start + lane][nch]: the rows of one group are contiguous in the output, so the warp
// transposes its [nch][32] tile through shared memory and writes len * nch consecutive floats.
#define MPM_MAX_NCH 26
__global__ void __launch_bounds__(256) gather_state_kernel(const float *__restrict__ data,
                                                           const long long *__restrict__ ids, int nch,
                                                           const int *__restrict__ group_len,
                                                           const int *__restrict__ group_start,
                                                           int n_groups, float *__restrict__ flat,
                                                           long long *__restrict__ out_ids)
{
    pdl_wait();
    pdl_launch_dependents();
    __shared__ float tile[8][32 * MPM_MAX_NCH];
    const int g = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (g >= n_groups) return;
    const int len = group_len[g];
    const size_t j0 = (size_t)group_start[g];
    const float *src = data + (size_t)g * nch * 32 + lane;
    for (int c = 0; c < nch; ++c) tile[warp][lane * nch + c] = src[c * 32];
    __syncwarp();
    float *dst = flat + j0 * nch;
    for (int k = lane; k < len * nch; k += 32) dst[k] = tile[warp][k];
    if (lane < len) out_ids[j0 + lane] = ids[g * 32 + lane];
}

__global__ void __launch_bounds__(256) gather_positions_kernel(const float *__restrict__ data,
                                                               const long long *__restrict__ ids, int nch,
                                                               const int *__restrict__ group_len,
                                                               const int *__restrict__ group_start,
                                                               int n_groups, float *__restrict__ pos,
                                                               long long *__restrict__ out_ids)
{
    pdl_wait();
    pdl_launch_dependents();
    const int g = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (g >= n_groups || lane >= group_len[g]) return;
    const size_t j = (size_t)group_start[g] + lane;
    const float *src = data + (size_t)g * nch * 32 + lane;
    pos[j * 3 + 0] = src[(CH_POS + 0) * 32];
    pos[j * 3 + 1] = src[(CH_POS + 1) * 32];
    pos[j * 3 + 2] = src[(CH_POS + 2) * 32];
    out_ids[j] = ids[g * 32 + lane];
}

__global__ void __launch_bounds__(256) tag_shared_kernel(const long long *__restrict__ peer_codes,
                                                         int n_peer, const long long *__restrict__ hkeys,
                                                         const int *__restrict__ hvals, int shift,
                                                         int mask, int *__restrict__ peer_map)
{
    pdl_wait();
    pdl_launch_dependents();
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= n_peer) return;
    const int slot = hash_find(hkeys, shift, mask, peer_codes[q]);
    if (slot >= 0 && hvals[slot] >= 0) peer_map[hvals[slot]] = q;
}

__global__ void fill_i32_kernel(int *p, int n, int v)
{
    pdl_wait();
    pdl_launch_dependents();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}

// One 128-byte context line per lane group (mpm_store_view.group_ctx): the neighbour row of the
// group's block as node indices, the block origin, the group length and the block index.
__global__ void __launch_bounds__(256) group_ctx_kernel(const int *__restrict__ group_len,
                                                        const int *__restrict__ group_block, int n_groups,
                                                        const int *__restrict__ n_groups_dev,
                                                        const int4 *__restrict__ origin,
                                                        const int *__restrict__ neighbor,
                                                        int *__restrict__ ctx)
{
    pdl_wait();
    pdl_launch_dependents();
    const int g = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (g >= n_groups || (n_groups_dev && g >= *n_groups_dev)) return;
    const int b = group_block[g];
    int v;
    if (lane < 27) v = neighbor[b * 27 + lane] * 64;
    else if (lane == 27) v = origin[b].x;
    else if (lane == 28) v = origin[b].y;
    else if (lane == 29) v = origin[b].z;
    else if (lane == 30) v = group_len[g];
    else v = b;
    ctx[g * 32 + lane] = v;
}

}  // namespace mpm

using namespace mpm;

static inline int nblk(int64_t n, int t) { return (int)((n + t - 1) / t); }

// Flat channel rows [n][nch] of staged particles from compact x, v, m (ParticleStore.stage_append
// defaults, particles.py:309-334): F = I (J = 1 for the fluid), C = 0, plastic scalar at rest.
// One thread per (particle, channel): coalesced stores of the 100-byte rows.
__global__ void __launch_bounds__(256) stage_particles_kernel(const float *__restrict__ pos,
                                                              const float *__restrict__ vel,
                                                              const float *__restrict__ mass, float mass_scalar,
                                                              long long n_elems, int nch, int mat_kind,
                                                              float *__restrict__ flat)
{
    pdl_wait();
    pdl_launch_dependents();
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n_elems) return;
    const long long i = e / nch;
    const int c = (int)(e - i * nch);
    float v = 0.0f;
    if (c < CH_VEL) v = pos[i * 3 + c];
    else if (c < CH_C) v = vel[i * 3 + (c - CH_VEL)];
    else if (c == CH_MASS) v = mass ? mass[i] : mass_scalar;
    else if (c == CH_DEF) v = 1.0f;
    else if (mat_kind != MPM_MAT_FLUID && (c == CH_DEF + 4 || c == CH_DEF + 8)) v = 1.0f;
    else if (c == CH_PLASTIC && mat_kind == MPM_MAT_SNOW) v = 1.0f;
    flat[e] = v;
}

extern "C" {

int mpm_fill_i32(int32_t *dst, int32_t n, int32_t value, void *stream_)
{
    if (n <= 0) return MPM_OK;
    if (!dst) return MPM_ERR_REJECTED_INPUT;
    launch_chained(fill_i32_kernel, nblk(n, 256), 256, (cudaStream_t)stream_, dst, n, value);
    return check_launch("mpm_fill_i32", 1);
}

int mpm_stage_particles(const float *pos, const float *vel, const float *mass, float mass_scalar, int32_t n,
                        int32_t nch, int32_t mat_kind, float *flat, void *stream_)
{
    if (n <= 0) return MPM_OK;
    if (!pos || !vel || !flat || nch <= CH_DEF) return MPM_ERR_REJECTED_INPUT;
    const long long n_elems = (long long)n * nch;
    launch_chained(stage_particles_kernel, nblk(n_elems, 256), 256, (cudaStream_t)stream_, pos, vel, mass,
                   mass_scalar, n_elems, nch, mat_kind, flat);
    return check_launch("mpm_stage_particles", 1);
}

int mpm_compact_live(const mpm_store_view *store, int drop_quarantined, int32_t *group_live_scratch,
                     int32_t *src_slot, int32_t *n_live, int32_t *scan_scratch, void *stream_)
{
    cudaStream_t stream = (cudaStream_t)stream_;
    const int G = store->n_groups;
    if (G <= 0) {
        cudaMemsetAsync(n_live, 0, sizeof(int32_t), stream);
        return check_launch("mpm_compact_live", 5);
    }
    launch_chained(live_count_kernel, nblk((int64_t)G * 32, 256), 256, stream, 
        store->lane_meta, store->group_len, G, store->n_groups_dev, drop_quarantined, group_live_scratch);
    exclusive_scan_i32(group_live_scratch, group_live_scratch, G, scan_scratch, n_live, stream);
    launch_chained(live_write_kernel, nblk((int64_t)G * 32, 256), 256, stream, 
        store->lane_meta, store->group_len, G, store->n_groups_dev, drop_quarantined, group_live_scratch, src_slot);
    return check_launch("mpm_compact_live", 5);
}

// `chained` = called from mpm_rebuild: the outputs (bad_index, overflow, bad_block, large_list[0])
// were initialised by rebuild_init_kernel, so the per-call fills are skipped.
static int particle_codes_impl(const mpm_store_view *store, const int32_t *src_slot, const int32_t *n_live_dev,
                               const float *staged, int32_t n_staged, int32_t n_upper, double dx,
                               int64_t *codes, int32_t *n_total, int32_t *bad_index, cudaStream_t stream,
                               bool chained)
{
    if (!(dx > 0.0)) return MPM_ERR_REJECTED_INPUT;
    if (!chained) launch_chained(fill_i32_kernel, 1, 32, stream, bad_index, 1, MPM_INT_MAX);
    if (n_live_dev) launch_chained(add_scalar_kernel, 1, 1, stream, n_total, n_live_dev, n_staged);
    else launch_chained(fill_i32_kernel, 1, 32, stream, n_total, 1, n_staged);
    if (n_upper > 0)
        launch_chained(particle_codes_kernel, nblk(n_upper, 256), 256, stream, 
            store->data, store->nch, src_slot, n_live_dev, staged, n_staged, n_upper, dx,
            (long long *)codes, bad_index);
    return check_launch("mpm_particle_codes", 3);
}

int mpm_particle_codes(const mpm_store_view *store, const int32_t *src_slot, const int32_t *n_live_dev,
                       const float *staged, int32_t n_staged, int32_t n_upper, double dx,
                       int64_t *codes, int32_t *n_total, int32_t *bad_index, void *stream_)
{
    return particle_codes_impl(store, src_slot, n_live_dev, staged, n_staged, n_upper, dx, codes, n_total,
                               bad_index, (cudaStream_t)stream_, false);
}

static int hash_insert_blocks_impl(const int64_t *codes, const int32_t *n_dev, int32_t n_upper,
                                   int64_t *hkeys, int32_t *hvals, int32_t *hfirst, int32_t hash_cap,
                                   int32_t *pslot, int32_t *flag_scratch, int32_t *scan_scratch,
                                   int32_t *gidx, int64_t *gcodes, int32_t *n_gblocks, int32_t *overflow,
                                   cudaStream_t stream, bool chained)
{
    if (hash_cap <= 0 || (hash_cap & (hash_cap - 1))) return MPM_ERR_REJECTED_INPUT;
    const int shift = hash_shift_for(hash_cap), mask = hash_cap - 1;
    launch_chained(hash_clear_kernel, nblk(hash_cap, 256), 256, stream, (long long *)hkeys, hvals, hfirst, hash_cap);
    if (!chained) cudaMemsetAsync(overflow, 0, sizeof(int32_t), stream);
    if (n_upper <= 0) {
        cudaMemsetAsync(n_gblocks, 0, sizeof(int32_t), stream);
        return check_launch("mpm_hash_insert_blocks", 8);
    }
    const int nb = nblk(n_upper, 256);
    launch_chained(block_insert_kernel, nb, 256, stream, (const long long *)codes, n_dev, n_upper,
                                                (long long *)hkeys, hfirst, shift, mask, pslot, overflow);
    launch_chained(first_flag_kernel, nb, 256, stream, pslot, hfirst, hvals, n_upper, (const int *)nullptr, 1, 0,
                   flag_scratch);
    exclusive_scan_i32(flag_scratch, flag_scratch, n_upper, scan_scratch, n_gblocks, stream);
    launch_chained(block_assign_kernel, nb, 256, stream, (const long long *)codes, pslot, hfirst, flag_scratch,
                                                n_upper, hvals, (long long *)gcodes);
    launch_chained(gidx_kernel, nb, 256, stream, pslot, hvals, n_upper, gidx);
    return check_launch("mpm_hash_insert_blocks", 8);
}

int mpm_hash_insert_blocks(const int64_t *codes, const int32_t *n_dev, int32_t n_upper,
                           int64_t *hkeys, int32_t *hvals, int32_t *hfirst, int32_t hash_cap,
                           int32_t *pslot, int32_t *flag_scratch, int32_t *scan_scratch,
                           int32_t *gidx, int64_t *gcodes, int32_t *n_gblocks, int32_t *overflow,
                           void *stream_)
{
    return hash_insert_blocks_impl(codes, n_dev, n_upper, hkeys, hvals, hfirst, hash_cap, pslot, flag_scratch,
                                   scan_scratch, gidx, gcodes, n_gblocks, overflow, (cudaStream_t)stream_, false);
}

// n_g lives on the device (*n_gblocks_dev, at most gblocks_bound): the launches are sized by the bound,
// so the host never waits for the block count in the middle of a rebuild.
static int dilate_and_link_impl(const int64_t *gcodes, const int32_t *n_g_dev, int32_t gblocks_bound,
                                int64_t *hkeys, int32_t *hvals, int32_t *hfirst, int32_t hash_cap,
                                int32_t *qslot, int32_t *flag_scratch, int32_t *scan_scratch, int64_t *codes,
                                int32_t *origin, int32_t *neighbor, int32_t pblock_cap, int32_t *count,
                                int32_t *bad_block, int32_t *overflow, cudaStream_t stream, bool chained)
{
    if (hash_cap <= 0 || (hash_cap & (hash_cap - 1))) return MPM_ERR_REJECTED_INPUT;
    const int shift = hash_shift_for(hash_cap), mask = hash_cap - 1;
    if (!chained) launch_chained(fill_i32_kernel, 1, 32, stream, bad_block, 1, MPM_INT_MAX);
    if (gblocks_bound <= 0) {
        cudaMemsetAsync(count, 0, sizeof(int32_t), stream);
        return check_launch("mpm_dilate_and_link", 9);
    }
    const int n_q = gblocks_bound * 27;
    const int nb = nblk(n_q, 256);
    // hfirst of the halo slots must start at INT_MAX: gblock slots already hold particle indices,
    // but those are never compared again (their hvals >= 0).
    launch_chained(dilate_insert_kernel, nb, 256, stream, (const long long *)gcodes, n_g_dev, (long long *)hkeys,
                                                 hvals, hfirst, shift, mask, qslot, bad_block, overflow);
    launch_chained(first_flag_kernel, nb, 256, stream, qslot, hfirst, hvals, n_q, n_g_dev, 27, 1, flag_scratch);
    // keep the flags: the scan result goes to a second array (flag_scratch + n_q)
    int32_t *rank = flag_scratch + n_q;
    exclusive_scan_i32(flag_scratch, rank, n_q, scan_scratch, count, stream, n_g_dev, 27, 0);
    launch_chained(dilate_assign_kernel, nb, 256, stream, qslot, flag_scratch, rank, n_g_dev, pblock_cap,
                                                 (const long long *)hkeys, (const long long *)gcodes, hvals,
                                                 (long long *)codes, overflow);
    launch_chained(dilate_link_kernel, nb, 256, stream, qslot, hvals, n_g_dev, neighbor);
    launch_chained(add_dev_kernel, 1, 1, stream, count, (const int *)count, n_g_dev);
    launch_chained(block_origin_kernel, nblk(pblock_cap, 256), 256, stream, (const long long *)codes, count,
                                                                   pblock_cap, (int4 *)origin);
    return check_launch("mpm_dilate_and_link", 9);
}

int mpm_dilate_and_link(const int64_t *gcodes, const int32_t *n_gblocks_dev, int32_t gblocks_bound,
                        int64_t *hkeys, int32_t *hvals, int32_t *hfirst, int32_t hash_cap, int32_t *qslot,
                        int32_t *flag_scratch, int32_t *scan_scratch, int64_t *codes, int32_t *origin,
                        int32_t *neighbor, int32_t pblock_cap, int32_t *count, int32_t *bad_block,
                        int32_t *overflow, void *stream_)
{
    if (!n_gblocks_dev) return MPM_ERR_REJECTED_INPUT;
    return dilate_and_link_impl(gcodes, n_gblocks_dev, gblocks_bound, hkeys, hvals, hfirst, hash_cap, qslot,
                                flag_scratch, scan_scratch, codes, origin, neighbor, pblock_cap, count, bad_block,
                                overflow, (cudaStream_t)stream_, false);
}

static int sort_and_group_impl(const int64_t *codes, const int32_t *gidx, const int32_t *n_dev, int32_t n_upper,
                               const int32_t *n_g_dev, int32_t gblocks_bound, int32_t *bin_start,
                               int32_t *tmp_perm, int32_t *perm, int32_t *block_group_first,
                               int32_t *scan_scratch, int32_t *n_groups, int32_t *large_scratch,
                               int32_t *large_list, cudaStream_t stream, bool chained)
{
    if (gblocks_bound <= 0 || n_upper <= 0) {
        cudaMemsetAsync(n_groups, 0, sizeof(int32_t), stream);
        return check_launch("mpm_sort_and_group", 12);
    }
    if (!large_scratch || !large_list) return MPM_ERR_REJECTED_INPUT;
    const int n_bins = gblocks_bound * 64;
    const int nb = nblk(n_upper, 256);
    // tickets live in `perm` until the final ranking overwrites it
    cudaMemsetAsync(bin_start, 0, sizeof(int32_t) * (size_t)(n_bins + 1), stream);
    launch_chained(hist_kernel, nb, 256, stream, (const long long *)codes, gidx, n_dev, n_upper, bin_start, perm);
    exclusive_scan_i32(bin_start, bin_start, n_bins + 1, scan_scratch, nullptr, stream, n_g_dev, 64, 1);
    launch_chained(place_kernel, nb, 256, stream, (const long long *)codes, gidx, n_dev, n_upper, bin_start,
                                         perm, tmp_perm);
    if (!chained) cudaMemsetAsync(large_list, 0, sizeof(int32_t), stream);
    launch_chained(stable_rank_kernel, nb, 256, stream, (const long long *)codes, gidx, n_dev, n_upper,
                                               bin_start, tmp_perm, perm, large_list);
    // bins above MPM_LARGE_BIN members (none in an ordinary scene: the kernel returns at once);
    // 2 * ceil(n/32) words per CTA fit n_upper words for every n that can hold a large bin
    if (n_upper > MPM_LARGE_BIN)
        launch_chained(large_bin_rank_kernel, LARGE_BIN_CTAS, 1024, stream, bin_start, tmp_perm, perm, large_list,
                       (unsigned *)large_scratch, (n_upper + 31) / 32);
    // n_g + 1 entries so that block_group_first[n_g] = n_groups after the scan
    launch_chained(block_groups_kernel, nblk(gblocks_bound + 1, 256), 256, stream, bin_start, n_g_dev,
                   block_group_first);
    exclusive_scan_i32(block_group_first, block_group_first, gblocks_bound + 1, scan_scratch, n_groups, stream,
                       n_g_dev, 1, 1);
    return check_launch("mpm_sort_and_group", 12);
}

int mpm_sort_and_group(const int64_t *codes, const int32_t *gidx, const int32_t *n_dev, int32_t n_upper,
                       const int32_t *n_gblocks_dev, int32_t gblocks_bound, int32_t *bin_start, int32_t *tmp_perm,
                       int32_t *perm, int32_t *block_group_first, int32_t *scan_scratch, int32_t *n_groups,
                       int32_t *large_scratch, int32_t *large_list, void *stream_)
{
    if (!n_gblocks_dev) return MPM_ERR_REJECTED_INPUT;
    return sort_and_group_impl(codes, gidx, n_dev, n_upper, n_gblocks_dev, gblocks_bound, bin_start, tmp_perm,
                               perm, block_group_first, scan_scratch, n_groups, large_scratch, large_list,
                               (cudaStream_t)stream_, false);
}

// n_groups / n_g from the device (new_store->n_groups is the launch bound when n_groups_dev is given)
static int scatter_sorted_impl(const mpm_store_view *old_store, const int32_t *src_slot, const int32_t *n_live_dev,
                               const float *staged, const int64_t *staged_ids, const int32_t *perm,
                               const int32_t *bin_start, const int32_t *block_group_first, const int32_t *n_g_dev,
                               const int32_t *table_origin, double dx, const mpm_store_view *new_store,
                               const int32_t *n_groups_dev, cudaStream_t stream)
{
    const int G = new_store->n_groups;
    if (G <= 0) return MPM_OK;
    const double inv_dx = 1.0 / dx;
#define MPM_SCATTER_SORTED(NCH)                                                                              \
    launch_chained(scatter_sorted_kernel<NCH>, nblk((int64_t)G * 32, 256), 256, stream, old_store->data,    \
                   (const long long *)old_store->orig_id, src_slot, n_live_dev, staged,                     \
                   (const long long *)staged_ids, perm, bin_start, block_group_first, n_g_dev,              \
                   (const int4 *)table_origin, inv_dx, new_store->data, (long long *)new_store->orig_id,    \
                   new_store->lane_meta, new_store->group_len, new_store->group_block,                      \
                   new_store->group_start, n_groups_dev, G)
    switch (new_store->nch) {
    case 17: MPM_SCATTER_SORTED(17); break;
    case 25: MPM_SCATTER_SORTED(25); break;
    case 26: MPM_SCATTER_SORTED(26); break;
    default: return MPM_ERR_CONFIG;
    }
#undef MPM_SCATTER_SORTED
    return check_launch("mpm_scatter_sorted", 1);
}

int mpm_scatter_sorted(const mpm_store_view *old_store, const int32_t *src_slot, const int32_t *n_live_dev,
                       const float *staged, const int64_t *staged_ids, const int32_t *perm,
                       const int32_t *bin_start, const int32_t *block_group_first, const int32_t *n_gblocks_dev,
                       const int32_t *table_origin, double dx, const mpm_store_view *new_store,
                       const int32_t *n_groups_dev, void *stream_)
{
    if (!n_gblocks_dev || !n_groups_dev) return MPM_ERR_REJECTED_INPUT;
    return scatter_sorted_impl(old_store, src_slot, n_live_dev, staged, staged_ids, perm, bin_start,
                               block_group_first, n_gblocks_dev, table_origin, dx, new_store, n_groups_dev,
                               (cudaStream_t)stream_);
}

}  // extern "C"

namespace mpm {
void rebuild_init(int32_t *S, int32_t *large_list, int32_t *guard_word, cudaStream_t stream)
{
    launch_chained(rebuild_init_kernel, 1, 32, stream, S, large_list, guard_word);
}
void rebuild_check_blocks(int32_t *S, int gblocks_bound, int hash_cap, int table_cap, int32_t *guard_word,
                          int guard_step, cudaStream_t stream)
{
    launch_chained(rebuild_check_blocks_kernel, 1, 1, stream, S, gblocks_bound, hash_cap, table_cap, guard_word,
                   guard_step);
}
void rebuild_check_groups(int32_t *S, int groups_cap, int nodes_cap, int32_t *guard_word, int guard_step,
                          int32_t *n_groups_out, cudaStream_t stream)
{
    launch_chained(rebuild_check_groups_kernel, 1, 1, stream, S, groups_cap, nodes_cap, guard_word, guard_step,
                   n_groups_out);
}
void zero_rows(float *rows, const int32_t *count_dev, int bound, cudaStream_t stream)
{
    if (bound > 0) launch_chained(zero_rows_kernel, (bound + 3) / 4, 256, stream, (float4 *)rows, count_dev, bound);
}
int rebuild_chain(const mpm_rebuild_plan *p, int32_t *S, int gblocks_bound, int groups_bound, cudaStream_t stream)
{
    const float *staged = p->n_staged ? p->staged : nullptr;
    const int64_t *staged_ids = p->n_staged ? p->staged_ids : nullptr;
    int rc = mpm_compact_live(&p->old_store, 1, p->glive, p->src_slot, S + 0, p->scan, stream);
    if (rc != MPM_OK) return rc;
    rc = particle_codes_impl(&p->old_store, p->src_slot, S + 0, staged, p->n_staged, p->n_upper, p->dx, p->codes,
                             S + 1, S + 2, stream, true);
    if (rc != MPM_OK) return rc;
    rc = hash_insert_blocks_impl(p->codes, S + 1, p->n_upper, p->hkeys, p->hvals, p->hfirst, p->hash_cap,
                                 p->pslot, p->flag, p->scan, p->gidx, p->gcodes, S + 3, S + 4, stream, true);
    if (rc != MPM_OK) return rc;
    rebuild_check_blocks(S, gblocks_bound, p->hash_cap, p->cap_table, p->guard_word, p->guard_step, stream);
    rc = dilate_and_link_impl(p->gcodes, S + 3, gblocks_bound, p->hkeys, p->hvals, p->hfirst, p->hash_cap,
                              p->qslot, p->qflag, p->scan, p->table_codes, p->table_origin, p->table_neighbor,
                              p->cap_table, S + 5, S + 6, S + 4, stream, true);
    if (rc != MPM_OK) return rc;
    // pslot / flag are free by now: scratch of the large-bin ranking (flag[0] was zeroed by rebuild_init)
    rc = sort_and_group_impl(p->codes, p->gidx, S + 1, p->n_upper, S + 3, gblocks_bound, p->bin_start,
                             p->tmp_perm, p->perm, p->bgf, p->scan, S + 7, p->pslot, p->large_list, stream, true);
    if (rc != MPM_OK) return rc;
    rebuild_check_groups(S, p->cap_groups, p->cap_nodes, p->guard_word, p->guard_step, p->n_groups_out, stream);
    mpm_store_view ns = p->new_store;
    ns.n_groups = groups_bound;
    ns.n_groups_dev = S + 7;
    rc = scatter_sorted_impl(&p->old_store, p->src_slot, S + 0, staged, staged_ids, p->perm, p->bin_start, p->bgf,
                             S + 3, p->table_origin, p->dx, &ns, S + 7, stream);
    return rc;
}
}  // namespace mpm

extern "C" {

int mpm_build_group_ctx(const mpm_store_view *store, const mpm_table_view *table, void *stream_)
{
    if (!store || !table || !store->group_ctx) return MPM_ERR_REJECTED_INPUT;
    const int G = store->n_groups;
    if (G <= 0) return MPM_OK;
    launch_chained(group_ctx_kernel, nblk((int64_t)G * 32, 256), 256, (cudaStream_t)stream_, 
        store->group_len, store->group_block, G, store->n_groups_dev, (const int4 *)table->origin,
        table->neighbor, store->group_ctx);
    return check_launch("mpm_build_group_ctx", 1);
}

int mpm_gather_state(const mpm_store_view *store, float *flat, int64_t *ids, void *stream_)
{
    cudaStream_t stream = (cudaStream_t)stream_;
    const int G = store->n_groups;
    if (G <= 0) return MPM_OK;
    if (store->nch > MPM_MAX_NCH) return MPM_ERR_CONFIG;
    launch_chained(gather_state_kernel, nblk((int64_t)G * 32, 256), 256, stream, 
        store->data, (const long long *)store->orig_id, store->nch, store->group_len,
        store->group_start, G, flat, (long long *)ids);
    return check_launch("mpm_gather_state", 1);
}

int mpm_gather_positions(const mpm_store_view *store, float *pos, int64_t *ids, void *stream_)
{
    cudaStream_t stream = (cudaStream_t)stream_;
    const int G = store->n_groups;
    if (G <= 0) return MPM_OK;
    launch_chained(gather_positions_kernel, nblk((int64_t)G * 32, 256), 256, stream, 
        store->data, (const long long *)store->orig_id, store->nch, store->group_len,
        store->group_start, G, pos, (long long *)ids);
    return check_launch("mpm_gather_positions", 1);
}

int mpm_tag_shared(const int64_t *peer_codes, int32_t n_peer_codes, const int64_t *hkeys,
                   const int32_t *hvals, int32_t hash_cap, int32_t *peer_map, int32_t local_count,
                   void *stream_)
{
    cudaStream_t stream = (cudaStream_t)stream_;
    if (hash_cap <= 0 || (hash_cap & (hash_cap - 1))) return MPM_ERR_REJECTED_INPUT;
    if (local_count > 0)
        launch_chained(fill_i32_kernel, nblk(local_count, 256), 256, stream, peer_map, local_count, -1);
    if (n_peer_codes > 0)
        launch_chained(tag_shared_kernel, nblk(n_peer_codes, 256), 256, stream, 
            (const long long *)peer_codes, n_peer_codes, (const long long *)hkeys, hvals,
            hash_shift_for(hash_cap), hash_cap - 1, peer_map);
    return check_launch("mpm_tag_shared", 2);
}

}  // extern "C"
