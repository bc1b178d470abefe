// Particle <-> grid transfers: P2G, G2P and the fused G2P2G kernel (sm_100a, fp32).
//
// Reference (paths relative to /root/reference/pkg/src/mpmbench/):
//   _scatter_prep      pipeline.py:160-238     _subgroup_scatter  pipeline.py:242-312
//   _p2g_kernel        pipeline.py:316-356     _gather_advect     pipeline.py:400-600
//   _g2p2g_kernel      pipeline.py:604-653
//
// Mapping: one warp per particle group (<= 32 particles of one gblock, cell-sorted at the
// last rebuild), lane = particle, one 128-byte row per channel.
// Scatter: runs of consecutive lanes with the same 10-bit cell key are summed with a
// segmented shuffle reduction and the run leader issues ONE vector reduction
// (RED.E.ADD.F32x4) per grid node -- the reference's "one += per (subgroup, node)" contract
// (pipeline.py:293-311) without sorting lanes first (its sort=none_between arm).
#include <type_traits>

#include "mpm_math.cuh"

namespace mpm {

struct TransferArgs {
    float *data;
    uint16_t *meta;
    const int *group_len;
    const int *group_block;
    const int *group_ctx;
    int n_groups;
    const int *n_groups_dev;   // optional: the count on the device (n_groups is then the launch bound)
    int nch;
    const int4 *origin;
    const int *neighbor;
    const float4 *vel;
    const float4 *vel_old;
    float4 *raw;
    uint8_t *touched;
    mpm_step_status *status;
    float dx, inv_dx, dt, dt_gather, d_inv, coeff_base;
    float mu, lam, kappa, gamma, flip;
    float margin_lo, margin_hi;
    float theta_c, theta_s, hardening, sand_alpha;
    int clamp_tension, count_stats, deterministic;
    // CFL-auto frames paced by the device: dt of the scatter / gather read from the clock
    const mpm_step_clock *clock;
    int clock_step, clock_gather_step;
    float coeff_per_dt;
    // particle sink: box in world coordinates, lanes inside it after advection are removed
    int sink_enabled;
    float sink_lo[3], sink_hi[3];
    long long *ids;
    DevGuard guard;
};

#ifndef MPM_TW
#define MPM_TW 8
#endif
#ifndef MPM_MINBLOCKS
#define MPM_MINBLOCKS 3
#endif
#ifndef MPM_LATE_F
#define MPM_LATE_F 1
#endif
#ifndef MPM_PREFETCH_F
#define MPM_PREFETCH_F 1  // deformation rows asked of L1 in the prologue (they are read after the node gather)
#endif
#ifndef MPM_ROLL_J
#define MPM_ROLL_J 0      // 1: scatter loops rolled over x and y (three nodes per trip)
#endif
#ifndef MPM_ONE_DEPTH
#define MPM_ONE_DEPTH 1   // 1: no separate instantiation for warps whose runs are all <= 2 lanes
#endif
#ifndef MPM_RUNCAP
#define MPM_RUNCAP 4      // power of two; 32 = one reduction per (subgroup, node) whatever the run length
#endif
#ifndef MPM_MASSFOLD
#define MPM_MASSFOLD 1    // scatter: particle mass folded into the x weight, Q carried per unit mass
#endif
#ifndef MPM_ROWLDS
#define MPM_ROWLDS 1      // neighbour-row lookups as explicit ld.shared on a byte address (one IADD each)
#endif
#ifndef MPM_GATHER_PREFETCH
#define MPM_GATHER_PREFETCH 0   // the eight node lines of a lane's stencil asked of L1 in the prologue
#endif
constexpr int TW = MPM_TW;   // warps (groups) per CTA

__device__ __forceinline__ void prefetch_l1(const void *p)
{
    asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}

// Neighbour-row lookup.  The row table of the warp sits in shared memory; `rowb` is the shared-space
// byte address of entry rx + 3 ry + 9 rz.  Written as an explicit ld.shared so that the address is
// one integer add per node (the compiler otherwise re-derives index * 4 + base with IMAD + LEA per
// node); the volatile form of the scatter keeps the load where it is written -- ahead of the
// shuffles whose latency it overlaps -- instead of being sunk into the run leader's branch.
__device__ __forceinline__ int row_lds(unsigned rowb)
{
    int v;
    asm("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(rowb));
    return v;
}
__device__ __forceinline__ int row_lds_pinned(unsigned rowb)
{
    int v;
    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(rowb));
    return v;
}

__device__ __forceinline__ void red_add_v4(float4 *addr, float a, float b, float c, float d)
{
    atomicAdd(addr, make_float4(a, b, c, d));   // RED.E.ADD.F32x4 on sm_90+
}

// Deterministic mode (pipeline.py:43-44, 297-301): contributions are quantised to integers,
// rint(c * 2^40) for mass and rint(c * 2^32) for momentum, and summed as int64 -- integer sums
// do not depend on the order of the atomics, so results are identical across worker counts,
// rebuild cadence and split / fused transfers.  A node is four int64 (32 bytes).
#define MPM_MASS_SCALE 1099511627776.0f
#define MPM_MOM_SCALE 4294967296.0f
__device__ __forceinline__ void red_add_det(long long *node, long long a, long long b, long long c, long long d)
{
    atomicAdd((unsigned long long *)node + 0, (unsigned long long)a);
    atomicAdd((unsigned long long *)node + 1, (unsigned long long)b);
    atomicAdd((unsigned long long *)node + 2, (unsigned long long)c);
    atomicAdd((unsigned long long *)node + 3, (unsigned long long)d);
}

__device__ __forceinline__ void quad_weights(float f, float *w)
{
    // pipeline.py:136-141
    w[0] = 0.5f * ((1.5f - f) * (1.5f - f));
    w[1] = 0.75f - (f - 1.0f) * (f - 1.0f);
    w[2] = 0.5f * ((f - 0.5f) * (f - 0.5f));
}
// the same weight for a loop index that is not a compile-time constant: with d = f - i,
// w_1 = 0.75 - d^2 and w_0, w_2 = 0.5 (1.5 - |d|)^2
__device__ __forceinline__ float quad_weight_at(float f, int i)
{
    const float d = f - (float)i;
    const float e = 1.5f - fabsf(d);
    return i == 1 ? 0.75f - d * d : 0.5f * (e * e);
}

// base cell (unbiased) of the quadratic stencil: floor(p * inv_dx - 0.5)
__device__ __forceinline__ float stencil_base(float p, float inv_dx, float *g)
{
    *g = p * inv_dx;
    return floorf(*g - 0.5f);
}

// ---------------------------------------------------------------------------------------
// Addressing from the lane key (pipeline.py:261-275).  A key digit k in 0..9 is the stencil
// base cell relative to (origin - 4); origin = 4 * block coordinate, so stencil cell
// t = k + i (0..11) lies in neighbour block t >> 2 (0..2) at in-block coordinate t & 3: every
// address is arithmetic on t, always inside the 3x3x3 neighbourhood, no validity branch.
// The node index is nrow[rx + 3 ry + 9 rz] + (sx | sy | sz) where nrow (shared memory) holds
// 64 * pblock of the 27 neighbours and s* are the slot bits of the axis (pipeline.py:144-147).
// ---------------------------------------------------------------------------------------
template <int AXIS>
__device__ __forceinline__ int slot_bits(int t)
{
    return ((t & 1) << AXIS) | ((t & 2) << (AXIS + 2));
}
__device__ __forceinline__ int axis_block_bits(int k)
{
    return (1 << (k >> 2)) | (1 << ((k + 2) >> 2));   // neighbour coordinates a stencil at digit k uses
}
// 27-bit mask of the neighbour blocks addressed by a stencil = outer product of the per-axis sets
__device__ __forceinline__ unsigned block_mask27(int kx, int ky, int kz)
{
    const unsigned row = (unsigned)axis_block_bits(kx);
    const int my = axis_block_bits(ky), mz = axis_block_bits(kz);
    const unsigned plane = ((my & 1) ? row : 0u) | ((my & 2) ? row << 3 : 0u) | ((my & 4) ? row << 6 : 0u);
    return ((mz & 1) ? plane : 0u) | ((mz & 2) ? plane << 9 : 0u) | ((mz & 4) ? plane << 18 : 0u);
}

// number of stencil cells that fall outside the 3x3x3 block neighbourhood, from the position
// (pipeline.py:266-275, 462-475): only evaluated for a particle whose key does not match its
// position any more (it left the neighbourhood: a contract violation, pipeline.py:1233-1238)
__device__ __noinline__ int count_bad_nodes(float px, float py, float pz, float inv_dx, int ox, int oy, int oz)
{
    const float p[3] = {px, py, pz};
    const int o[3] = {ox, oy, oz};
    int good[3];
#pragma unroll 1
    for (int a = 0; a < 3; ++a) {
        float g;
        const int cell = (int)stencil_base(p[a], inv_dx, &g) + MPM_CELL_BIAS;
        int n = 0;
#pragma unroll 1
        for (int i = 0; i < 3; ++i) {
            const int r = ((cell + i) >> 2) - (o[a] >> 2) + 1;
            n += (r >= 0 && r <= 2);
        }
        good[a] = n;
    }
    const int bad = 27 - good[0] * good[1] * good[2];
    return bad ? bad : 27;
}

// ---------------------------------------------------------------------------------------
// gather (pipeline.py:459-501): v = sum w v_n and B = sum w v_n (x) dpos evaluated as
// separable partial sums along z, then y, then x.  With node indices centred on the middle
// node (i-1 in {-1,0,1}) the first moments are M = sum w v_n (i-1), and
// B = dx (M - (f-1) v): ~240 flops instead of ~460 for the direct triple loop.  The x loop is
// kept rolled (nine nodes per trip): a third of the code, which matters because the kernel
// is far larger than the 32 KB instruction cache level next to the SM.
// ---------------------------------------------------------------------------------------
struct Gathered {
    float v[3];
    float B[9];     // row-major, B[a][b] = sum w v_a dpos_b
};

__device__ __forceinline__ void gather27(const float4 *__restrict__ vel, const int *nrow, int kx, int ky,
                                         int kz, float fx, float fy, float fz, float dx, Gathered &out)
{
    float wy[3], wz[3];
    quad_weights(fy, wy); quad_weights(fz, wz);
    int ry[3], rz[3], sy[3], sz[3];
#if MPM_ROWLDS
    const int nb = (int)__cvta_generic_to_shared(nrow);   // rows addressed in bytes (row_lds)
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        ry[q] = ((ky + q) >> 2) * 12; sy[q] = slot_bits<1>(ky + q);
        rz[q] = ((kz + q) >> 2) * 36 + nb; sz[q] = slot_bits<2>(kz + q);
    }
#else
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        ry[q] = ((ky + q) >> 2) * 3; sy[q] = slot_bits<1>(ky + q);
        rz[q] = ((kz + q) >> 2) * 9; sz[q] = slot_bits<2>(kz + q);
    }
#endif
    float V[3] = {0.f, 0.f, 0.f}, Mx[3] = {0.f, 0.f, 0.f}, My[3] = {0.f, 0.f, 0.f}, Mz[3] = {0.f, 0.f, 0.f};
#pragma unroll 1
    for (int i = 0; i < 3; ++i) {
#if MPM_ROWLDS
        const int rx = ((kx + i) >> 2) * 4, sx = slot_bits<0>(kx + i);
#else
        const int rx = (kx + i) >> 2, sx = slot_bits<0>(kx + i);
#endif
        const float wxi = quad_weight_at(fx, i);
        const float cmi = (float)(i - 1) * wxi;
        float S[3] = {0.f, 0.f, 0.f}, Ty[3] = {0.f, 0.f, 0.f}, Tz[3] = {0.f, 0.f, 0.f};
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            const int rxy = rx + ry[j];
            const int sxy = sx + sy[j];
            float4 n[3];
#if MPM_ROWLDS
#pragma unroll
            for (int k = 0; k < 3; ++k) n[k] = __ldg(&vel[row_lds((unsigned)(rxy + rz[k])) + sxy + sz[k]]);
#else
#pragma unroll
            for (int k = 0; k < 3; ++k) n[k] = __ldg(&vel[nrow[rxy + rz[k]] + sxy + sz[k]]);
#endif
            // along z: s = sum_k wz_k v_k, t = wz_2 v_2 - wz_0 v_0
            const float s0 = wz[0] * n[0].y + wz[1] * n[1].y + wz[2] * n[2].y;
            const float s1 = wz[0] * n[0].z + wz[1] * n[1].z + wz[2] * n[2].z;
            const float s2 = wz[0] * n[0].w + wz[1] * n[1].w + wz[2] * n[2].w;
            const float t0 = wz[2] * n[2].y - wz[0] * n[0].y;
            const float t1 = wz[2] * n[2].z - wz[0] * n[0].z;
            const float t2 = wz[2] * n[2].w - wz[0] * n[0].w;
            S[0] += wy[j] * s0; S[1] += wy[j] * s1; S[2] += wy[j] * s2;
            Tz[0] += wy[j] * t0; Tz[1] += wy[j] * t1; Tz[2] += wy[j] * t2;
            if (j != 1) {
                const float wj = j == 0 ? -wy[0] : wy[2];
                Ty[0] += wj * s0; Ty[1] += wj * s1; Ty[2] += wj * s2;
            }
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            V[c] += wxi * S[c];
            My[c] += wxi * Ty[c];
            Mz[c] += wxi * Tz[c];
            Mx[c] += cmi * S[c];
        }
    }
    const float gx = fx - 1.0f, gy = fy - 1.0f, gz = fz - 1.0f;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        out.v[c] = V[c];
        out.B[3 * c + 0] = dx * (Mx[c] - gx * V[c]);
        out.B[3 * c + 1] = dx * (My[c] - gy * V[c]);
        out.B[3 * c + 2] = dx * (Mz[c] - gz * V[c]);
    }
}

// FLIP increment sum w (v_n - v_old_n) (pipeline.py:489-495).  Only evaluated when blending:
// out of line and fully rolled, it costs the APIC path nothing.
__device__ __noinline__ void gather27_delta(const float4 *__restrict__ vel,
                                            const float4 *__restrict__ vel_old, const int *nrow,
                                            int kx, int ky, int kz, float fx, float fy, float fz,
                                            float *dv)
{
    float d0 = 0.f, d1 = 0.f, d2 = 0.f;
#pragma unroll 1
    for (int i = 0; i < 3; ++i) {
        const float wxi = quad_weight_at(fx, i);
#pragma unroll 1
        for (int j = 0; j < 3; ++j) {
            const float wxy = wxi * quad_weight_at(fy, j);
#pragma unroll 1
            for (int k = 0; k < 3; ++k) {
                const int r = ((kx + i) >> 2) + ((ky + j) >> 2) * 3 + ((kz + k) >> 2) * 9;
                const int idx = nrow[r] + (slot_bits<0>(kx + i) | slot_bits<1>(ky + j) | slot_bits<2>(kz + k));
                const float4 vn = __ldg(&vel[idx]), vo = __ldg(&vel_old[idx]);
                const float w = wxy * quad_weight_at(fz, k);
                d0 += w * (vn.y - vo.y); d1 += w * (vn.z - vo.z); d2 += w * (vn.w - vo.w);
            }
        }
    }
    dv[0] = d0; dv[1] = d1; dv[2] = d2;
}

// ---------------------------------------------------------------------------------------
// scatter (pipeline.py:242-312).  Momentum of node (i,j,k): w (m v + Q dpos) with
// dpos = ((i,j,k) - f) dx, built up axis by axis.  Runs of consecutive lanes with the same key
// are summed with a segmented shuffle reduction of NSTEPS = ceil(log2(longest run of the warp))
// steps and the run leader issues one vector reduction per node.  `reach` = lanes of my run
// after me; the step of distance D adds lane + D when reach >= D, expressed as a multiply by a
// 0/1 float so that the 27 x NSTEPS adds need no predicate.  NSTEPS is a template parameter
// (one dispatch per warp instead of a uniform branch per node and step); x loop rolled.
// ---------------------------------------------------------------------------------------
template <int NSTEPS, bool DET>
__device__ __forceinline__ void scatter27(float4 *__restrict__ raw, const int *nrow, int kx, int ky, int kz,
                                          float fx, float fy, float fz, float dx, float mm, float vx,
                                          float vy, float vz, const float *Q, int reach, int maxd,
                                          bool leader)
{
    const unsigned FULL = 0xffffffffu;
    typedef typename std::conditional<DET, long long, float>::type acc_t;
    float wy[3], wz[3];
    quad_weights(fy, wy); quad_weights(fz, wz);
    int ry[3], rz[3], sy[3], sz[3];
#if MPM_ROWLDS
    const int nb = (int)__cvta_generic_to_shared(nrow);   // rows addressed in bytes (row_lds)
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        ry[q] = ((ky + q) >> 2) * 12; sy[q] = slot_bits<1>(ky + q);
        rz[q] = ((kz + q) >> 2) * 36 + nb; sz[q] = slot_bits<2>(kz + q);
    }
#else
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        ry[q] = ((ky + q) >> 2) * 3; sy[q] = slot_bits<1>(ky + q);
        rz[q] = ((kz + q) >> 2) * 9; sz[q] = slot_bits<2>(kz + q);
    }
#endif
    float QZ[3][3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const float dpz = ((float)k - fz) * dx;
        QZ[k][0] = Q[2] * dpz; QZ[k][1] = Q[5] * dpz; QZ[k][2] = Q[8] * dpz;
    }
    const float f1 = reach >= 1 ? 1.0f : 0.0f, f2 = reach >= 2 ? 1.0f : 0.0f, f4 = reach >= 4 ? 1.0f : 0.0f,
                f8 = reach >= 8 ? 1.0f : 0.0f, f16 = reach >= 16 ? 1.0f : 0.0f;
#pragma unroll 1
    for (int i = 0; i < 3; ++i) {
#if MPM_ROWLDS
        const int rx = ((kx + i) >> 2) * 4, sx = slot_bits<0>(kx + i);
#else
        const int rx = (kx + i) >> 2, sx = slot_bits<0>(kx + i);
#endif
        const float dpx = ((float)i - fx) * dx;
#if MPM_MASSFOLD
        // Q is per unit mass here and the mass rides on the x weight: the node's mass share IS the
        // weight product, momentum = w (v + Q dpos); inactive lanes (mm = 0) contribute exact zeros
        const float wxi = mm * quad_weight_at(fx, i);
        const float X0 = vx + Q[0] * dpx, X1 = vy + Q[3] * dpx, X2 = vz + Q[6] * dpx;
#else
        const float wxi = mm > 0.0f ? quad_weight_at(fx, i) : 0.0f;   // inactive lanes contribute zeros
        const float X0 = mm * vx + Q[0] * dpx, X1 = mm * vy + Q[3] * dpx, X2 = mm * vz + Q[6] * dpx;
#endif
#if MPM_ROLL_J
#pragma unroll 1
#else
#pragma unroll
#endif
        for (int j = 0; j < 3; ++j) {
            const float dpy = ((float)j - fy) * dx;
#if MPM_ROLL_J
            const float wxy = wxi * quad_weight_at(fy, j);
            const int rxy = rx + ((ky + j) >> 2) * 3;
            const int sxy = sx + slot_bits<1>(ky + j);
#else
            const float wxy = wxi * wy[j];
            const int rxy = rx + ry[j];
            const int sxy = sx + sy[j];
#endif
            const float XY0 = X0 + Q[1] * dpy, XY1 = X1 + Q[4] * dpy, XY2 = X2 + Q[7] * dpy;
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const float w = wxy * wz[k];
                // issued before the shuffles so that its shared-memory latency overlaps them
#if MPM_ROWLDS
                const int node = row_lds_pinned((unsigned)(rxy + rz[k])) + sxy + sz[k];
#else
                const int node = nrow[rxy + rz[k]] + sxy + sz[k];
#endif
#if MPM_MASSFOLD
                const float wm = w;
#else
                const float wm = w * mm;
#endif
                acc_t c0, c1, c2, c3;
                if (DET) {
                    c0 = (acc_t)__float2ll_rn(wm * MPM_MASS_SCALE);
                    c1 = (acc_t)__float2ll_rn((w * (XY0 + QZ[k][0])) * MPM_MOM_SCALE);
                    c2 = (acc_t)__float2ll_rn((w * (XY1 + QZ[k][1])) * MPM_MOM_SCALE);
                    c3 = (acc_t)__float2ll_rn((w * (XY2 + QZ[k][2])) * MPM_MOM_SCALE);
                } else {
                    c0 = (acc_t)wm;
                    c1 = (acc_t)(w * (XY0 + QZ[k][0]));
                    c2 = (acc_t)(w * (XY1 + QZ[k][1]));
                    c3 = (acc_t)(w * (XY2 + QZ[k][2]));
                }
#define MPM_SEG_STEP(D, FD)                                                                         \
    if ((1 << (NSTEPS - 1)) >= D && (!DET || maxd >= D)) {                                          \
        const acc_t t0 = __shfl_down_sync(FULL, c0, D);                                             \
        const acc_t t1 = __shfl_down_sync(FULL, c1, D);                                             \
        const acc_t t2 = __shfl_down_sync(FULL, c2, D);                                             \
        const acc_t t3 = __shfl_down_sync(FULL, c3, D);                                             \
        if (DET) {                                                                                  \
            if (reach >= D) { c0 += t0; c1 += t1; c2 += t2; c3 += t3; }                             \
        } else {                                                                                    \
            c0 = (acc_t)fmaf((float)t0, FD, (float)c0); c1 = (acc_t)fmaf((float)t1, FD, (float)c1); \
            c2 = (acc_t)fmaf((float)t2, FD, (float)c2); c3 = (acc_t)fmaf((float)t3, FD, (float)c3); \
        }                                                                                           \
    }
                MPM_SEG_STEP(1, f1)
                MPM_SEG_STEP(2, f2)
                MPM_SEG_STEP(4, f4)
                MPM_SEG_STEP(8, f8)
                MPM_SEG_STEP(16, f16)
#undef MPM_SEG_STEP
                if (leader) {
                    if (DET) red_add_det((long long *)raw + (size_t)node * 4, (long long)c0, (long long)c1,
                                         (long long)c2, (long long)c3);
                    else red_add_v4(&raw[node], (float)c0, (float)c1, (float)c2, (float)c3);
                }
            }
        }
    }
}

template <int MAT>
__device__ __forceinline__ void load_deformation(const float *gd, float *F, float &plastic)
{
    if (MAT == MPM_MAT_FLUID) F[0] = gd[CH_DEF * 32];
    else {
#pragma unroll
        for (int r = 0; r < 9; ++r) F[r] = gd[(CH_DEF + r) * 32];
        if (MAT >= MPM_MAT_SNOW) plastic = gd[CH_PLASTIC * 32];
    }
}

template <int MAT, bool GATHER, bool SCATTER, bool DET>
__global__ void __launch_bounds__(TW * 32, MPM_MINBLOCKS) transfer_kernel(const TransferArgs a)
{
    pdl_wait();
    pdl_launch_dependents();
    if (guarded_out(a.guard)) return;
    __shared__ int s_nrow[TW][32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = blockIdx.x * TW + warp;
    const unsigned FULL = 0xffffffffu;
    if (g >= a.n_groups) return;     // warps are independent: no CTA-wide barrier below
    if (a.n_groups_dev && g >= __ldg(a.n_groups_dev)) return;

    // group context: neighbour row (as node indices of slot 0), block origin, group length.  One
    // 128-byte line per group written at the rebuild (mpm_build_group_ctx) -- every load of the
    // prologue depends on g alone; without it, the dependent chain through the block table.
    // Every prologue load is issued before the first use of any of them: context line, lane
    // meta, mass and position cost ONE trip to memory instead of three dependent ones (rows are
    // 32 lanes wide whatever the group length, and the rebuild zeroes the padding lanes).
    float *gd = a.data + (size_t)g * a.nch * 32 + lane;
    uint16_t meta = a.meta[g * 32 + lane];
    float m = gd[CH_MASS * 32];
    float px = gd[(CH_POS + 0) * 32], py = gd[(CH_POS + 1) * 32], pz = gd[(CH_POS + 2) * 32];
    // the running max |v|^2 is only a filter for the atomicMax at the end of the gather: an early
    // (possibly stale, never too large) copy saves a dependent trip to L2 there
    unsigned vmax_seen = 0;
    if (GATHER && lane == 0) vmax_seen = *((volatile unsigned *)&a.status->vmax2_bits);
#if MPM_LATE_F && MPM_PREFETCH_F
    if (GATHER) {
        // the deformation rows are read after the 27-node gather (register budget); asking L1 for
        // them now makes that read a hit
#pragma unroll
        for (int r = 0; r < (MAT == MPM_MAT_FLUID ? 1 : 9); ++r) prefetch_l1(gd + (CH_DEF + r) * 32);
        if (MAT >= MPM_MAT_SNOW) prefetch_l1(gd + CH_PLASTIC * 32);
    }
#endif
    int len;
    int4 org;
    if (a.group_ctx) {
        s_nrow[warp][lane] = __ldg(&a.group_ctx[g * 32 + lane]);
        __syncwarp();
        org.x = s_nrow[warp][27]; org.y = s_nrow[warp][28]; org.z = s_nrow[warp][29]; org.w = 0;
        len = s_nrow[warp][30];
    } else {
        len = a.group_len[g];
        const int block = a.group_block[g];
        org = a.origin[block];
        if (lane < 27) s_nrow[warp][lane] = a.neighbor[block * 27 + lane] * 64;
        __syncwarp();
    }
    const int *nrow = s_nrow[warp];

    bool active = lane < len && !(meta & MPM_LANE_QUARANTINED) && (m > 0.0f);
    if (!active) { m = 0.0f; px = py = pz = 0.0f; }
    int key = min(meta & 0x3ff, 999);     // three digits 0..9: every address below stays inside nrow

    float vx = 0.f, vy = 0.f, vz = 0.f;
    float C[9];
    float F[9];   // F (elastic kinds) or F[0] = J (fluid)
    float tau[9]; // plastic kinds: stress of the projected state, produced by the gather
    float plastic = 0.f;
    const PlasticParams pp = {a.mu, a.lam, a.theta_c, a.theta_s, a.hardening, a.sand_alpha};

    int addr_err = 0;
    unsigned vmax_bits = 0;
    // the deformation state is loaded after the 27-node gather (MPM_LATE_F): nine registers less
    // across the gather loop
    if (active && !(GATHER && MPM_LATE_F)) load_deformation<MAT>(gd, F, plastic);

    // =========================== gather (pipeline.py:400-600) ===========================
    if (GATHER) {
        if (active) {
            // The key was refreshed from this very position by the previous gather (or computed at
            // the rebuild), so its digits are the stencil base; the position relative to that base
            // must lie in [0.5, 1.5) cells.  If it does not, the particle has left the
            // neighbourhood its key can express (the digits were clamped).
            const int kx = key % 10, ky = (key / 10) % 10, kz = key / 100;
#if MPM_GATHER_PREFETCH
            // A stencil of three cells per axis covers two 2-cell pairs per axis: eight 128-byte node
            // lines.  Asking L1 for them now turns the nine dependent load batches of the node
            // gather into hits (they otherwise each expose an L2 round trip).
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int tx = kx + ((q & 1) << 1), ty = ky + (q & 2), tz = kz + ((q & 4) >> 1);
                const int row = nrow[(tx >> 2) + (ty >> 2) * 3 + (tz >> 2) * 9];
                prefetch_l1(&a.vel[row + (slot_bits<0>(tx) | slot_bits<1>(ty) | slot_bits<2>(tz))]);
            }
#endif
            const float fx = px * a.inv_dx - (float)(org.x - 4 + kx - MPM_CELL_BIAS);
            const float fy = py * a.inv_dx - (float)(org.y - 4 + ky - MPM_CELL_BIAS);
            const float fz = pz * a.inv_dx - (float)(org.z - 4 + kz - MPM_CELL_BIAS);
            if (!(fabsf(fx - 1.0f) <= 0.501f && fabsf(fy - 1.0f) <= 0.501f && fabsf(fz - 1.0f) <= 0.501f)) {
                // contract violation (pipeline.py:1233-1238): counted, particle left untouched
                addr_err += count_bad_nodes(px, py, pz, a.inv_dx, org.x, org.y, org.z);
                active = false;
            } else {
                Gathered G;
                gather27(a.vel, nrow, kx, ky, kz, fx, fy, fz, a.dx, G);
                if (MPM_LATE_F) load_deformation<MAT>(gd, F, plastic);
                float nvx = G.v[0], nvy = G.v[1], nvz = G.v[2];
#pragma unroll
                for (int r = 0; r < 9; ++r) C[r] = a.d_inv * G.B[r];
                if (a.flip > 0.0f) {
                    float dv[3];
                    gather27_delta(a.vel, a.vel_old, nrow, kx, ky, kz, fx, fy, fz, dv);
                    const float ovx = gd[(CH_VEL + 0) * 32], ovy = gd[(CH_VEL + 1) * 32],
                                ovz = gd[(CH_VEL + 2) * 32];
                    nvx = (1.0f - a.flip) * nvx + a.flip * (ovx + dv[0]);
                    nvy = (1.0f - a.flip) * nvy + a.flip * (ovy + dv[1]);
                    nvz = (1.0f - a.flip) * nvz + a.flip * (ovz + dv[2]);
                }
                // adaptive step size kept on the device (mpm_step_clock): a warp-uniform load, at the
                // point of use (the kernel has no register to carry it across the node gather)
                const float dtg = a.clock ? (float)__ldcg(&a.clock->dt[a.clock_gather_step & 1]) : a.dt_gather;
                const float npx = px + dtg * nvx, npy = py + dtg * nvy, npz = pz + dtg * nvz;
                if (!(isfinite(npx) && isfinite(npy) && isfinite(npz) && isfinite(nvx) &&
                      isfinite(nvy) && isfinite(nvz))) {
                    // quarantine (pipeline.py:525-531): state left as it was, mass zeroed
                    meta |= MPM_LANE_QUARANTINED;
                    a.meta[g * 32 + lane] = meta;
                    gd[CH_MASS * 32] = 0.0f;
                    atomicAdd(&a.status->counters[MPM_C_QUARANTINE], 1ull);
                    active = false;
                } else if (a.sink_enabled && npx >= a.sink_lo[0] && npx < a.sink_hi[0] && npy >= a.sink_lo[1] &&
                           npy < a.sink_hi[1] && npz >= a.sink_lo[2] && npz < a.sink_hi[2]) {
                    // sink: the particle arrives in the sink box and leaves the simulation -- like a
                    // quarantined lane it is skipped from here on (no deformation update, no free-zone
                    // test, no scatter) and dropped by the next rebuild's compaction
                    a.meta[g * 32 + lane] = (uint16_t)(meta | MPM_LANE_QUARANTINED | MPM_LANE_SUNK);
                    gd[(CH_POS + 0) * 32] = npx; gd[(CH_POS + 1) * 32] = npy; gd[(CH_POS + 2) * 32] = npz;
                    gd[CH_MASS * 32] = 0.0f;
                    a.ids[g * 32 + lane] = -1;
                    atomicAdd(&a.status->removed, 1ull);
                    active = false;
                } else {
                    px = npx; py = npy; pz = npz; vx = nvx; vy = nvy; vz = nvz;
                    gd[(CH_POS + 0) * 32] = px; gd[(CH_POS + 1) * 32] = py; gd[(CH_POS + 2) * 32] = pz;
                    gd[(CH_VEL + 0) * 32] = vx; gd[(CH_VEL + 1) * 32] = vy; gd[(CH_VEL + 2) * 32] = vz;
                    if (!SCATTER) {
                        // the fused kernel keeps C in registers; the split path stores it for P2G
#pragma unroll
                        for (int r = 0; r < 9; ++r) gd[(CH_C + r) * 32] = C[r];
                    }
                    if (MAT == MPM_MAT_FLUID) {
                        F[0] *= 1.0f + dtg * (C[0] + C[4] + C[8]);
                        gd[CH_DEF * 32] = F[0];
                    } else {
                        float A[9], Fn[9];
#pragma unroll
                        for (int r = 0; r < 9; ++r) A[r] = dtg * C[r];
                        A[0] += 1.0f; A[4] += 1.0f; A[8] += 1.0f;
#pragma unroll
                        for (int r = 0; r < 3; ++r)
#pragma unroll
                            for (int c = 0; c < 3; ++c)
                                Fn[3 * r + c] = A[3 * r] * F[c] + A[3 * r + 1] * F[3 + c] + A[3 * r + 2] * F[6 + c];
                        if (MAT >= MPM_MAT_SNOW) {
                            // return mapping (not in the reference; oracle: orc_snow_project / orc_sand_project)
                            plastic_project<MAT>(Fn, plastic, pp, tau);
                            gd[CH_PLASTIC * 32] = plastic;
                        }
#pragma unroll
                        for (int r = 0; r < 9; ++r) { F[r] = Fn[r]; gd[(CH_DEF + r) * 32] = Fn[r]; }
                    }
                    // new stencil base relative to (origin - 4): the lane key digits before clamping
                    // (pipeline.py:585-599); the free zone [origin - margin_lo, origin + 4 + margin_hi)
                    // cells is tested on the position itself (pipeline.py:560-575)
                    const float zx0 = ((float)(org.x - MPM_CELL_BIAS) - a.margin_lo) * a.dx;
                    const float zy0 = ((float)(org.y - MPM_CELL_BIAS) - a.margin_lo) * a.dx;
                    const float zz0 = ((float)(org.z - MPM_CELL_BIAS) - a.margin_lo) * a.dx;
                    const float zx1 = ((float)(org.x - MPM_CELL_BIAS) + 4.0f + a.margin_hi) * a.dx;
                    const float zy1 = ((float)(org.y - MPM_CELL_BIAS) + 4.0f + a.margin_hi) * a.dx;
                    const float zz1 = ((float)(org.z - MPM_CELL_BIAS) + 4.0f + a.margin_hi) * a.dx;
                    if (px < zx0 || px >= zx1 || py < zy0 || py >= zy1 || pz < zz0 || pz >= zz1) {
                        // bit 0 of the word (bit 1 belongs to the grid update's frame clock)
                        if (!(*(volatile int *)&a.status->zone_violation & MPM_STATUS_ZONE))
                            atomicOr(&a.status->zone_violation, MPM_STATUS_ZONE);
                        guard_raise(a.guard);
                    }
                    vmax_bits = __float_as_uint(vx * vx + vy * vy + vz * vz);
                    float tmp;
                    int nkx = (int)stencil_base(px, a.inv_dx, &tmp) + MPM_CELL_BIAS - (org.x - 4);
                    int nky = (int)stencil_base(py, a.inv_dx, &tmp) + MPM_CELL_BIAS - (org.y - 4);
                    int nkz = (int)stencil_base(pz, a.inv_dx, &tmp) + MPM_CELL_BIAS - (org.z - 4);
                    nkx = min(max(nkx, 0), 9); nky = min(max(nky, 0), 9); nkz = min(max(nkz, 0), 9);
                    key = nkx + 10 * (nky + 10 * nkz);
                    a.meta[g * 32 + lane] = (uint16_t)key;
                }
            }
        }
        // max |v|^2 of the warp -> one conditional atomicMax (pipeline.py:576-578)
        vmax_bits = __reduce_max_sync(FULL, vmax_bits);
        if (lane == 0 && vmax_bits > vmax_seen) atomicMax(&a.status->vmax2_bits, vmax_bits);
    } else if (SCATTER) {
        if (active) {
            vx = gd[(CH_VEL + 0) * 32]; vy = gd[(CH_VEL + 1) * 32]; vz = gd[(CH_VEL + 2) * 32];
#pragma unroll
            for (int r = 0; r < 9; ++r) C[r] = gd[(CH_C + r) * 32];
        }
    }

    // =========================== scatter (pipeline.py:160-312) ==========================
    if (SCATTER) {
        float Q[9];
        if (active && !GATHER) {
            if (!(isfinite(px) && isfinite(py) && isfinite(pz) && isfinite(vx) && isfinite(vy) &&
                  isfinite(vz))) {
                meta |= MPM_LANE_QUARANTINED;
                a.meta[g * 32 + lane] = meta;
                gd[CH_MASS * 32] = 0.0f;
                atomicAdd(&a.status->counters[MPM_C_QUARANTINE], 1ull);
                active = false;
            }
        }
        if (active) {
            // Q = m C - 4 dt / (rho dx^2) m tau (pipeline.py:226-238); MPM_MASSFOLD carries it per unit
            // mass (qm = 1) and scatter27 puts the mass on the weights
            const float cb = a.clock ? a.coeff_per_dt * (float)__ldcg(&a.clock->dt[a.clock_step & 1]) : a.coeff_base;
            const float qm = MPM_MASSFOLD ? 1.0f : m;
            const float coeff = cb * qm;
            if (MAT == MPM_MAT_FLUID) {
                float tau;
                if (F[0] <= 0.0f) {
                    atomicAdd(&a.status->counters[MPM_C_DEGENERATE], 1ull);
                    tau = 0.0f;
                } else tau = fluid_tau(F[0], a.kappa, a.gamma, a.clamp_tension);
#pragma unroll
                for (int r = 0; r < 9; ++r) Q[r] = qm * C[r];
                Q[0] += coeff * tau; Q[4] += coeff * tau; Q[8] += coeff * tau;
            } else if (MAT == MPM_MAT_FIXED_COROTATED) {
                float t[9];
                if (corotated_tau(F, a.mu, a.lam, t))
                    atomicAdd(&a.status->counters[MPM_C_SVD_CLAMP], 1ull);
#pragma unroll
                for (int r = 0; r < 9; ++r) Q[r] = qm * C[r] + coeff * t[r];
            } else {
                if (!GATHER) plastic_tau<MAT>(F, plastic, pp, tau);
#pragma unroll
                for (int r = 0; r < 9; ++r) Q[r] = qm * C[r] + coeff * tau[r];
            }
        } else {
            // lanes outside any run still take part in the shuffles: their payload must be exact
            // zeros (a 0/1 multiplier does not stop a NaN)
#pragma unroll
            for (int r = 0; r < 9; ++r) Q[r] = 0.0f;
            px = py = pz = 0.0f; vx = vy = vz = 0.0f;
        }
        // runs of consecutive active lanes with equal keys
        const unsigned act = __ballot_sync(FULL, active);
        const int prev_key = __shfl_up_sync(FULL, key, 1);
        bool head = !active || lane == 0 || prev_key != key || !((act >> (lane - 1)) & 1u);
        const unsigned run_heads = __ballot_sync(FULL, head);      // the reference's subgroups
        unsigned heads = run_heads;
#if MPM_RUNCAP < 32
        {
            // A run longer than MPM_RUNCAP lanes is reduced in pieces of MPM_RUNCAP, each with its
            // own leader: the reduction depth of the whole warp is bounded by log2(MPM_RUNCAP)
            // instead of being set by its longest run (just after a rebuild runs average 7 lanes),
            // at the price of one more vector reduction per node and extra piece.  Counters keep
            // the reference's meaning (runs, not pieces).
            const unsigned below = run_heads & ((2u << lane) - 1u);
            const int run_first = 31 - __clz(below);
            head = head || (((lane - run_first) & (MPM_RUNCAP - 1)) == 0);
            heads = __ballot_sync(FULL, head);
        }
#endif
        const unsigned above = lane == 31 ? 0u : (heads & ~((2u << lane) - 1u));
        const int reach = (above ? (__ffs(above) - 2) : 31) - lane;
        const int maxd = __reduce_max_sync(FULL, reach);
        if (act) {
            // addressing from the lane key (pipeline.py:261-272); weights relative to that base
            const int kx = key % 10, ky = (key / 10) % 10, kz = key / 100;
            const float fx = px * a.inv_dx - (float)(org.x - 4 + kx - MPM_CELL_BIAS);
            const float fy = py * a.inv_dx - (float)(org.y - 4 + ky - MPM_CELL_BIAS);
            const float fz = pz * a.inv_dx - (float)(org.z - 4 + kz - MPM_CELL_BIAS);
            const float mm = active ? m : 0.0f;
            const bool leader = head && active;
            if (DET) scatter27<5, true>((float4 *)a.raw, nrow, kx, ky, kz, fx, fy, fz, a.dx, mm, vx, vy, vz, Q, reach, maxd, leader);
#if !MPM_ONE_DEPTH
            else if (maxd < 2) scatter27<1, false>(a.raw, nrow, kx, ky, kz, fx, fy, fz, a.dx, mm, vx, vy, vz, Q, reach, maxd, leader);
#endif
            else if (MPM_RUNCAP <= 4 || maxd < 4) scatter27<2, false>(a.raw, nrow, kx, ky, kz, fx, fy, fz, a.dx, mm, vx, vy, vz, Q, reach, maxd, leader);
#if MPM_RUNCAP > 4
            else if (MPM_RUNCAP <= 8 || maxd < 8) scatter27<3, false>(a.raw, nrow, kx, ky, kz, fx, fy, fz, a.dx, mm, vx, vy, vz, Q, reach, maxd, leader);
#endif
#if MPM_RUNCAP > 8
            else scatter27<5, false>(a.raw, nrow, kx, ky, kz, fx, fy, fz, a.dx, mm, vx, vy, vz, Q, reach, maxd, leader);
#endif
            unsigned nbmask = leader ? block_mask27(kx, ky, kz) : 0u;
            nbmask = __reduce_or_sync(FULL, nbmask);
            if (lane < 27 && ((nbmask >> lane) & 1u)) a.touched[nrow[lane] >> 6] = 1;
            if (a.count_stats && lane == 0) {
                const int runs = __popc(run_heads & act);
                atomicAdd(&a.status->counters[MPM_C_SUBGROUPS], (unsigned long long)runs);
                atomicAdd(&a.status->counters[MPM_C_ACCUM], (unsigned long long)runs * 27ull);
            }
        }
    }
    if (addr_err) atomicAdd(&a.status->counters[MPM_C_ADDRESS_ERR], (unsigned long long)addr_err);
}

static int fill_args(TransferArgs &a, const mpm_store_view *store, const mpm_table_view *table,
                     const float *vel, const float *vel_old, float *raw, uint8_t *touched,
                     const mpm_transfer_params *p, mpm_step_status *status, const mpm_guard *guard)
{
    if (!store || !table || !p || !status) return MPM_ERR_REJECTED_INPUT;
    if (!(p->dx > 0.0) || !(p->density > 0.0)) return MPM_ERR_REJECTED_INPUT;
    if (p->mat_kind < 0 || p->mat_kind > MPM_MAT_SAND) return MPM_ERR_CONFIG;
    a.data = store->data;
    a.meta = store->lane_meta;
    a.group_len = store->group_len;
    a.group_block = store->group_block;
    a.group_ctx = store->group_ctx;
    a.n_groups = store->n_groups;
    a.n_groups_dev = store->n_groups_dev;
    a.nch = store->nch;
    a.origin = (const int4 *)table->origin;
    a.neighbor = table->neighbor;
    a.vel = (const float4 *)vel;
    a.vel_old = (const float4 *)vel_old;
    a.raw = (float4 *)raw;
    a.touched = touched;
    a.status = status;
    const double inv_dx = 1.0 / p->dx;
    a.dx = (float)p->dx;
    a.inv_dx = (float)inv_dx;
    a.dt = (float)p->dt;
    a.dt_gather = (float)p->dt_gather;
    a.d_inv = (float)(4.0 * inv_dx * inv_dx);
    a.coeff_base = (float)(-4.0 * p->dt * inv_dx * inv_dx / p->density);
    a.coeff_per_dt = (float)(-4.0 * inv_dx * inv_dx / p->density);
    a.clock = p->clock;
    a.clock_step = p->clock_step;
    a.clock_gather_step = p->clock_gather_step;
    a.sink_enabled = p->sink_enabled;
    for (int k = 0; k < 3; ++k) { a.sink_lo[k] = (float)p->sink_lo[k]; a.sink_hi[k] = (float)p->sink_hi[k]; }
    a.ids = (long long *)store->orig_id;
    if (a.sink_enabled && !a.ids) return MPM_ERR_REJECTED_INPUT;
    a.mu = (float)p->mu; a.lam = (float)p->lam; a.kappa = (float)p->kappa; a.gamma = (float)p->gamma;
    a.flip = (float)p->flip_blend;
    a.margin_lo = (float)p->margin_lo; a.margin_hi = (float)p->margin_hi;
    a.theta_c = (float)p->theta_c; a.theta_s = (float)p->theta_s;
    a.hardening = (float)p->hardening; a.sand_alpha = (float)p->sand_alpha;
    a.clamp_tension = p->clamp_tension;
    a.count_stats = p->count_stats;
    a.deterministic = p->deterministic;
    a.guard = make_guard(guard);
    if (a.flip > 0.0f && !vel_old) return MPM_ERR_REJECTED_INPUT;
    return MPM_OK;
}

template <bool GATHER, bool SCATTER>
static int launch_transfer(const TransferArgs &a, int mat, cudaStream_t stream)
{
    if (a.n_groups <= 0) return MPM_OK;
    const int grid = (a.n_groups + TW - 1) / TW;
    if (a.deterministic && SCATTER) {
        // fixed-point accumulation exists for the reference's own material kinds
        switch (mat) {
        case MPM_MAT_FLUID:
            launch_chained(transfer_kernel<MPM_MAT_FLUID, GATHER, SCATTER, true>, grid, TW * 32, stream, a);
            return MPM_OK;
        case MPM_MAT_FIXED_COROTATED:
            launch_chained(transfer_kernel<MPM_MAT_FIXED_COROTATED, GATHER, SCATTER, true>, grid, TW * 32, stream, a);
            return MPM_OK;
        default:
            return MPM_ERR_CONFIG;
        }
    }
    switch (mat) {
    case MPM_MAT_FLUID:
        launch_chained(transfer_kernel<MPM_MAT_FLUID, GATHER, SCATTER, false>, grid, TW * 32, stream, a);
        break;
    case MPM_MAT_FIXED_COROTATED:
        launch_chained(transfer_kernel<MPM_MAT_FIXED_COROTATED, GATHER, SCATTER, false>, grid, TW * 32, stream, a);
        break;
    case MPM_MAT_SNOW:
        launch_chained(transfer_kernel<MPM_MAT_SNOW, GATHER, SCATTER, false>, grid, TW * 32, stream, a);
        break;
    case MPM_MAT_SAND:
        launch_chained(transfer_kernel<MPM_MAT_SAND, GATHER, SCATTER, false>, grid, TW * 32, stream, a);
        break;
    default:
        return MPM_ERR_CONFIG;
    }
    return MPM_OK;
}

}  // namespace mpm

using namespace mpm;

extern "C" {

int mpm_p2g(const mpm_store_view *store, const mpm_table_view *table, float *raw, uint8_t *touched,
            const mpm_transfer_params *params, mpm_step_status *status, const mpm_guard *guard, void *stream)
{
    TransferArgs a;
    int rc = fill_args(a, store, table, nullptr, nullptr, raw, touched, params, status, guard);
    if (rc == MPM_ERR_REJECTED_INPUT && params && params->flip_blend > 0.0) {
        // P2G does not read vel_old
        mpm_transfer_params q = *params;
        q.flip_blend = 0.0;
        rc = fill_args(a, store, table, nullptr, nullptr, raw, touched, &q, status, guard);
    }
    if (rc != MPM_OK) return rc;
    rc = launch_transfer<false, true>(a, params->mat_kind, (cudaStream_t)stream);
    if (rc != MPM_OK) return rc;
    return check_launch("mpm_p2g", 1);
}

int mpm_g2p(const mpm_store_view *store, const mpm_table_view *table, const float *vel,
            const float *vel_old, const mpm_transfer_params *params, mpm_step_status *status,
            const mpm_guard *guard, void *stream)
{
    TransferArgs a;
    int rc = fill_args(a, store, table, vel, vel_old, nullptr, nullptr, params, status, guard);
    if (rc != MPM_OK) return rc;
    rc = launch_transfer<true, false>(a, params->mat_kind, (cudaStream_t)stream);
    if (rc != MPM_OK) return rc;
    return check_launch("mpm_g2p", 1);
}

int mpm_g2p2g(const mpm_store_view *store, const mpm_table_view *table, const float *vel,
              const float *vel_old, float *raw, uint8_t *touched, const mpm_transfer_params *params,
              mpm_step_status *status, const mpm_guard *guard, void *stream)
{
    TransferArgs a;
    int rc = fill_args(a, store, table, vel, vel_old, raw, touched, params, status, guard);
    if (rc != MPM_OK) return rc;
    rc = launch_transfer<true, true>(a, params->mat_kind, (cudaStream_t)stream);
    if (rc != MPM_OK) return rc;
    return check_launch("mpm_g2p2g", 1);
}

}  // extern "C"
