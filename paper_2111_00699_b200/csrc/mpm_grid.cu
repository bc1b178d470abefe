// Grid kernels: buffer clear and the fused reduce + update + boundary kernel (sm_100a).
//
// Reference (paths relative to /root/reference/pkg/src/mpmbench/):
//   Worker._clear             pipeline.py:1022-1037
//   Worker._reduce_and_update pipeline.py:1166-1231
//   _grid_finalize            pipeline.py:660-722
//
// One thread per grid node, four 4^3 blocks (256 nodes) per CTA; a node is one float4
// (mass, momentum) so every access is a 16-byte vector and a warp covers 512 contiguous
// bytes.  Untouched blocks exit after one flag read, so the launch covers the whole block
// table and no compacted index list (the reference's flatnonzero) is needed.
#include "mpm_common.cuh"

namespace mpm {

struct PeerSet {
    const float4 *raw[MPM_MAX_PEERS];
    const uint8_t *touched[MPM_MAX_PEERS];
    const int *map[MPM_MAX_PEERS];
    int n;
};

__global__ void __launch_bounds__(256) clear_kernel(float4 *raw, uint8_t *touched, int count,
                                                    const int *__restrict__ count_dev, int full,
                                                    int vec_per_node, const DevGuard guard)
{
    pdl_wait();
    pdl_launch_dependents();
    if (guarded_out(guard)) return;
    if (count_dev) count = min(count, *count_dev);
    const int b = blockIdx.x * 4 + (threadIdx.x >> 6);
    const int slot = threadIdx.x & 63;
    const bool hit = b < count && (full || touched[b]);
    __syncthreads();   // every thread has read the flag before it is reset
    if (hit) {
        for (int v = 0; v < vec_per_node; ++v)
            raw[((size_t)b * 64 + slot) * vec_per_node + v] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (slot == 0) touched[b] = 0;
    }
}

struct GridArgs {
    const float4 *raw;
    const uint8_t *touched;
    float4 *vel;
    float4 *vel_old;
    const int4 *origin;
    int count;
    const int *count_dev;      // optional: the count on the device (count is then the launch bound)
    PeerSet peers;
    float dt;
    float gx, gy, gz;
    int apply_bc, bc_sticky;
    double blo[3], bhi[3];
    double dx;
    int fuse_clear;
    int block_filter;
    int deterministic;
    float4 *raw_mut;
    uint8_t *touched_mut;
    DevGuard guard;
    mpm_step_status *reset_status;
    // device-side step barrier (peer rows read in place)
    int n_wait, wait_value, wait_timeout_ms;
    const int *wait_flags[MPM_MAX_PEERS];
    int *wait_error;
    // status publication to mapped host memory (mpm_grid_params.publish_*)
    const mpm_step_status *publish_src;
    mpm_step_status *publish_dst;
    const int *publish_guard_src;
    int *publish_guard_dst;
    // device step clock of CFL-auto frames (mpm_grid_params.clock)
    mpm_step_clock *clock;
    int clock_step, vmax_ring_len, n_vmax_peers;
    const mpm_step_status *vmax_ring;
    mpm_step_status *clock_status;
    double frame_dt, cfl_dx, c_sound;
    const mpm_step_status *vmax_peer_rings[MPM_MAX_PEERS];
    unsigned long long *prof;      // optional counters: launches, barrier wait ns, peer bytes, waiting CTAs
};

// Worker.run_frame's CFL loop (pipeline.py:856-871) for ONE step, on the device: account for step
// s = clock_step, decide whether it completed the frame, and set the size of step s + 1 from the
// max speed of step s - 1 (the reference's two-step lag, pipeline.py:866).  float64 like the
// reference; one thread.
__device__ __forceinline__ void advance_clock(const GridArgs &a)
{
    const int s = a.clock_step;
    const double dt_s = a.clock->dt[s & 1];
    double t = a.clock->t + dt_s;
    const bool frame_end = !(t < a.frame_dt - 1e-12);
    if (frame_end) t = 0.0;
    const int slot = (s - 1 + a.vmax_ring_len) % a.vmax_ring_len;
    unsigned bits = *(volatile const unsigned *)&a.vmax_ring[slot].vmax2_bits;
    for (int p = 0; p < a.n_vmax_peers; ++p) {
        unsigned o;
        asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(o) : "l"(&a.vmax_peer_rings[p][slot].vmax2_bits) : "memory");
        bits = o > bits ? o : bits;          // nonnegative floats: unsigned order = float order
    }
    const double vmax = sqrt((double)__uint_as_float(bits));
    const double speed = vmax + a.c_sound;
    double dt_next = a.cfl_dx / (speed > 1e-12 ? speed : 1e-12);
    const double remaining = a.frame_dt - t;
    if (remaining < dt_next) dt_next = remaining;
    a.clock->dt[(s + 1) & 1] = dt_next;
    a.clock->t = t;
    if (a.clock_status) {
        a.clock_status->dt = dt_s;
        if (frame_end) atomicOr(&a.clock_status->zone_violation, MPM_STATUS_FRAME_END);
    }
    if (frame_end) guard_raise(a.guard);     // steps enqueued beyond the frame are void
}

// 56-byte status block (+ guard word) to mapped pinned host memory: lanes 0..6 one 8-byte word each
__device__ __forceinline__ void publish_status(const mpm_step_status *src, mpm_step_status *dst,
                                               const int *guard_src, int *guard_dst, int lane)
{
    static_assert(sizeof(mpm_step_status) % 8 == 0, "status block is copied in 8-byte words");
    if (dst && lane < (int)(sizeof(mpm_step_status) / 8))
        ((volatile unsigned long long *)dst)[lane] = ((const volatile unsigned long long *)src)[lane];
    if (guard_dst && lane == 31) *(volatile int *)guard_dst = *(const volatile int *)guard_src;
    __threadfence_system();
}

__device__ __forceinline__ int ld_acquire_sys(const int *p)
{
    int v;
    asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long global_timer_ns()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

__global__ void __launch_bounds__(256) grid_update_kernel(const GridArgs a)
{
    pdl_wait();
    pdl_launch_dependents();
    if (guarded_out(a.guard)) {
        // a skipped step still tells the host where the guard stood
        if (a.publish_guard_dst && blockIdx.x == 0 && threadIdx.x == 31)
            publish_status(nullptr, nullptr, a.publish_guard_src, a.publish_guard_dst, 31);
        return;
    }
    if (a.reset_status && blockIdx.x == 0 && threadIdx.x == 0) {
        // fresh out_stats for the gather that follows this update in stream order
        a.reset_status->zone_violation = 0;
        a.reset_status->vmax2_bits = 0;
    }
    const int b = blockIdx.x * 4 + (threadIdx.x >> 6);
    const int slot = threadIdx.x & 63;
    bool hit = b < a.count && (!a.count_dev || b < __ldg(a.count_dev)) && a.touched[b];
    if (a.n_wait) {
        // Step barrier on the device: the peers' scatter of this step must be complete before
        // their rows are read.  Only CTAs that own a block shared with a peer wait (and CTA 0, so
        // that the kernel as a whole -- hence everything after it in the stream -- is ordered
        // after every peer's signal and after any guard the peers raised).
        __shared__ int s_wait, s_void;
        if (threadIdx.x == 0) { s_wait = blockIdx.x == 0; s_void = 0; }
        __syncthreads();
        if (hit && slot == 0) {
            bool shared = false;
            for (int p = 0; p < a.peers.n; ++p) shared = shared || a.peers.map[p][b] >= 0;
            if (shared) s_wait = 1;
        }
        __syncthreads();
        if (s_wait) {
            if (a.prof && threadIdx.x == 0) atomicAdd(&a.prof[3], 1ull);
            if (threadIdx.x < a.n_wait) {
                const int *flag = a.wait_flags[threadIdx.x];
                const unsigned long long t0 = global_timer_ns();
                const unsigned long long limit = (unsigned long long)a.wait_timeout_ms * 1000000ull;
                while (ld_acquire_sys(flag) < a.wait_value) {
                    // Split transfers gather AFTER this barrier: a peer whose gather of step s left
                    // its free zone raises the guard while this rank may already be waiting in step
                    // s + 1 for a signal the peer will never send (its step s + 1 is guarded out).
                    // The raise reaches this rank's word too: the step is void, stop waiting.
                    if (a.guard.word && ld_acquire_sys(a.guard.word) < a.guard.step) {
                        s_void = 1;
                        break;
                    }
                    if (global_timer_ns() - t0 > limit) {
                        if (a.wait_error) atomicExch(a.wait_error, 1);
                        break;
                    }
                    __nanosleep(200);
                }
                if (a.prof && blockIdx.x == 0) atomicMax(&a.prof[4], global_timer_ns() - t0);
            }
            __syncthreads();
            if (a.prof && blockIdx.x == 0 && threadIdx.x == 0) {
                // CTA 0 waits for every peer: its longest wait is the barrier latency of this launch
                atomicAdd(&a.prof[0], 1ull);
                atomicAdd(&a.prof[1], atomicExch(&a.prof[4], 0ull));
            }
            if (s_void) {
                if (a.publish_guard_dst && blockIdx.x == 0 && threadIdx.x == 31)
                    publish_status(nullptr, nullptr, a.publish_guard_src, a.publish_guard_dst, 31);
                return;
            }
        }
    }
    float dt = a.dt;
    if (a.clock) {
        dt = (float)__ldcg(&a.clock->dt[a.clock_step & 1]);
        if (blockIdx.x == 0 && threadIdx.x < 32) {
            // entry (s + 1) & 1 is written, entry s & 1 (read by every CTA) is not
            if (threadIdx.x == 0) advance_clock(a);
            __threadfence();
            __syncwarp();
        }
    }
    // after the barrier: a guard raised by a peer during this step has landed
    if ((a.publish_dst || a.publish_guard_dst) && blockIdx.x == 0 && threadIdx.x < 32)
        publish_status(a.publish_src, a.publish_dst, a.publish_guard_src, a.publish_guard_dst, threadIdx.x);
    if (hit && a.block_filter) {
        // 1: only blocks no peer holds (can run while the halo rows are in flight), 2: the rest
        bool shared = false;
        for (int p = 0; p < a.peers.n; ++p) shared = shared || a.peers.map[p][b] >= 0;
        hit = (a.block_filter == 2) == shared;
    }
    if (a.fuse_clear) __syncthreads();
    if (!hit) return;
    const size_t idx = (size_t)b * 64 + slot;
    float m, vx, vy, vz;
    if (a.deterministic) {
        // integer sums (pipeline.py:682-686): mass = m 2^-40, v = (p 2^-32) / mass, in float64
        const longlong4 *rawd = (const longlong4 *)a.raw;
        longlong4 node = rawd[idx];
        for (int p = 0; p < a.peers.n; ++p) {
            const int q = a.peers.map[p][b];
            if (q < 0 || (a.peers.touched[p] && __ldcv(&a.peers.touched[p][q]) != 1)) continue;
            const longlong2 *src = (const longlong2 *)a.peers.raw[p] + ((size_t)q * 64 + slot) * 2;
            const longlong2 lo = __ldcg(src), hi = __ldcg(src + 1);
            const longlong4 o = make_longlong4(lo.x, lo.y, hi.x, hi.y);
            node.x += o.x; node.y += o.y; node.z += o.z; node.w += o.w;
        }
        if (a.fuse_clear) {
            ((longlong4 *)a.raw_mut)[idx] = make_longlong4(0, 0, 0, 0);
            if (slot == 0) a.touched_mut[b] = 0;
        }
        if (node.x <= 0) {
            a.vel[idx] = make_float4(0.f, 0.f, 0.f, 0.f);
            return;
        }
        const double mass = (double)node.x * (1.0 / 1099511627776.0);
        const double inv = (1.0 / 4294967296.0) / mass;
        m = (float)mass;
        vx = (float)((double)node.y * inv); vy = (float)((double)node.z * inv); vz = (float)((double)node.w * inv);
    } else {
        float4 node = a.raw[idx];
        // cross-worker reduction (pipeline.py:1172-1188): peers' raw rows are only read
        for (int p = 0; p < a.peers.n; ++p) {
            const int q = a.peers.map[p][b];
            if (q < 0 || (a.peers.touched[p] && __ldcv(&a.peers.touched[p][q]) != 1)) continue;
            const float4 o = __ldcg(&a.peers.raw[p][(size_t)q * 64 + slot]);
            node.x += o.x; node.y += o.y; node.z += o.z; node.w += o.w;
            if (a.prof && slot == 0) atomicAdd(&a.prof[2], 1024ull);
        }
        if (a.fuse_clear) {
            a.raw_mut[idx] = make_float4(0.f, 0.f, 0.f, 0.f);
            if (slot == 0) a.touched_mut[b] = 0;
        }
        m = node.x;
        if (!(m > 0.0f)) {   // m <= 0 (pipeline.py:676-681)
            a.vel[idx] = make_float4(0.f, 0.f, 0.f, 0.f);
            return;
        }
        vx = node.y / m; vy = node.z / m; vz = node.w / m;
    }
    if (a.vel_old) a.vel_old[idx] = make_float4(0.f, vx, vy, vz);   // saved before gravity (:692-698)
    vx += dt * a.gx; vy += dt * a.gy; vz += dt * a.gz;
    if (a.apply_bc) {
        // node world position in float64 so that the inclusive comparisons of
        // pipeline.py:707-718 classify nodes exactly like the reference
        const int4 org = a.origin[b];
        const int sx = (slot & 1) | ((slot >> 2) & 2);
        const int sy = ((slot >> 1) & 1) | ((slot >> 3) & 2);
        const int sz = ((slot >> 2) & 1) | ((slot >> 4) & 2);
        const double px = (double)(org.x - MPM_CELL_BIAS + sx) * a.dx;
        const double py = (double)(org.y - MPM_CELL_BIAS + sy) * a.dx;
        const double pz = (double)(org.z - MPM_CELL_BIAS + sz) * a.dx;
        if (a.bc_sticky) {
            if (px <= a.blo[0] || px >= a.bhi[0] || py <= a.blo[1] || py >= a.bhi[1] ||
                pz <= a.blo[2] || pz >= a.bhi[2]) { vx = 0.f; vy = 0.f; vz = 0.f; }
        } else {
            if ((px <= a.blo[0] && vx < 0.f) || (px >= a.bhi[0] && vx > 0.f)) vx = 0.f;
            if ((py <= a.blo[1] && vy < 0.f) || (py >= a.bhi[1] && vy > 0.f)) vy = 0.f;
            if ((pz <= a.blo[2] && vz < 0.f) || (pz >= a.bhi[2] && vz > 0.f)) vz = 0.f;
        }
    }
    a.vel[idx] = make_float4(m, vx, vy, vz);
}

// ---- aggregates (float64 accumulation) ----------------------------------------------
__device__ __forceinline__ double warp_sum(double v)
{
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v += __shfl_down_sync(0xffffffffu, v, d);
    return v;
}

__global__ void __launch_bounds__(256) particle_aggregates_kernel(const float *__restrict__ data, int nch,
                                                                  const int *__restrict__ group_len,
                                                                  int n_groups, double *out5)
{
    pdl_wait();
    pdl_launch_dependents();
    const int g = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    double m = 0, mx = 0, my = 0, mz = 0, ke = 0;
    if (g < n_groups && lane < group_len[g]) {
        const float *gd = data + (size_t)g * nch * 32 + lane;
        m = gd[CH_MASS * 32];
        if (m > 0.0) {   // quarantined lanes carry mass 0 and possibly non-finite velocities
            const double vx = gd[(CH_VEL + 0) * 32], vy = gd[(CH_VEL + 1) * 32], vz = gd[(CH_VEL + 2) * 32];
            mx = m * vx; my = m * vy; mz = m * vz;
            ke = 0.5 * m * (vx * vx + vy * vy + vz * vz);
        }
    }
    m = warp_sum(m); mx = warp_sum(mx); my = warp_sum(my); mz = warp_sum(mz); ke = warp_sum(ke);
    if (lane == 0 && g < n_groups) {
        atomicAdd(&out5[0], m); atomicAdd(&out5[1], mx); atomicAdd(&out5[2], my);
        atomicAdd(&out5[3], mz); atomicAdd(&out5[4], ke);
    }
}

__global__ void __launch_bounds__(256) grid_aggregates_kernel(const float4 *__restrict__ raw,
                                                              const uint8_t *__restrict__ touched,
                                                              int count, int det, double *out4)
{
    pdl_wait();
    pdl_launch_dependents();
    const int b = blockIdx.x * 4 + (threadIdx.x >> 6);
    const int slot = threadIdx.x & 63;
    const int lane = threadIdx.x & 31;
    double m = 0, mx = 0, my = 0, mz = 0;
    if (b < count && touched[b]) {
        if (det) {
            const longlong4 n = ((const longlong4 *)raw)[(size_t)b * 64 + slot];
            m = (double)n.x / 1099511627776.0;
            mx = (double)n.y / 4294967296.0; my = (double)n.z / 4294967296.0; mz = (double)n.w / 4294967296.0;
        } else {
            const float4 n = raw[(size_t)b * 64 + slot];
            m = n.x; mx = n.y; my = n.z; mz = n.w;
        }
    }
    m = warp_sum(m); mx = warp_sum(mx); my = warp_sum(my); mz = warp_sum(mz);
    if (lane == 0 && m != 0.0) {
        atomicAdd(&out4[0], m); atomicAdd(&out4[1], mx); atomicAdd(&out4[2], my); atomicAdd(&out4[3], mz);
    }
}

// Halo rows for one peer: out[i] = raw row of block send_idx[i], or zeros when this worker did
// not touch the block this step (the reference skips such rows, pipeline.py:1183-1186).
__global__ void __launch_bounds__(256) pack_halo_kernel(const float4 *__restrict__ raw,
                                                        const uint8_t *__restrict__ touched,
                                                        const int *__restrict__ send_idx, int n,
                                                        float4 *__restrict__ out)
{
    pdl_wait();
    pdl_launch_dependents();
    const int i = blockIdx.x * 4 + (threadIdx.x >> 6);
    const int slot = threadIdx.x & 63;
    if (i >= n) return;
    const int b = send_idx[i];
    out[(size_t)i * 64 + slot] = touched[b] ? raw[(size_t)b * 64 + slot] : make_float4(0.f, 0.f, 0.f, 0.f);
}

__global__ void signal_step_kernel(int *word, int value, const DevGuard guard)
{
    pdl_wait();
    pdl_launch_dependents();
    if (guarded_out(guard)) return;
    // everything enqueued before this kernel on the stream has completed; make it visible to the
    // peers before the word they poll changes
    __threadfence_system();
    asm volatile("st.release.sys.global.s32 [%0], %1;" :: "l"(word), "r"(value) : "memory");
}

struct WaitArgs {
    int n_wait, wait_value, wait_timeout_ms;
    const int *wait_flags[MPM_MAX_PEERS];
    int *wait_error;
};
// the step barrier alone (a rank whose block table is empty has no grid update to hang it on)
__global__ void wait_step_kernel(const WaitArgs a, const DevGuard guard)
{
    pdl_wait();
    pdl_launch_dependents();
    if (guarded_out(guard)) return;
    if (threadIdx.x < a.n_wait) {
        const int *flag = a.wait_flags[threadIdx.x];
        const unsigned long long t0 = global_timer_ns();
        const unsigned long long limit = (unsigned long long)a.wait_timeout_ms * 1000000ull;
        while (ld_acquire_sys(flag) < a.wait_value) {
            if (guard.word && ld_acquire_sys(guard.word) < guard.step) break;   // void step (see grid_update_kernel)
            if (global_timer_ns() - t0 > limit) {
                if (a.wait_error) atomicExch(a.wait_error, 1);
                break;
            }
            __nanosleep(200);
        }
    }
}

__global__ void status_publish_kernel(const mpm_step_status *src, mpm_step_status *dst, const int *guard_src,
                                      int *guard_dst)
{
    pdl_wait();
    pdl_launch_dependents();
    publish_status(src, dst, guard_src, guard_dst, threadIdx.x);
}

__global__ void status_reset_kernel(mpm_step_status *status, const DevGuard guard)
{
    pdl_wait();
    pdl_launch_dependents();
    if (guarded_out(guard)) return;
    status->zone_violation = 0;
    status->vmax2_bits = 0;
}

}  // namespace mpm

using namespace mpm;

extern "C" {

int mpm_clear(float *raw, uint8_t *touched, int32_t count, int full, int32_t node_bytes,
              const mpm_guard *guard, void *stream)
{
    if (count <= 0) return MPM_OK;
    if (node_bytes != 16 && node_bytes != 32) return MPM_ERR_REJECTED_INPUT;
    launch_chained(clear_kernel, (count + 3) / 4, 256, (cudaStream_t)stream, (float4 *)raw, touched, count,
                   (const int *)nullptr, full, node_bytes / 16, make_guard(guard));
    return check_launch("mpm_clear", 1);
}

}  // extern "C"

namespace mpm {
// mpm_clear with the row count on the device (`bound` sizes the launch)
int clear_rows_dev(float *raw, uint8_t *touched, int32_t bound, const int32_t *count_dev, int full,
                   int32_t node_bytes, const mpm_guard *guard, cudaStream_t stream)
{
    if (bound <= 0) return MPM_OK;
    launch_chained(clear_kernel, (bound + 3) / 4, 256, stream, (float4 *)raw, touched, bound, count_dev, full,
                   node_bytes / 16, make_guard(guard));
    return check_launch("mpm_clear", 1);
}
}  // namespace mpm

extern "C" {

int mpm_status_reset(mpm_step_status *status, const mpm_guard *guard, void *stream)
{
    launch_chained(status_reset_kernel, 1, 1, (cudaStream_t)stream, status, make_guard(guard));
    return check_launch("mpm_status_reset", 1);
}

int mpm_status_publish(const mpm_step_status *src, mpm_step_status *dst_mapped, const int32_t *guard_src,
                       int32_t *guard_dst_mapped, void *stream)
{
    if ((dst_mapped && !src) || (guard_dst_mapped && !guard_src)) return MPM_ERR_REJECTED_INPUT;
    if (!dst_mapped && !guard_dst_mapped) return MPM_OK;
    launch_chained(status_publish_kernel, 1, 32, (cudaStream_t)stream, src, dst_mapped, guard_src, guard_dst_mapped);
    return check_launch("mpm_status_publish", 1);
}

int mpm_grid_update(float *raw, uint8_t *touched, float *vel, float *vel_old,
                    const mpm_table_view *table, const mpm_grid_params *p,
                    mpm_step_status *reset_status, const mpm_guard *guard, void *stream)
{
    if (!table || !p) return MPM_ERR_REJECTED_INPUT;
    if (p->n_peers < 0 || p->n_peers > MPM_MAX_PEERS) return MPM_ERR_CONFIG;
    if (p->fuse_clear && p->n_peers > 0) return MPM_ERR_MODE_CONFLICT;
    if (p->block_filter < 0 || p->block_filter > 2) return MPM_ERR_CONFIG;
    if (table->count <= 0) return MPM_OK;
    GridArgs a;
    a.raw = (const float4 *)raw;
    a.touched = touched;
    a.vel = (float4 *)vel;
    a.vel_old = (float4 *)vel_old;
    a.origin = (const int4 *)table->origin;
    a.count = table->count;
    a.count_dev = table->count_dev;
    a.peers.n = p->n_peers;
    for (int k = 0; k < p->n_peers; ++k) {
        a.peers.raw[k] = (const float4 *)p->peer_raw[k];
        a.peers.touched[k] = p->peer_touched[k];
        a.peers.map[k] = p->peer_map[k];
    }
    a.dt = (float)p->dt;
    a.gx = (float)p->gravity[0]; a.gy = (float)p->gravity[1]; a.gz = (float)p->gravity[2];
    a.apply_bc = p->apply_bc;
    a.bc_sticky = p->bc_sticky;
    for (int k = 0; k < 3; ++k) {
        a.blo[k] = p->apply_bc ? p->box_lo[k] : -1e30;
        a.bhi[k] = p->apply_bc ? p->box_hi[k] : 1e30;
    }
    a.dx = p->dx;
    a.fuse_clear = p->fuse_clear;
    a.block_filter = p->block_filter;
    a.deterministic = p->deterministic;
    a.raw_mut = (float4 *)raw;
    a.touched_mut = touched;
    a.guard = make_guard(guard);
    a.reset_status = reset_status;
    if (p->n_wait < 0 || p->n_wait > MPM_MAX_PEERS) return MPM_ERR_CONFIG;
    a.n_wait = p->n_wait;
    a.wait_value = p->wait_value;
    a.wait_timeout_ms = p->wait_timeout_ms > 0 ? p->wait_timeout_ms : 10000;
    for (int k = 0; k < MPM_MAX_PEERS; ++k) a.wait_flags[k] = k < p->n_wait ? p->wait_flags[k] : nullptr;
    a.wait_error = p->wait_error;
    if ((p->publish_dst && !p->publish_src) || (p->publish_guard_dst && !p->publish_guard_src))
        return MPM_ERR_REJECTED_INPUT;
    a.publish_src = p->publish_src;
    a.publish_dst = p->publish_dst;
    a.publish_guard_src = p->publish_guard_src;
    a.publish_guard_dst = p->publish_guard_dst;
    a.clock = p->clock;
    a.clock_step = p->clock_step;
    a.vmax_ring = p->vmax_ring;
    a.vmax_ring_len = p->vmax_ring_len;
    a.clock_status = p->clock_status;
    a.frame_dt = p->frame_dt; a.cfl_dx = p->cfl_dx; a.c_sound = p->c_sound;
    a.prof = p->prof;
    a.n_vmax_peers = p->clock ? p->n_vmax_peers : 0;
    if (p->clock && (!p->vmax_ring || p->vmax_ring_len < 3 || !(p->frame_dt > 0.0) ||
                     a.n_vmax_peers < 0 || a.n_vmax_peers > MPM_MAX_PEERS))
        return MPM_ERR_REJECTED_INPUT;
    for (int k = 0; k < MPM_MAX_PEERS; ++k) a.vmax_peer_rings[k] = k < a.n_vmax_peers ? p->vmax_peer_rings[k] : nullptr;
    launch_chained(grid_update_kernel, (a.count + 3) / 4, 256, (cudaStream_t)stream, a);
    return check_launch("mpm_grid_update", 1);
}

int mpm_signal_step(int32_t *word, int32_t value, const mpm_guard *guard, void *stream)
{
    if (!word) return MPM_ERR_REJECTED_INPUT;
    launch_chained(signal_step_kernel, 1, 1, (cudaStream_t)stream, word, value, make_guard(guard));
    return check_launch("mpm_signal_step", 1);
}

int mpm_wait_step(const mpm_grid_params *p, const mpm_guard *guard, void *stream)
{
    if (!p || p->n_wait < 0 || p->n_wait > MPM_MAX_PEERS) return MPM_ERR_REJECTED_INPUT;
    if (p->n_wait == 0) return MPM_OK;
    WaitArgs a;
    a.n_wait = p->n_wait;
    a.wait_value = p->wait_value;
    a.wait_timeout_ms = p->wait_timeout_ms > 0 ? p->wait_timeout_ms : 10000;
    for (int k = 0; k < MPM_MAX_PEERS; ++k) a.wait_flags[k] = k < p->n_wait ? p->wait_flags[k] : nullptr;
    a.wait_error = p->wait_error;
    launch_chained(wait_step_kernel, 1, 32, (cudaStream_t)stream, a, make_guard(guard));
    return check_launch("mpm_wait_step", 1);
}

int mpm_pack_halo(const float *raw, const uint8_t *touched, const int32_t *send_idx, int32_t n,
                  float *out_rows, void *stream)
{
    if (n <= 0) return MPM_OK;
    launch_chained(pack_halo_kernel, (n + 3) / 4, 256, (cudaStream_t)stream, (const float4 *)raw, touched, send_idx, n,
                                                                    (float4 *)out_rows);
    return check_launch("mpm_pack_halo", 1);
}

int mpm_particle_aggregates(const mpm_store_view *store, double *out5, void *stream_)
{
    cudaStream_t stream = (cudaStream_t)stream_;
    cudaMemsetAsync(out5, 0, 5 * sizeof(double), stream);
    const int G = store->n_groups;
    if (G > 0)
        launch_chained(particle_aggregates_kernel, (int)(((int64_t)G * 32 + 255) / 256), 256, stream, 
            store->data, store->nch, store->group_len, G, out5);
    return check_launch("mpm_particle_aggregates", 1);
}

int mpm_grid_aggregates(const float *raw, const uint8_t *touched, int32_t count, int32_t deterministic,
                        double *out4, void *stream_)
{
    cudaStream_t stream = (cudaStream_t)stream_;
    cudaMemsetAsync(out4, 0, 4 * sizeof(double), stream);
    if (count > 0)
        launch_chained(grid_aggregates_kernel, (count + 3) / 4, 256, stream, (const float4 *)raw, touched, count,
                                                                  deterministic, out4);
    return check_launch("mpm_grid_aggregates", 1);
}

}  // extern "C"
