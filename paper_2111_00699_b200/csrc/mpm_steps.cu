// Batched enqueue of guarded substeps: the host side of Worker.run_frame's inner loop
// (pipeline.py:872-876 + run_step :905-940, no-rebuild path) for a single worker, issued from C
// so that small scenes are not bound by per-launch interpreter overhead.
//
// For every step s in [first_step, first_step + n_steps):
//   fused (transfer = g2p2g):  [clear(par)] -> g2p2g(s) -> grid update(s), which also stores status
//                              slot s % ring to pinned host memory through its device alias -> event
//   split:                     [clear(par)] -> p2g(s) -> grid update(s) -> g2p(s) -> status
//                              publication (one-warp kernel) -> event
// The status never goes through cudaMemcpyAsync when the host ring is mapped: a kernel -> copy ->
// kernel chain idles the device for a copy-engine round trip per step (measured ~20 us of a
// 280 us step at 1.37 M particles, and the same 20 us of a 30 us step at 64 K).
// All kernels carry the guard {word, s}: once a gather raises the word to its step, every later
// step of the batch is a no-op on the device and the host re-issues from there after rebuilding.
#include "mpm_common.cuh"

namespace mpm {
int clear_rows_dev(float *raw, uint8_t *touched, int32_t bound, const int32_t *count_dev, int full,
                   int32_t node_bytes, const mpm_guard *guard, cudaStream_t stream);
}

extern "C" int mpm_enqueue_steps(const mpm_step_plan *p, int32_t first_step, int32_t n_steps, void *stream_)
{
    if (!p || n_steps < 0 || n_steps > MPM_MAX_STATUS_RING) return MPM_ERR_REJECTED_INPUT;
    if (p->status_ring < 2 || p->status_ring > MPM_MAX_STATUS_RING) return MPM_ERR_CONFIG;
    if (!p->guard_word || !p->status_dev || !p->status_host) return MPM_ERR_REJECTED_INPUT;
    cudaStream_t stream = (cudaStream_t)stream_;
    mpm_transfer_params tp = p->transfer;
    mpm_grid_params gp = p->grid;
    // device aliases of the pinned host rings; without them (memory not mapped) or without a
    // grid update to carry them (empty table) the slots are copied as before
    mpm_step_status *status_alias = nullptr;
    int32_t *guard_alias = nullptr;
    bool mapped = cudaHostGetDevicePointer((void **)&status_alias, p->status_host, 0) == cudaSuccess &&
                  (!p->guard_host ||
                   cudaHostGetDevicePointer((void **)&guard_alias, p->guard_host, 0) == cudaSuccess);
    if (!mapped) (void)cudaGetLastError();
    const bool in_update = mapped && p->table.count > 0;
    for (int k = 0; k < n_steps; ++k) {
        const int s = first_step + k;
        const int slot = s % p->status_ring;
        const int par = s & 1;
        mpm_guard guard;
        guard.first_bad_step = p->guard_word;
        guard.step = s;
        guard.n_peer_words = p->n_peer_words;
        for (int q = 0; q < MPM_MAX_PEERS; ++q) guard.peer_words[q] = p->peer_guard_words[q];
        if (gp.n_wait > 0) gp.wait_value = s + 1;
        if (gp.clock) {
            // CFL-auto frame: every kernel of the step reads its dt from the device clock; the
            // update of step s also sets the size of step s + 1 and reports dt_s / the frame end
            // in the step's status block
            gp.clock_step = s;
            gp.clock_status = p->status_dev + slot;
            tp.clock = gp.clock;
            tp.clock_step = s;
            tp.clock_gather_step = s;      // split G2P: the update of the same step
        } else {
            tp.clock = nullptr;
        }
        if (p->signal_word)
            for (int q = 0; q < gp.n_peers; ++q) {
                gp.peer_raw[q] = p->peer_raw[par][q];
                gp.peer_touched[q] = p->peer_touched[par][q];
            }
        mpm_step_status *st_dev = p->status_dev + slot;
        int rc;
        // after the first step of a batch the gather dt is the batch's own dt (pipeline.py:1230)
        if (k > 0) tp.dt_gather = tp.dt;
        if (k == 0 && p->full_clear_first) {
            // first use of the parity the last rebuild left untouched: every row, not only the
            // touched ones (pipeline.py:1022-1037)
            rc = mpm::clear_rows_dev(p->raw[par], p->touched[par], p->table.count, p->table.count_dev, 1,
                                     gp.deterministic ? 32 : 16, &guard, stream);
            if (rc != MPM_OK) return rc;
        } else if (!gp.fuse_clear) {
            // Worker._clear (pipeline.py:1022-1037): rows of this parity touched two steps ago
            rc = mpm::clear_rows_dev(p->raw[par], p->touched[par], p->table.count, p->table.count_dev, 0,
                                     gp.deterministic ? 32 : 16, &guard, stream);
            if (rc != MPM_OK) return rc;
        }
        if (p->fused) {
            mpm_transfer_params fp = tp;
            fp.margin_lo = p->fused_margin_lo;
            fp.margin_hi = p->fused_margin_hi;
            fp.clock_gather_step = s - 1;  // the fused gather completes the previous step
            if (p->time_events[2 * k]) cudaEventRecord((cudaEvent_t)p->time_events[2 * k], stream);
            rc = mpm_g2p2g(&p->store, &p->table, p->vel, p->vel_old, p->raw[par], p->touched[par], &fp,
                           st_dev, &guard, stream);
            if (rc != MPM_OK) return rc;
            if (p->time_events[2 * k + 1]) cudaEventRecord((cudaEvent_t)p->time_events[2 * k + 1], stream);
            if (p->signal_word) {
                rc = mpm_signal_step(p->signal_word, s + 1, &guard, stream);
                if (rc != MPM_OK) return rc;
            }
            if (in_update) {
                gp.publish_src = st_dev;
                gp.publish_dst = status_alias + slot;
                gp.publish_guard_src = p->guard_host ? p->guard_word : nullptr;
                gp.publish_guard_dst = p->guard_host ? guard_alias + slot : nullptr;
            } else {
                cudaMemcpyAsync(p->status_host + slot, st_dev, sizeof(mpm_step_status), cudaMemcpyDeviceToHost, stream);
                if (p->guard_host)
                    cudaMemcpyAsync(p->guard_host + slot, p->guard_word, sizeof(int32_t), cudaMemcpyDeviceToHost, stream);
                cudaEventRecord((cudaEvent_t)p->events[slot], stream);
            }
            rc = mpm_grid_update(p->raw[par], p->touched[par], p->vel, p->vel_old, &p->table, &gp,
                                 p->status_dev + (s + 1) % p->status_ring, &guard, stream);
            if (rc != MPM_OK) return rc;
            if (in_update) cudaEventRecord((cudaEvent_t)p->events[slot], stream);
        } else {
            if (p->time_events[2 * k]) cudaEventRecord((cudaEvent_t)p->time_events[2 * k], stream);
            rc = mpm_p2g(&p->store, &p->table, p->raw[par], p->touched[par], &tp, st_dev, &guard, stream);
            if (rc != MPM_OK) return rc;
            if (p->time_events[2 * k + 1]) cudaEventRecord((cudaEvent_t)p->time_events[2 * k + 1], stream);
            if (p->signal_word) {
                rc = mpm_signal_step(p->signal_word, s + 1, &guard, stream);
                if (rc != MPM_OK) return rc;
            }
            rc = mpm_grid_update(p->raw[par], p->touched[par], p->vel, p->vel_old, &p->table, &gp, st_dev,
                                 &guard, stream);
            if (rc != MPM_OK) return rc;
            mpm_transfer_params g2 = tp;
            g2.dt_gather = tp.dt;            // split G2P advects with the dt of the update just done
            rc = mpm_g2p(&p->store, &p->table, p->vel, p->vel_old, &g2, st_dev, &guard, stream);
            if (rc != MPM_OK) return rc;
            if (mapped) {
                rc = mpm_status_publish(st_dev, status_alias + slot, p->guard_host ? p->guard_word : nullptr,
                                        p->guard_host ? guard_alias + slot : nullptr, stream);
                if (rc != MPM_OK) return rc;
            } else {
                cudaMemcpyAsync(p->status_host + slot, st_dev, sizeof(mpm_step_status), cudaMemcpyDeviceToHost, stream);
                if (p->guard_host)
                    cudaMemcpyAsync(p->guard_host + slot, p->guard_word, sizeof(int32_t), cudaMemcpyDeviceToHost, stream);
            }
            cudaEventRecord((cudaEvent_t)p->events[slot], stream);
        }
    }
    return mpm::check_launch("mpm_enqueue_steps", 0);
}
