// Worker._rebuild (pipeline.py:958-1015) as ONE call without a host round trip inside it.
//
// The paper's rebuild takes two CPU-GPU sync points (block count, then pblock + group counts;
// PAPER.md:141) because the host sizes the next launches from them.  Here every launch is sized by
// the caller's CAPACITIES and the kernels read the counts from device memory, so the whole chain
//     compact -> codes -> hash insert -> dilate -> sort -> groups -> permute -> group context ->
//     nodal resets [-> P2G -> grid update [-> G2P] [-> first batch of steady steps]]
// is enqueued in one go.  The scalars are copied to pinned host memory right behind the sort and an
// event is recorded there: the host waits for THAT (mpm_rebuild_wait) while the permutation, the rest
// of the rebuild step and the next batch keep the device busy; its bookkeeping of the new tables
// overlaps them.  At 64 K particles (a rebuild every 5-8 steps) the two waits and the interpreter
// around them cost ~140 us per rebuild against ~100 us of kernels.
//
// Ownership is unchanged: every buffer belongs to the caller, who states its capacities.  A count
// that outgrows one aborts the chain on the device (rebuild_check_*: the counts later kernels read
// are zeroed, the guard of everything enqueued behind is lowered) and mpm_rebuild_wait answers
// MPM_NEED_CAPACITY with the sizes needed; the old store is read-only here, so the caller grows
// the buffers (4x rule, memory.py:18-22) and calls again.
#include "mpm_common.cuh"

namespace mpm {
void rebuild_init(int32_t *S, int32_t *large_list, int32_t *guard_word, cudaStream_t stream);
void zero_rows(float *rows, const int32_t *count_dev, int bound, cudaStream_t stream);
int rebuild_chain(const mpm_rebuild_plan *p, int32_t *S, int gblocks_bound, int groups_bound, cudaStream_t stream);
int clear_rows_dev(float *raw, uint8_t *touched, int32_t bound, const int32_t *count_dev, int full,
                   int32_t node_bytes, const mpm_guard *guard, cudaStream_t stream);
}  // namespace mpm

extern "C" int mpm_rebuild_wait(const mpm_rebuild_plan *p, mpm_rebuild_result *r)
{
    if (!p || !r || !p->scalars_host) return MPM_ERR_REJECTED_INPUT;
    if (p->done_event) {
        cudaError_t e = cudaEventSynchronize((cudaEvent_t)p->done_event);
        if (e != cudaSuccess) {
            mpm::set_last_error("mpm_rebuild_wait", e);
            return MPM_ERR_RESOURCE;
        }
    }
    // 0 n_live, 1 n_total, 2 bad particle, 3 n_gblocks, 4 hash overflow, 5 count, 6 bad block, 7 n_groups,
    // 8 abort mask, 9..12 needed gblocks / table entries / groups / nodes
    const int32_t *H = p->scalars_host;
    const int32_t tail = r->tail_done, g2p = r->g2p_done, next = r->next_done;
    memset(r, 0, sizeof *r);
    r->tail_done = tail; r->g2p_done = g2p; r->next_done = next;
    r->bad_particle = H[2];
    r->bad_block = H[6];
    const int why = H[8];
    if (why & (8 | 16)) return MPM_ERR_SPATIAL_DOMAIN;
    r->bad_particle = r->bad_block = MPM_INT_MAX;
    if (why) {
        r->need_hash = (why & 1) ? 1 : 0;
        r->need_gblocks = H[9];
        r->need_table = H[10];
        r->need_groups = H[11];
        r->need_nodes = H[12];
        r->tail_done = r->g2p_done = r->next_done = 0;      // they ran as no-ops
        return MPM_NEED_CAPACITY;
    }
    r->n = H[1];
    r->n_gblocks = H[3];
    r->count = H[5];
    r->n_groups = H[7];
    return MPM_OK;
}

extern "C" int mpm_rebuild(const mpm_rebuild_plan *p, mpm_rebuild_result *r, void *stream_)
{
    if (!p || !r || !p->scalars_dev || !p->scalars_host || !p->large_list) return MPM_ERR_REJECTED_INPUT;
    if (p->hash_cap <= 0 || (p->hash_cap & (p->hash_cap - 1))) return MPM_ERR_CONFIG;
    if (p->async && !p->done_event) return MPM_ERR_REJECTED_INPUT;
    cudaStream_t stream = (cudaStream_t)stream_;
    int32_t *S = p->scalars_dev;
    memset(r, 0, sizeof *r);
    r->bad_particle = r->bad_block = MPM_INT_MAX;

    // launch bounds from the caller's capacities
    const int gblocks_bound = p->cap_gblocks < p->cap_table / 27 ? p->cap_gblocks : p->cap_table / 27;
    long long gb = (long long)p->n_upper / 32 + gblocks_bound + 1;     // n_groups <= n / 32 + n_g
    const int groups_bound = (int)(gb < p->cap_groups ? gb : p->cap_groups);
    const int nodes_bound = p->cap_nodes < p->cap_table ? p->cap_nodes : p->cap_table;
    if (gblocks_bound <= 0 || groups_bound <= 0 || nodes_bound <= 0) {
        // nothing fits: the first guess the caller should size for
        r->need_gblocks = 1; r->need_table = 27; r->need_groups = p->n_upper / 32 + 2; r->need_nodes = 27;
        return MPM_NEED_CAPACITY;
    }

    mpm::rebuild_init(S, p->large_list, p->guard_word, stream);
    int rc = mpm::rebuild_chain(p, S, gblocks_bound, groups_bound, stream);
    if (rc != MPM_OK) return rc;

    // the counts, to the host: everything below keeps the device busy while the host waits for them
    cudaMemcpyAsync(p->scalars_host, S, 16 * sizeof(int32_t), cudaMemcpyDeviceToHost, stream);
    if (p->done_event) cudaEventRecord((cudaEvent_t)p->done_event, stream);

    mpm_store_view ns = p->new_store;
    ns.n_groups = groups_bound;
    ns.n_groups_dev = S + 7;
    mpm_table_view tv;
    memset(&tv, 0, sizeof tv);
    tv.codes = p->table_codes;
    tv.origin = p->table_origin;
    tv.neighbor = p->table_neighbor;
    tv.count = nodes_bound;
    tv.count_dev = S + 5;
    tv.n_gblocks = gblocks_bound;
    rc = mpm_build_group_ctx(&ns, &tv, stream);
    if (rc != MPM_OK) return rc;
    // pipeline.py:996-1006: vel and raw[par] start from zero (raw[1 - par] is cleared in full at its
    // next use)
    if (p->vel) mpm::zero_rows(p->vel, S + 5, nodes_bound, stream);
    rc = mpm::clear_rows_dev(p->raw_par, p->touched_par, nodes_bound, S + 5, 1, p->node_bytes, nullptr, stream);
    if (rc != MPM_OK) return rc;

    if (p->p2g_params && p->grid_params) {
        // the rest of the rebuild step: P2G of the new store, then reduce + update (+ split gather)
        mpm_guard guard;
        memset(&guard, 0, sizeof guard);
        guard.first_bad_step = p->guard_word;
        guard.step = p->guard_step;
        const mpm_guard *g = p->guard_word ? &guard : nullptr;
        rc = mpm_p2g(&ns, &tv, p->raw_par, p->touched_par, p->p2g_params, p->p2g_status, g, stream);
        if (rc != MPM_OK) return rc;
        rc = mpm_grid_update(p->raw_par, p->touched_par, p->vel, p->vel_old, &tv, p->grid_params,
                             p->grid_reset_status, g, stream);
        if (rc != MPM_OK) return rc;
        r->tail_done = 1;
        if (p->g2p_params && p->g2p_status) {
            rc = mpm_g2p(&ns, &tv, p->vel, p->vel_old, p->g2p_params, p->g2p_status, g, stream);
            if (rc != MPM_OK) return rc;
            if (p->status_publish_dst) {
                rc = mpm_status_publish(p->g2p_status, p->status_publish_dst, nullptr, nullptr, stream);
                if (rc != MPM_OK) return rc;
            }
            if (p->status_event) cudaEventRecord((cudaEvent_t)p->status_event, stream);
            r->g2p_done = 1;
        }
        if (p->next_steps && p->next_n_steps > 0) {
            mpm_step_plan sp = *p->next_steps;
            sp.store = ns;
            sp.table = tv;
            sp.table.touched[0] = sp.touched[0];
            sp.table.touched[1] = sp.touched[1];
            rc = mpm_enqueue_steps(&sp, p->next_first_step, p->next_n_steps, stream);
            if (rc != MPM_OK) return rc;
            r->next_done = p->next_n_steps;
        }
    }
    rc = mpm::check_launch("mpm_rebuild", 0);
    if (rc != MPM_OK) return rc;
    if (p->async) return MPM_OK;
    if (!p->done_event) {
        cudaError_t e = cudaStreamSynchronize(stream);
        if (e != cudaSuccess) {
            mpm::set_last_error("mpm_rebuild", e);
            return MPM_ERR_RESOURCE;
        }
    }
    return mpm_rebuild_wait(p, r);
}
