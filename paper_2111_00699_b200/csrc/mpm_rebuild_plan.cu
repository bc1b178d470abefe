// Worker._rebuild (pipeline.py:958-1015) as ONE call: the eight rebuild-mapping entry points of
// mpm_rebuild.cu issued back to back from C with the two host syncs of the paper's rebuild
// (block count, then pblock + group counts) taken here.  The interpreter is off
// the path between the syncs: at 64 K particles a rebuild every 5-8 steps cost ~0.3 ms of host
// time (the device idle meanwhile) against ~0.1 ms of kernels.
//
// Ownership is unchanged: every buffer belongs to the caller, who states its capacities.  When a
// count outgrows a capacity the call returns MPM_NEED_CAPACITY with the sizes it needs; nothing
// the caller still uses has been overwritten (the old store is read-only here), so it grows the
// buffers (4x rule, memory.py:18-22) and calls again.
#include "mpm_common.cuh"

namespace {

int read_scalars(const mpm_rebuild_plan *p, cudaStream_t stream)
{
    cudaMemcpyAsync(p->scalars_host, p->scalars_dev, 16 * sizeof(int32_t), cudaMemcpyDeviceToHost, stream);
    cudaError_t e = cudaStreamSynchronize(stream);
    if (e != cudaSuccess) {
        mpm::set_last_error("mpm_rebuild", e);
        return MPM_ERR_RESOURCE;
    }
    return MPM_OK;
}

}  // namespace

extern "C" int mpm_rebuild(const mpm_rebuild_plan *p, mpm_rebuild_result *r, void *stream_)
{
    if (!p || !r || !p->scalars_dev || !p->scalars_host) return MPM_ERR_REJECTED_INPUT;
    if (p->hash_cap <= 0 || (p->hash_cap & (p->hash_cap - 1))) return MPM_ERR_CONFIG;
    cudaStream_t stream = (cudaStream_t)stream_;
    int32_t *S = p->scalars_dev;   // 0 n_live, 1 n_total, 2 bad_index, 3 n_gblocks, 4 overflow, 5 count,
                                   // 6 bad_block, 7 n_groups (the slots Worker._rebuild uses)
    const int32_t *H = p->scalars_host;
    memset(r, 0, sizeof *r);
    r->bad_particle = r->bad_block = MPM_INT_MAX;
    const float *staged = p->n_staged ? p->staged : nullptr;
    const int64_t *staged_ids = p->n_staged ? p->staged_ids : nullptr;
    int rc;
    if (p->guard_word) {
        rc = mpm_fill_i32(p->guard_word, 1, MPM_INT_MAX, stream);
        if (rc != MPM_OK) return rc;
    }

    // ---- particles -> codes -> gblocks (first sync: block count) ----------------------------
    rc = mpm_compact_live(&p->old_store, 1, p->glive, p->src_slot, S + 0, p->scan, stream);
    if (rc != MPM_OK) return rc;
    rc = mpm_particle_codes(&p->old_store, p->src_slot, S + 0, staged, p->n_staged, p->n_upper, p->dx,
                            p->codes, S + 1, S + 2, stream);
    if (rc != MPM_OK) return rc;
    rc = mpm_hash_insert_blocks(p->codes, S + 1, p->n_upper, p->hkeys, p->hvals, p->hfirst, p->hash_cap,
                                p->pslot, p->flag, p->scan, p->gidx, p->gcodes, S + 3, S + 4, stream);
    if (rc != MPM_OK) return rc;
    rc = read_scalars(p, stream);
    if (rc != MPM_OK) return rc;
    r->n = H[1];
    r->bad_particle = H[2];
    r->n_gblocks = H[3];
    if (r->bad_particle != MPM_INT_MAX) return MPM_ERR_SPATIAL_DOMAIN;
    const int n_g = r->n_gblocks;
    if (H[4] || 8ll * n_g > p->hash_cap) r->need_hash = 1;
    if (n_g > p->cap_gblocks) r->need_gblocks = n_g;
    if (27ll * n_g > p->cap_table) r->need_table = 27 * n_g;       // worst case of the dilation
    if (r->need_hash || r->need_gblocks || r->need_table) return MPM_NEED_CAPACITY;

    // ---- dilation, sort, groups (second sync: pblock and group counts) ----------------------
    rc = mpm_dilate_and_link(p->gcodes, n_g, p->hkeys, p->hvals, p->hfirst, p->hash_cap, p->qslot, p->qflag,
                             p->scan, p->table_codes, p->table_origin, p->table_neighbor, p->cap_table,
                             S + 5, S + 6, S + 4, stream);
    if (rc != MPM_OK) return rc;
    rc = mpm_sort_and_group(p->codes, p->gidx, S + 1, p->n_upper, n_g, p->bin_start, p->tmp_perm, p->perm,
                            p->bgf, p->scan, S + 7, p->pslot, p->flag, stream);   // pslot / flag are free by now
    if (rc != MPM_OK) return rc;
    rc = read_scalars(p, stream);
    if (rc != MPM_OK) return rc;
    r->count = H[5];
    r->bad_block = H[6];
    r->n_groups = H[7];
    if (r->bad_block != MPM_INT_MAX) return MPM_ERR_SPATIAL_DOMAIN;
    if (H[4] == 1) {               // the halo did not fit the hash table
        r->need_hash = 1;
        return MPM_NEED_CAPACITY;
    }
    if (r->n_groups > p->cap_groups) r->need_groups = r->n_groups;
    if (r->count > p->cap_nodes) r->need_nodes = r->count;
    if (r->need_groups || r->need_nodes) return MPM_NEED_CAPACITY;

    // ---- permute the particles into the new store, reset the nodal buffers ------------------
    mpm_store_view ns = p->new_store;
    ns.n_groups = r->n_groups;
    rc = mpm_scatter_sorted(&p->old_store, p->src_slot, S + 0, staged, staged_ids, p->perm, p->bin_start,
                            p->bgf, n_g, p->table_origin, p->dx, &ns, stream);
    if (rc != MPM_OK) return rc;
    if (r->n_groups > 0) {
        mpm_table_view tv;
        memset(&tv, 0, sizeof tv);
        tv.codes = p->table_codes;
        tv.origin = p->table_origin;
        tv.neighbor = p->table_neighbor;
        tv.count = r->count;
        tv.n_gblocks = n_g;
        rc = mpm_build_group_ctx(&ns, &tv, stream);
        if (rc != MPM_OK) return rc;
    }
    if (r->count > 0) {
        // pipeline.py:996-1006: vel and raw[par] start from zero (raw[1 - par] is cleared in full at
        // its next use)
        if (p->vel) cudaMemsetAsync(p->vel, 0, (size_t)r->count * 64 * 16, stream);
        rc = mpm_clear(p->raw_par, p->touched_par, r->count, 1, p->node_bytes, nullptr, stream);
        if (rc != MPM_OK) return rc;
    }
    if (p->p2g_params && p->grid_params && r->count > 0) {
        // the rest of the rebuild step: P2G of the new store, then reduce + update
        mpm_table_view tv;
        memset(&tv, 0, sizeof tv);
        tv.codes = p->table_codes;
        tv.origin = p->table_origin;
        tv.neighbor = p->table_neighbor;
        tv.count = r->count;
        tv.n_gblocks = n_g;
        if (r->n_groups > 0) {
            rc = mpm_p2g(&ns, &tv, p->raw_par, p->touched_par, p->p2g_params, p->p2g_status, nullptr, stream);
            if (rc != MPM_OK) return rc;
        }
        rc = mpm_grid_update(p->raw_par, p->touched_par, p->vel, p->vel_old, &tv, p->grid_params,
                             p->grid_reset_status, nullptr, stream);
        if (rc != MPM_OK) return rc;
        r->tail_done = 1;
    }
    return mpm::check_launch("mpm_rebuild", 0);
}
