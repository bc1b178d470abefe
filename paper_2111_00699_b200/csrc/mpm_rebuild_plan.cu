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
#include <stdlib.h>
#include <string.h>

#include <mutex>

#include "mpm_common.cuh"

namespace mpm {
void rebuild_init(int32_t *S, int32_t *large_list, int32_t *guard_word, cudaStream_t stream);
void zero_rows(float *rows, const int32_t *count_dev, int bound, cudaStream_t stream);
int rebuild_chain(const mpm_rebuild_plan *p, int32_t *S, int gblocks_bound, int groups_bound, cudaStream_t stream);
int clear_rows_dev(float *raw, uint8_t *touched, int32_t bound, const int32_t *count_dev, int full,
                   int32_t node_bytes, const mpm_guard *guard, cudaStream_t stream);
}  // namespace mpm

// ---------------------------------------------------------------------------------------------------
// The rebuild kernels as a CUDA graph.  Nothing in the chain depends on a host-side count any more
// (launches sized by capacities, counts read on the device, the old store's group count included),
// so a rebuild whose buffers, capacities and particle count equal an earlier one's enqueues the very
// same ~35 launches -- and is replayed with ONE cudaGraphLaunch.  At 64 K particles (a rebuild every
// 5-6 steps) launching the chain kernel by kernel costs ~120 us of host time per rebuild against
// ~70 us of device time: the host was the bound.  The rest of the rebuild step (P2G, grid update,
// the first batch of steady steps) depends on the step number and stays out of the graph.
// ---------------------------------------------------------------------------------------------------
namespace mpm {
namespace {
struct GraphEntry {
    mpm_rebuild_plan key;       // the plan with every field the chain does not read zeroed
    int bounds[3];
    cudaGraphExec_t exec;
    unsigned long long kernels; // launches one replay stands for (mpm_launch_count)
    unsigned long long stamp;
};
constexpr int GRAPH_SLOTS = 32;     // four per logical worker in steady state (store parity x grid parity)
GraphEntry g_graphs[GRAPH_SLOTS];
int g_n_graphs = 0;
unsigned long long g_graph_stamp = 0;
cudaStream_t g_capture_stream = nullptr;
constexpr int SEEN_SLOTS = 64;
unsigned long long g_seen[SEEN_SLOTS];
unsigned g_seen_next = 0;
int g_graphs_ok = -1;           // -1 not decided, 0 off (MPM_REBUILD_GRAPH=0 or a capture failed), 1 on

bool graphs_enabled()
{
    if (g_graphs_ok < 0) {
        const char *e = getenv("MPM_REBUILD_GRAPH");
        g_graphs_ok = (e && e[0] == '0') ? 0 : 1;
    }
    return g_graphs_ok == 1;
}

void graph_key(const mpm_rebuild_plan *p, mpm_rebuild_plan *k)
{
    memcpy(k, p, sizeof *k);
    k->p2g_params = nullptr; k->p2g_status = nullptr; k->grid_params = nullptr; k->grid_reset_status = nullptr;
    k->vel_old = nullptr; k->guard_step = 0; k->async = 0;
    k->g2p_params = nullptr; k->g2p_status = nullptr; k->status_publish_dst = nullptr; k->status_event = nullptr;
    k->next_steps = nullptr; k->next_first_step = 0; k->next_n_steps = 0;
    k->use_graph = 0; k->reserved1 = 0;
}
}  // namespace

// rebuild proper: every kernel in front of the step-dependent tail
static int enqueue_rebuild_kernels(const mpm_rebuild_plan *p, int32_t *S, int gblocks_bound, int groups_bound,
                                   int nodes_bound, cudaStream_t stream, bool capturing)
{
    rebuild_init(S, p->large_list, p->guard_word, stream);
    int rc = rebuild_chain(p, S, gblocks_bound, groups_bound, stream);
    if (rc != MPM_OK) return rc;
    // the counts, to the host: everything below keeps the device busy while the host waits for them
    cudaMemcpyAsync(p->scalars_host, S, 16 * sizeof(int32_t), cudaMemcpyDeviceToHost, stream);
    // (a graph records the event behind its launch instead: an event-record NODE only turns the event
    // pending when it executes, so a host that waits right after cudaGraphLaunch would find the
    // previous rebuild's recording complete and read stale counts)
    if (p->done_event && !capturing) cudaEventRecord((cudaEvent_t)p->done_event, stream);
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
    if (p->vel) zero_rows(p->vel, S + 5, nodes_bound, stream);
    return clear_rows_dev(p->raw_par, p->touched_par, nodes_bound, S + 5, 1, p->node_bytes, nullptr, stream);
}

// Returns MPM_OK with *how = 1 (captured now) / 2 (replayed), or a negative status / *how = 0 when the
// graph route is not available (the caller then launches kernel by kernel).
static int rebuild_by_graph(const mpm_rebuild_plan *p, int32_t *S, int gblocks_bound, int groups_bound,
                            int nodes_bound, cudaStream_t stream, int *how)
{
    *how = 0;
    // worker handles may be driven from different host threads: the cache and the capture stream are shared
    static std::mutex lock;
    std::lock_guard<std::mutex> hold(lock);
    if (!graphs_enabled() || p->n_staged != 0) return MPM_OK;
    mpm_rebuild_plan key;
    graph_key(p, &key);
    const int bounds[3] = {gblocks_bound, groups_bound, nodes_bound};
    GraphEntry *hit = nullptr;
    for (int i = 0; i < g_n_graphs; ++i)
        if (!memcmp(&g_graphs[i].key, &key, sizeof key) && !memcmp(g_graphs[i].bounds, bounds, sizeof bounds)) {
            hit = &g_graphs[i];
            break;
        }
    if (!hit) {
        // A shape is captured when it comes back (capturing costs about a millisecond): a scene whose
        // particle count changes at every rebuild (sink, emitter) never pays for graphs it would not reuse.
        unsigned long long h = 1469598103934665603ull;
        const unsigned char *kb = (const unsigned char *)&key;
        for (size_t i = 0; i < sizeof key; ++i) h = (h ^ kb[i]) * 1099511628211ull;
        for (int i = 0; i < 3; ++i) h = (h ^ (unsigned)bounds[i]) * 1099511628211ull;
        bool seen = false;
        for (int i = 0; i < SEEN_SLOTS; ++i) seen = seen || g_seen[i] == h;
        if (!seen) {
            g_seen[g_seen_next++ % SEEN_SLOTS] = h;
            return MPM_OK;
        }
        if (!g_capture_stream &&
            cudaStreamCreateWithFlags(&g_capture_stream, cudaStreamNonBlocking) != cudaSuccess) {
            (void)cudaGetLastError();
            g_graphs_ok = 0;
            return MPM_OK;
        }
        cudaGraph_t graph = nullptr;
        cudaGraphExec_t exec = nullptr;
        const unsigned long long before = launch_counter_add(0);
        bool ok = cudaStreamBeginCapture(g_capture_stream, cudaStreamCaptureModeRelaxed) == cudaSuccess;
        int rc = MPM_OK;
        if (ok) {
            g_plain_launch = true;
            rc = enqueue_rebuild_kernels(p, S, gblocks_bound, groups_bound, nodes_bound, g_capture_stream, true);
            g_plain_launch = false;
            ok = cudaStreamEndCapture(g_capture_stream, &graph) == cudaSuccess && graph && rc == MPM_OK;
        }
        const unsigned long long kernels = launch_counter_add(0) - before;
        if (ok) ok = cudaGraphInstantiate(&exec, graph, 0) == cudaSuccess;
        if (graph) cudaGraphDestroy(graph);
        if (!ok) {
            (void)cudaGetLastError();
            g_graphs_ok = 0;             // this driver / chain cannot be captured: kernel by kernel from now on
            launch_counter_add(0ull - kernels);
            return rc < 0 ? rc : MPM_OK;
        }
        launch_counter_add(0ull - kernels);     // counted per replay below
        int slot = g_n_graphs;
        if (g_n_graphs < GRAPH_SLOTS) ++g_n_graphs;
        else {
            slot = 0;
            for (int i = 1; i < GRAPH_SLOTS; ++i) if (g_graphs[i].stamp < g_graphs[slot].stamp) slot = i;
            cudaGraphExecDestroy(g_graphs[slot].exec);
        }
        hit = &g_graphs[slot];
        hit->key = key;
        memcpy(hit->bounds, bounds, sizeof bounds);
        hit->exec = exec;
        hit->kernels = kernels;
        *how = 1;
    } else {
        *how = 2;
    }
    hit->stamp = ++g_graph_stamp;
    if (cudaGraphLaunch(hit->exec, stream) != cudaSuccess) {
        set_last_error("mpm_rebuild (graph launch)", cudaGetLastError());
        return MPM_ERR_RESOURCE;
    }
    launch_counter_add(hit->kernels);
    if (p->done_event) cudaEventRecord((cudaEvent_t)p->done_event, stream);
    return MPM_OK;
}
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
    const int32_t tail = r->tail_done, g2p = r->g2p_done, next = r->next_done, graph = r->graph;
    memset(r, 0, sizeof *r);
    r->tail_done = tail; r->g2p_done = g2p; r->next_done = next; r->graph = graph;
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

    int how = 0;
    int rc = MPM_OK;
    if (p->use_graph) {
        rc = mpm::rebuild_by_graph(p, S, gblocks_bound, groups_bound, nodes_bound, stream, &how);
        if (rc != MPM_OK) return rc;
    }
    if (!how) {
        rc = mpm::enqueue_rebuild_kernels(p, S, gblocks_bound, groups_bound, nodes_bound, stream, false);
        if (rc != MPM_OK) return rc;
    }
    r->graph = how;
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
