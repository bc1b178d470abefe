/*
 * mpm_b200.h -- C ABI of the B200-native MLS-MPM substep core (libmpm_b200.so).
 *
 * This is the drop-in boundary for the substep loop of the reference package `mpmbench`
 * (arxiv/paper_2111_00699).  The reference is Python + numba: its "kernels" are plain
 * functions that borrow contiguous numpy buffers plus scalars and report problems through
 * a counters array.  Every entry point below replaces one of those functions and keeps
 * that contract, with device pointers instead of numpy views:
 *
 *   - the caller owns every buffer (the host layer grows them with the reference's
 *     4x GrowBuffer rule, memory.py:18-22); the library borrows pointers for the
 *     duration of the call, never retains them, and never allocates device memory;
 *   - kernels never raise: they count into `counters[6]` (pipeline.py:57-63) and
 *     `stats` and the host maps those onto the reference's exception classes;
 *   - every call is asynchronous on `stream` and returns an mpm_status immediately;
 *   - different worker handles may be driven from different host threads.
 *
 * Reference paths are relative to /root/reference/pkg/src/mpmbench/.
 *
 * Device data layout (fp32; the reference is fp64 with the same index structure):
 *   particles  pdata[group][channel][32]   channel map of particles.py:24-31:
 *              pos 0-2, vel 3-5, C 6-14 (row-major), mass 15, F 16-24 | J 16,
 *              plastic scalar 25 (snow Jp / sand volume correction; not in the reference)
 *   lane_meta  u16[group][32]   bits 0-9 lane key (pipeline.py:261-263), bit 15 quarantined
 *   grid       float4 node[pblock][64] = (mass, mom_x, mom_y, mom_z) in raw buffers,
 *              (mass, v_x, v_y, v_z) in vel; slot = Morton of the low two bits per axis
 *              (pipeline.py:144-147).  The reference stores the same values channel-major
 *              as [pblock][4][64] (grid.py:427-429).
 */
#ifndef MPM_B200_H
#define MPM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MPM_LANES 32          /* lane_width of a particle group (SimParams.lane_width default) */
#define MPM_CELL_BIAS 64      /* grid.py CELL_BIAS */
#define MPM_N_COUNTERS 6      /* pipeline.py:57-63 */
#define MPM_LANE_QUARANTINED 0x8000u
#define MPM_LANE_SUNK 0x4000u        /* removed by a particle sink (always together with QUARANTINED) */

enum mpm_status {
    MPM_OK = 0,
    MPM_ERR_REJECTED_INPUT = -1,     /* RejectedInputError   */
    MPM_ERR_SPATIAL_DOMAIN = -2,     /* SpatialDomainError   */
    MPM_ERR_RESOURCE = -3,           /* ResourceError (CUDA runtime failure, capacity)    */
    MPM_ERR_CONTRACT = -4,           /* ContractViolationError */
    MPM_ERR_MODE_CONFLICT = -5,      /* ModeConflictError    */
    MPM_ERR_DEGENERATE = -6,         /* DegenerateStateError */
    MPM_ERR_CONFIG = -7,             /* ConfigError          */
    MPM_ERR_BARRIER_TIMEOUT = -8,    /* BarrierTimeoutError  */
    MPM_NEED_CAPACITY = 1            /* mpm_rebuild: a caller-owned buffer is too small (not an error) */
};

enum mpm_material_kind {             /* domain.py:26-28 (+ two plastic kinds) */
    MPM_MAT_FLUID = 0,
    MPM_MAT_FIXED_COROTATED = 1,
    MPM_MAT_SNOW = 2,
    MPM_MAT_SAND = 3
};

enum mpm_counter {                   /* pipeline.py:57-63 */
    MPM_C_ACCUM = 0, MPM_C_QUARANTINE = 1, MPM_C_DEGENERATE = 2,
    MPM_C_SVD_CLAMP = 3, MPM_C_ADDRESS_ERR = 4, MPM_C_SUBGROUPS = 5
};

/* Step clock of CFL-auto frames (Worker.run_frame, pipeline.py:856-871; cfl_dt, domain.py:523-532)
 * kept in DEVICE memory, so that frames with an adaptive step size are paced by the device like
 * fixed-dt frames: the host enqueues steps ahead without knowing their dt.
 *   dt[s & 1]  size of step s.  Written by the grid update of step s - 1 (mpm_grid_params.clock):
 *              dt_s = min(frame_dt - t, cfl dx / max(vmax_{s-2} + c_sound, 1e-12)), vmax_{s-2} read
 *              from the status ring (the reference's 3-slot ring with its two-step lag,
 *              pipeline.py:866, 1104, 1135); by the host for the first step.
 *   t          frame time elapsed before the newest step that has a dt.
 * The grid update of the step that completes a frame (t + dt >= frame_dt - 1e-12) sets bit 1 of
 * that step's status word and raises the guard at its own step: later steps already enqueued are
 * no-ops, the host re-issues them as the next frame.  All arithmetic is float64, as in the
 * reference; kernels convert to float32 where they consume dt. */
typedef struct mpm_step_clock {
    double dt[2];
    double t;
    double reserved;
} mpm_step_clock;

/* Material + step scalars of the transfer kernels: the scalar tail of
 * _p2g_kernel / _gather_advect / _g2p2g_kernel (pipeline.py:316-320, 400-403, 604-610). */
typedef struct mpm_transfer_params {
    int32_t mat_kind;        /* enum mpm_material_kind */
    int32_t nch;             /* channels per particle: 17 fluid, 25 corotated, 26 snow/sand */
    double mu, lam;          /* Lame parameters */
    double kappa, gamma;     /* fluid bulk modulus / exponent */
    int32_t clamp_tension;   /* fluid: clamp negative pressure (pipeline.py:151-156) */
    int32_t count_stats;     /* also maintain C_ACCUM / C_SUBGROUPS (costs atomics) */
    int32_t deterministic;   /* fixed-point accumulation (pipeline.py:43-44, 297-301): raw nodes are
                                four int64 = rint(c 2^40) mass, rint(c 2^32) momentum (32 B per node) */
    int32_t reserved0;
    double density;
    double dx;
    double dt;               /* scatter dt (this step) */
    double dt_gather;        /* gather dt = dt of the grid update that produced vel (pipeline.py:1230) */
    double flip_blend;       /* 0 = APIC only (pipeline.py:489-517) */
    double margin_lo, margin_hi; /* free zone in cells: [origin-margin_lo, origin+4+margin_hi) */
    double theta_c, theta_s, hardening;   /* snow */
    double sand_alpha;       /* sand: sqrt(2/3) 2 sin(phi) / (3 - sin(phi)) */
    /* CFL-auto frames paced by the device (NULL = dt / dt_gather above): the scatter takes
     * clock->dt[clock_step & 1], the gather clock->dt[clock_gather_step & 1] (the step whose grid
     * update produced vel: the same step for a split G2P, the previous one for the fused kernel
     * and for a flush). */
    const mpm_step_clock *clock;
    int32_t clock_step, clock_gather_step;
    /* Particle sink (not in the reference): a particle whose advected position lies
     * in the box [sink_lo, sink_hi) is taken out of the simulation by the gather that moved it there:
     * position stored, mass 0, lane flagged MPM_LANE_QUARANTINED | MPM_LANE_SUNK, orig_id -1,
     * status->removed + 1; no deformation update, free-zone test or max-speed contribution.  Like a
     * quarantined lane it stops scattering at once and is dropped by the next rebuild's compaction
     * (particles.py:177-188). */
    int32_t sink_enabled, reserved5;
    double sink_lo[3], sink_hi[3];
} mpm_transfer_params;

/* Particle store view: ParticleStore (particles.py:268-287). */
typedef struct mpm_store_view {
    float *data;             /* [n_groups][nch][32] */
    int64_t *orig_id;        /* [n_groups][32] */
    uint16_t *lane_meta;     /* [n_groups][32] */
    int32_t *group_len;      /* [n_groups] */
    int32_t *group_block;    /* [n_groups] */
    int32_t *group_start;    /* [n_groups] sorted position of lane 0 (exclusive scan of group_len) */
    int32_t n_groups;
    int32_t nch;
    /* Per-group context row [n_groups][32] (one 128-byte line, written by mpm_build_group_ctx after
     * every rebuild): words 0..26 = 64 * pblock of the 27 neighbours of the group's block
     * (neighbor[group_block]), 27..29 = origin of the block, 30 = group_len, 31 = group_block.
     * The transfer kernels read this one line instead of the dependent chain group_block ->
     * origin / neighbor row.  NULL = read the tables. */
    int32_t *group_ctx;
    /* Optional: the group count lives on the device (a rebuild just produced it and the host has not
     * read it yet).  n_groups above is then only the launch bound; kernels stop at *n_groups_dev. */
    const int32_t *n_groups_dev;
} mpm_store_view;

/* Block table view: BlockTable (grid.py:325-386). */
typedef struct mpm_table_view {
    int64_t *codes;          /* [count] Morton block codes, gblocks first */
    int32_t *origin;         /* [count][4] biased cell coords of node 0 of the block (x,y,z,0) */
    int32_t *neighbor;       /* [n_gblocks][27], index (rz*3+ry)*3+rx, centre 13 */
    uint8_t *touched[2];     /* [count] per parity */
    int32_t count;
    int32_t n_gblocks;
    /* Optional: pblock count on the device; `count` is then the launch bound (see n_groups_dev). */
    const int32_t *count_dev;
} mpm_table_view;

/* Step status block written by the transfer kernels and the grid update (device memory, 72 bytes):
 *   out_stats[0] (free-zone violation) and out_stats[1] (max speed^2) of
 *   _gather_advect (pipeline.py:408-409), plus counters[6] (pipeline.py:57-63). */
typedef struct mpm_step_status {
    int32_t zone_violation;          /* bit 0: a particle left its free zone (out_stats[0]);
                                        bit 1: this step completed a CFL-auto frame (mpm_step_clock) */
    uint32_t vmax2_bits;             /* float bits of max |v|^2 (nonnegative, so uint order = float order) */
    unsigned long long counters[MPM_N_COUNTERS];
    double dt;                       /* size of the step, when a device clock paces it (else untouched) */
    unsigned long long removed;      /* particles taken out by the sink (accumulates like the counters) */
} mpm_step_status;
#define MPM_STATUS_ZONE 1
#define MPM_STATUS_FRAME_END 2

/* ---- library ---------------------------------------------------------------------- */
const char *mpm_version(void);
const char *mpm_last_error(void);       /* text of the last CUDA error seen by this thread */
int mpm_device_arch(void);              /* 100 for sm_100 */
unsigned long long mpm_launch_count(void);  /* kernels launched by this library so far (process-wide) */
/* device alias of page-locked host memory (cudaHostGetDevicePointer), NULL when it is not mapped:
 * the address kernels store status blocks to (mpm_status_publish, mpm_grid_params.publish_*) */
void *mpm_host_alias(void *pinned_host);
/* Map a device allocation exported by another process (64-byte cudaIpcMemHandle_t) into the
 * current device's context, enabling peer access to the exporting GPU when it is another device
 * (cudaIpcMemLazyEnablePeerAccess): the rows a worker reads from its peers (pipeline.py:1172-1188)
 * are then plain device pointers, NVLink loads on an NVSwitch node.  *base_out is the base of the
 * exporter's allocation; one open per (process, handle). */
int mpm_ipc_open(const void *handle64, void **base_out);
int mpm_ipc_close(void *base);
/* *out_host = *dev_ptr (blocking): probe of a mapping opened with mpm_ipc_open. */
int mpm_peek_i32(const int32_t *dev_ptr, int32_t *out_host);

/* Host rendezvous of the ranks of ONE node over a shared-memory segment mapped by the caller
 * (zero-filled, >= mpm_shm_bytes(n_ranks) long): the SpinBarrier + shared Python state of the
 * reference's SharedRuntime (multiworker.py:27-107) for one process per GPU.  Every rank passes
 * n_values (<= MPM_SHM_MAX_VALUES) integers and receives out[n_ranks][n_values]; the call is a
 * full barrier.  MPM_ERR_BARRIER_TIMEOUT after timeout_ms (multiworker.py:66-69). */
#define MPM_SHM_MAX_VALUES 15
int64_t mpm_shm_bytes(int32_t n_ranks);
int mpm_shm_allgather_i64(void *base, int32_t n_ranks, int32_t rank, const int64_t *values, int32_t n_values,
                          int64_t *out, int32_t timeout_ms);

/* ---- rebuild-mapping: Worker._rebuild (pipeline.py:958-1015) ------------------------ */

/* dst[0..n) = value (device words: guard words, flags). */
int mpm_fill_i32(int32_t *dst, int32_t n, int32_t value, void *stream);

/* Staged particles (ParticleStore.stage_append, particles.py:309-334) as the flat channel rows the
 * rebuild reads: flat[i][nch] from compact pos[n][3], vel[n][3] and mass[n] (or mass_scalar when
 * mass is NULL), with the defaults F = I (J = 1), C = 0, plastic scalar at rest. */
int mpm_stage_particles(const float *pos, const float *vel, const float *mass, float mass_scalar, int32_t n,
                        int32_t nch, int32_t mat_kind, float *flat, void *stream);

/* Compaction of the live lanes of the old store into rebuild input order
 * (ParticleStore.gather_flat, particles.py:336-358; _gather_live, particles.py:177-188):
 * group-major, lane-minor, quarantined lanes dropped (drop_quarantined=1) or kept.
 * src_slot[i] = group*32+lane of input particle i; *n_live (device int32) = count. */
int mpm_compact_live(const mpm_store_view *store, int drop_quarantined, int32_t *group_live_scratch,
                     int32_t *src_slot, int32_t *n_live, int32_t *scan_scratch, void *stream);

/* particle_code_batch (particles.py:52-58) + encode_batch (grid.py:92-107):
 * code = Morton(floor(pos/dx - 0.5) + 64) evaluated in float64 with a DIVISION.
 * Input particle i < n_live comes from the old store slot src_slot[i]; i >= n_live comes
 * from the staged flat array staged[(i-n_live)*nch + ch].  *n_total (device) = n_live + n_staged.
 * bad_index (device int32, reset to INT32_MAX by this call) receives the smallest i whose
 * cell leaves [0, 2^21). */
int mpm_particle_codes(const mpm_store_view *store, const int32_t *src_slot, const int32_t *n_live_dev,
                       const float *staged, int32_t n_staged, int32_t n_upper, double dx,
                       int64_t *codes, int32_t *n_total, int32_t *bad_index, void *stream);

/* BlockHashTable.insert_batch in first-occurrence order (grid.py:136-157, 354-357):
 * gidx[i] = dense index of block codes[i]>>6, indices issued in order of first occurrence
 * over i.  Hash = multiply-shift of grid.py:130-133 on a table of hash_cap (power of two)
 * entries that this call clears first.  *n_gblocks (device) receives the block count,
 * gcodes[0..n_gblocks) the unique codes in index order.  overflow (device int32) is set
 * when the table is too small. */
int mpm_hash_insert_blocks(const int64_t *codes, const int32_t *n_dev, int32_t n_upper,
                           int64_t *hkeys, int32_t *hvals, int32_t *hfirst, int32_t hash_cap,
                           int32_t *pslot, int32_t *flag_scratch, int32_t *scan_scratch,
                           int32_t *gidx, int64_t *gcodes, int32_t *n_gblocks, int32_t *overflow,
                           void *stream);

/* _dilate_and_link (grid.py:282-322) + the tail of BlockTable.rebuild (grid.py:362-386):
 * 27-neighbourhood of every gblock inserted in (gblock, dz, dy, dx) order, new blocks
 * numbered from n_gblocks in order of first appearance; fills codes, origin, neighbor.
 * The block count is read from the device (*n_gblocks_dev <= gblocks_bound, the launch bound;
 * flag_scratch holds 2 x 27 x gblocks_bound words): no host round trip between the phases.
 * *count (device) = pblock count; bad_block (device, preset INT32_MAX) = smallest gblock
 * index with a neighbour outside [0, 2^19). */
int mpm_dilate_and_link(const int64_t *gcodes, const int32_t *n_gblocks_dev, int32_t gblocks_bound,
                        int64_t *hkeys, int32_t *hvals, int32_t *hfirst, int32_t hash_cap, int32_t *qslot,
                        int32_t *flag_scratch, int32_t *scan_scratch, int64_t *codes, int32_t *origin,
                        int32_t *neighbor, int32_t pblock_cap, int32_t *count, int32_t *bad_block,
                        int32_t *overflow, void *stream);

/* ParticleStore.histogram_sort part 1 (particles.py:360-399; _counting_sort_perm :66-80,
 * _build_groups :152-173): stable counting sort by key=(gidx<<6)|(code&63) and the lane
 * group structure.  perm[j] = input index of sorted position j.  bin_start has
 * gblocks_bound*64+1 entries, block_group_first gblocks_bound+1 (block count on the device).  *n_groups (device) = group count.  Members of a (block, cell) bin rank
 * themselves by input index; bins with more than 1024 members (particles piled into one cell)
 * are ranked from a bitmap over the input order instead, linear in the bin size:
 * large_scratch (n_upper words) and large_list (n_upper / 1024 + 2 words) are its scratch. */
int mpm_sort_and_group(const int64_t *codes, const int32_t *gidx, const int32_t *n_dev, int32_t n_upper,
                       const int32_t *n_gblocks_dev, int32_t gblocks_bound, int32_t *bin_start, int32_t *tmp_perm,
                       int32_t *perm, int32_t *block_group_first, int32_t *scan_scratch, int32_t *n_groups,
                       int32_t *large_scratch, int32_t *large_list, void *stream);

/* ParticleStore.histogram_sort part 2 (_scatter_sorted particles.py:192-199) fused with
 * set_group_origins + _recompute_lane_keys (particles.py:235-261, 453): permutes all
 * channels and ids from the old store / staged arrays into the new store, zero-fills
 * padding lanes, writes group_len/group_block/group_start and the 10-bit lane keys
 * (float64, MULTIPLICATION by 1/dx as in the reference).  new_store->n_groups is the launch
 * bound, the group and block counts are read from the device. */
int mpm_scatter_sorted(const mpm_store_view *old_store, const int32_t *src_slot, const int32_t *n_live_dev,
                       const float *staged, const int64_t *staged_ids, const int32_t *perm,
                       const int32_t *bin_start, const int32_t *block_group_first, const int32_t *n_gblocks_dev,
                       const int32_t *table_origin, double dx, const mpm_store_view *new_store,
                       const int32_t *n_groups_dev, void *stream);

/* Worker._rebuild (pipeline.py:958-1015) in one call, WITHOUT a host round trip inside it:
 *   compact_live -> particle_codes -> hash_insert_blocks -> dilate_and_link -> sort_and_group ->
 *   scatter_sorted -> build_group_ctx -> vel rows zeroed, raw rows of this parity cleared
 *   [-> the rest of the rebuild step -> the first batch of steady steps].
 * Every count the chain produces (blocks, pblocks, groups) stays on the device: launches are sized
 * by the caller's capacities and the kernels read the counts where they lie (the paper's rebuild
 * takes two CPU-GPU sync points for them; at 64 K particles those two waits and the
 * interpreter around them cost more than the rebuild's kernels).  The scalars are copied to pinned
 * host memory behind the sort and `done_event` is recorded there; mpm_rebuild_wait blocks on that
 * event only -- the kernels enqueued behind it keep the device busy meanwhile -- and fills the
 * result.  Every buffer is the caller's and is described with its capacity.  When a count outgrows
 * one, the chain aborts ON THE DEVICE: the counts later kernels read are zeroed (they become
 * no-ops), the guard of the steps enqueued behind the rebuild is lowered below guard_step, and
 * mpm_rebuild_wait returns MPM_NEED_CAPACITY with the sizes needed (the old store has not been
 * touched: grow and call again).  MPM_ERR_SPATIAL_DOMAIN: result.bad_particle / result.bad_block
 * say which (particles.py:54-57, grid.py:372-377). */
typedef struct mpm_rebuild_plan {
    mpm_store_view old_store;          /* current store (read only) */
    mpm_store_view new_store;          /* other half of the double buffer, room for cap_groups groups */
    int32_t cap_groups;
    int32_t n_staged;                  /* staged appends: flat [n_staged][nch] + ids, or 0 */
    const float *staged;
    const int64_t *staged_ids;
    int32_t n_upper;                   /* particles of the old store + n_staged */
    int32_t cap_gblocks;               /* bounds neighbor [*][27], qslot 27x, qflag 54x, bin_start 64x + 1, bgf + 1 */
    double dx;
    /* scratch (ScratchPool, memory.py:72-114) */
    int32_t *glive;                    /* old n_groups + 1 */
    int32_t *src_slot, *pslot, *flag, *gidx, *tmp_perm, *perm;   /* n_upper each */
    int64_t *codes, *gcodes;           /* n_upper each */
    int32_t *scan;                     /* n_upper / 16 + 1024 */
    int32_t *qslot, *qflag, *bin_start, *bgf;
    /* block table (BlockTable, grid.py:325-386) */
    int64_t *hkeys;
    int32_t *hvals, *hfirst;
    int32_t hash_cap;                  /* power of two; load factor kept below 1/8 */
    int32_t cap_table;                 /* capacity of table_codes / table_origin (>= 27 n_gblocks needed) */
    int64_t *table_codes;
    int32_t *table_origin;
    int32_t *table_neighbor;
    /* nodal buffers reset by the rebuild (pipeline.py:996-1006) */
    float *vel;                        /* [cap_nodes][64] float4 */
    float *raw_par;                    /* rows of this step's parity, node_bytes per node */
    uint8_t *touched_par;
    int32_t cap_nodes;
    int32_t node_bytes;                /* 16, or 32 in deterministic mode */
    int32_t *scalars_dev;              /* 16 device words */
    int32_t *scalars_host;             /* 16 pinned host words */
    /* Optional rest of the rebuild step for a single worker (p2g_params NULL = none): the
     * scatter of the step (pipeline.py:924-926, always split P2G on a rebuild step) and its grid
     * update (pipeline.py:933) are issued right behind the rebuild kernels, so the device does
     * not wait for the host's bookkeeping of the new tables.  Declared later in this header. */
    const struct mpm_transfer_params *p2g_params;
    struct mpm_step_status *p2g_status;
    const struct mpm_grid_params *grid_params;
    struct mpm_step_status *grid_reset_status;
    float *vel_old;                    /* FLIP only */
    int32_t *guard_word;               /* optional: reset to INT32_MAX first (the guard of the speculative
                                          launches that asked for this rebuild, see mpm_guard); it then
                                          guards the rest of the step and the next batch at guard_step */
    int32_t guard_step;                /* step of the rebuild (the tail runs as {guard_word, guard_step}) */
    int32_t async;                     /* 1: return once everything is enqueued; the caller fetches the
                                          result with mpm_rebuild_wait.  0: wait before returning */
    int32_t *large_list;               /* scratch: n_upper / 1024 + 2 words (bins the bitmap ranking takes) */
    void *done_event;                  /* cudaEvent_t recorded behind the copy of the scalars (async) */
    /* split transfer: the gather of the rebuild step (pipeline.py:934-938) issued behind its grid
     * update, its status block stored to status_publish_dst (device alias of pinned memory, or NULL =
     * the caller copies) and status_event recorded.  g2p_params NULL = the caller runs it. */
    const struct mpm_transfer_params *g2p_params;
    struct mpm_step_status *g2p_status;
    struct mpm_step_status *status_publish_dst;
    void *status_event;
    /* The first batch of steady steps (mpm_enqueue_steps) issued right behind the rebuild step, so
     * that the device does not wait for the host's bookkeeping of the new tables.  The plan's store /
     * table views are taken from this rebuild (counts on the device); next_steps NULL = none. */
    const struct mpm_step_plan *next_steps;
    int32_t next_first_step, next_n_steps;
    /* Optional: device word that receives the group count of the new store.  With it the NEXT rebuild
     * can describe this store as old_store {n_groups = capacity of its buffers, n_groups_dev = this
     * word}: nothing in the kernel chain then depends on a host-side count of the previous rebuild,
     * and a rebuild whose buffers, capacities and particle count equal an earlier one's is replayed
     * as a CUDA graph (one launch instead of ~35; use_graph). */
    int32_t *n_groups_out;
    int32_t use_graph;                 /* 1: capture / replay the rebuild kernels as a CUDA graph (n_staged == 0) */
    int32_t reserved1;
} mpm_rebuild_plan;
typedef struct mpm_rebuild_result {
    int32_t n, n_gblocks, count, n_groups;
    int32_t bad_particle, bad_block;   /* INT32_MAX = none */
    int32_t need_hash, need_gblocks, need_table, need_groups, need_nodes;   /* 0 = fits */
    int32_t tail_done;                 /* 1: the P2G and the grid update of the step were issued */
    int32_t g2p_done;                  /* 1: ... and the split gather + its status publication */
    int32_t next_done;                 /* steps of next_steps that were enqueued */
    int32_t graph;                     /* 0 launched kernel by kernel, 1 graph captured by this call, 2 replayed */
} mpm_rebuild_result;
int mpm_rebuild(const mpm_rebuild_plan *plan, mpm_rebuild_result *result, void *stream);
/* Blocks until the scalars of an async mpm_rebuild are on the host, then fills `result` and returns
 * the rebuild's status (MPM_OK / MPM_NEED_CAPACITY / MPM_ERR_SPATIAL_DOMAIN). */
int mpm_rebuild_wait(const mpm_rebuild_plan *plan, mpm_rebuild_result *result);

/* ---- substep: Worker.run_step (pipeline.py:905-940) ---------------------------------
 *
 * Every substep entry point takes `guard`: NULL, or a host struct naming a device int32 and
 * the step being enqueued.  The device word holds the first step whose gather found a
 * particle outside its free zone (INT32_MAX while none; the gather kernels atomicMin their
 * step into it together with status->zone_violation).  A kernel of step s returns without
 * touching memory when the word is < s.  This lets the host enqueue step s+1 before it has
 * read step s's rebuild flag: if step s asked for a rebuild, step s+1's kernels are no-ops
 * and the host re-issues the step after rebuilding (and resetting the word).  Results are
 * identical to the reference's "check flag, then step" order (pipeline.py:911-915). */
#define MPM_MAX_PEERS 15
typedef struct mpm_guard {
    int32_t *first_bad_step;     /* device */
    int32_t step;
    /* One process per GPU with peer-mapped memory (paper_2111_00699_b200/peer.py): the guard
     * words of the other ranks (their HBM, mapped over NVLink).  The gather that raises the local
     * word raises them too (system-scope atomicMin), so that every rank stops after the same step;
     * the write is ordered before this rank's step signal (mpm_signal_step). */
    int32_t n_peer_words;
    int32_t *peer_words[MPM_MAX_PEERS];
} mpm_guard;

/* Worker._clear (pipeline.py:1022-1037): zero the rows of raw flagged in touched and reset
 * the flags; full=1 clears every row (first use of a parity after a rebuild). */
int mpm_clear(float *raw, uint8_t *touched, int32_t count, int full, int32_t node_bytes,
              const mpm_guard *guard, void *stream);   /* node_bytes: 16 (float4) or 32 (deterministic) */

/* _p2g_kernel (pipeline.py:316-356): scatter_prep + subgroup scatter of every group into
 * raw (float4 nodes), touched flags set for every addressed block. */
int mpm_p2g(const mpm_store_view *store, const mpm_table_view *table, float *raw, uint8_t *touched,
            const mpm_transfer_params *params, mpm_step_status *status, const mpm_guard *guard, void *stream);

/* Fill store->group_ctx from the block table (after mpm_scatter_sorted; groups do not change
 * between rebuilds). */
int mpm_build_group_ctx(const mpm_store_view *store, const mpm_table_view *table, void *stream);

/* _reduce_and_update + _grid_finalize (pipeline.py:1166-1231, 660-722): for every block
 * flagged in touched: vel = raw (+ peer raw rows through peer_map where the peer touched
 * the block) ; zero-mass nodes -> 0 ; v = mom/m ; vel_old saved before gravity when
 * vel_old != NULL ; v += dt*g ; box boundary (inclusive comparisons on node world position).
 * reset_status (may be NULL): status block whose zone flag / max speed are zeroed by this
 * kernel for the gather that follows it in stream order. */
typedef struct mpm_grid_params {
    double dt;
    double gravity[3];
    int32_t apply_bc, bc_sticky;        /* BoundaryBox present / mode == "sticky" */
    double box_lo[3], box_hi[3];
    double dx;
    int32_t fuse_clear;                 /* single worker only: also zero the consumed raw rows and
                                           reset their touched flags (saves the next _clear pass) */
    int32_t block_filter;               /* 0 every touched block; 1 only blocks no peer holds;
                                           2 only blocks shared with a peer (halo) */
    int32_t deterministic;              /* raw / peer_raw hold int64 fixed-point nodes (pipeline.py:682-686) */
    int32_t n_peers;                    /* 0..MPM_MAX_PEERS */
    const float *peer_raw[MPM_MAX_PEERS];        /* float4 rows [*, 64] of each peer */
    const uint8_t *peer_touched[MPM_MAX_PEERS];  /* per-row flags, or NULL = every row counts */
    const int32_t *peer_map[MPM_MAX_PEERS];      /* [count]: row of local block b at that peer, or -1 */
    /* Device-side step barrier for peer rows read in place (no packing, no send/recv): CTAs that
     * hold a block shared with a peer, and CTA 0, spin (ld.acquire.sys) until every wait_flags[k]
     * >= wait_value before any peer row is read; CTAs of interior blocks do not wait, so interior
     * work overlaps the peers' scatter.  After wait_timeout_ms the kernel
     * stores 1 to *wait_error and carries on (the host raises BarrierTimeoutError). */
    int32_t n_wait;                     /* 0 = no device-side wait */
    int32_t wait_value;
    int32_t wait_timeout_ms;
    int32_t reserved1;
    const int32_t *wait_flags[MPM_MAX_PEERS];    /* peers' step words (written by mpm_signal_step) */
    int32_t *wait_error;                         /* local device word */
    /* Status publication without the copy engine (all optional, NULL = off): after the step
     * barrier CTA 0 stores *publish_src to *publish_dst and *publish_guard_src to
     * *publish_guard_dst, both device aliases of pinned host memory (cudaHostGetDevicePointer).
     * A kernel -> copy -> kernel chain costs a copy-engine round trip (~20 us) per step; these
     * 60 bytes ride on the update kernel instead.  A guarded-out launch still publishes the guard
     * word (the host tells a skipped step by guard < step). */
    const mpm_step_status *publish_src;
    mpm_step_status *publish_dst;
    const int32_t *publish_guard_src;
    int32_t *publish_guard_dst;
    /* CFL-auto frames paced by the device (clock NULL = dt above).  The update of step clock_step
     * uses clock->dt[clock_step & 1], then advances the clock (see mpm_step_clock): vmax of step
     * clock_step - 1 comes from vmax_ring[(clock_step - 1) % vmax_ring_len] (and from the same slot
     * of every vmax_peer_rings entry: ranks / logical workers that share the frame clock), the
     * step's dt and the frame-end bit go to *clock_status. */
    mpm_step_clock *clock;
    int32_t clock_step;
    int32_t vmax_ring_len;
    const mpm_step_status *vmax_ring;
    mpm_step_status *clock_status;
    double frame_dt, cfl_dx, c_sound;
    int32_t n_vmax_peers, reserved4;
    const mpm_step_status *vmax_peer_rings[MPM_MAX_PEERS];
    /* Optional instrumentation of the multi-GPU step (NULL = off): eight device words, of which
     * four counters accumulate over launches ([4] is scratch): [0] launches, [1] ns CTA 0 spent in the device-side step barrier
     * (%globaltimer: the latency of the slowest peer's signal as this rank sees it), [2] bytes of
     * peer rows read (NVLink traffic on a multi-GPU node: 1 KB per shared touched block and peer),
     * [3] CTAs that had to wait (they own a block shared with a peer). */
    unsigned long long *prof;
} mpm_grid_params;
int mpm_grid_update(float *raw, uint8_t *touched, float *vel, float *vel_old,
                    const mpm_table_view *table, const mpm_grid_params *params,
                    mpm_step_status *reset_status, const mpm_guard *guard, void *stream);

/* Publish "my scatter of this step is complete" to the peers: after everything enqueued before
 * it on `stream`, *word = value with system scope (release).  Peers wait for it inside
 * mpm_grid_update (wait_flags).  Guarded like every step kernel. */
int mpm_signal_step(int32_t *word, int32_t value, const mpm_guard *guard, void *stream);
/* The step barrier of mpm_grid_update on its own (wait_flags / wait_value / wait_timeout_ms /
 * wait_error of `params`): for a rank whose block table is empty. */
int mpm_wait_step(const mpm_grid_params *params, const mpm_guard *guard, void *stream);

/* Pack the raw rows this worker contributes to one peer (one process per GPU: the rows are
 * then exchanged with NCCL send/recv): out_rows[i] = raw row of block send_idx[i], zeros when
 * the block was not touched this step. */
int mpm_pack_halo(const float *raw, const uint8_t *touched, const int32_t *send_idx, int32_t n,
                  float *out_rows, void *stream);

/* _gather_advect (pipeline.py:400-600). */
int mpm_g2p(const mpm_store_view *store, const mpm_table_view *table, const float *vel,
            const float *vel_old, const mpm_transfer_params *params, mpm_step_status *status,
            const mpm_guard *guard, void *stream);

/* _g2p2g_kernel (pipeline.py:604-653): previous step's gather (dt_gather) fused with this
 * step's scatter (dt). */
int mpm_g2p2g(const mpm_store_view *store, const mpm_table_view *table, const float *vel,
              const float *vel_old, float *raw, uint8_t *touched, const mpm_transfer_params *params,
              mpm_step_status *status, const mpm_guard *guard, void *stream);

/* Reset zone_violation and vmax2_bits of a status block before a gather (the reference
 * passes a fresh out_stats = zeros(2) per call, pipeline.py:1090). */
int mpm_status_reset(mpm_step_status *status, const mpm_guard *guard, void *stream);
/* Store *src (and *guard_src, optional) to mapped pinned host memory from a one-warp kernel: the
 * readback of out_stats (pipeline.py:1102-1104) in stream order without the copy engine.  Not
 * guarded: a skipped step still reports where the guard stood. */
int mpm_status_publish(const mpm_step_status *src, mpm_step_status *dst_mapped, const int32_t *guard_src,
                       int32_t *guard_dst_mapped, void *stream);

/* Batched enqueue of n_steps guarded no-rebuild substeps of ONE worker (the inner loop of
 * Worker.run_frame, pipeline.py:872-876, issued from C: small scenes are bound by launch
 * overhead, not by the kernels).  Step s uses raw/touched[s & 1] and status slot s % ring; the
 * slot is stored to `status_host` (pinned, written through its device alias by the grid update
 * (fused) or by mpm_status_publish (split); cudaMemcpyAsync when the memory is not mapped) and
 * `events[slot]` (cudaEvent_t handles owned by the caller) is recorded after it.  Fused: g2p2g ->
 * grid update (+ publication).  Split: [clear] -> p2g -> grid update -> g2p -> publication.
 * Every kernel carries the guard {guard_word, s}. */
#define MPM_MAX_STATUS_RING 32
typedef struct mpm_step_plan {
    mpm_store_view store;
    mpm_table_view table;
    float *raw[2];
    uint8_t *touched[2];
    float *vel, *vel_old;
    mpm_transfer_params transfer;      /* dt, dt_gather of the first step, split-mode free zone */
    double fused_margin_lo, fused_margin_hi;   /* free zone of the fused gather (shrunk, pipeline.py:1128) */
    mpm_grid_params grid;
    int32_t fused;                     /* 1: transfer = g2p2g with a pending gather; 0: split */
    int32_t status_ring;               /* slots in status_dev / status_host / events */
    mpm_step_status *status_dev;       /* device [status_ring] */
    mpm_step_status *status_host;      /* pinned host [status_ring] */
    void *events[MPM_MAX_STATUS_RING]; /* cudaEvent_t per slot */
    int32_t *guard_word;               /* device */
    /* peer-mapped stepping (all optional, zero = single worker): guard words of the other ranks,
     * this rank's step word (signalled with s + 1 after the scatter of step s; the grid update of
     * step s waits for grid.wait_flags >= s + 1), and a pinned host ring that receives the guard
     * word next to each status slot */
    int32_t n_peer_words;
    int32_t reserved2;
    int32_t *peer_guard_words[MPM_MAX_PEERS];
    int32_t *signal_word;
    int32_t *guard_host;               /* pinned host [status_ring] or NULL */
    /* peers' raw rows / touched flags per step parity (grid.n_peers entries each; grid.peer_map
     * holds the maps, grid.peer_raw / peer_touched are filled per step from these) */
    const float *peer_raw[2][MPM_MAX_PEERS];
    const uint8_t *peer_touched[2][MPM_MAX_PEERS];
    void *time_events[2 * MPM_MAX_STATUS_RING]; /* optional (NULL): cudaEvent_t pairs recorded around the
                                          dominant transfer kernel (g2p2g / p2g) of step first+k */
    int32_t full_clear_first;          /* 1: the first step of the batch clears its raw parity in full
                                          before scattering -- the first use of the parity a rebuild
                                          left untouched (pipeline.py:1002-1006, 1022-1037) */
    int32_t reserved3;
    /* CFL-auto frames: grid.clock (and frame_dt / cfl_dx / c_sound / vmax rings) set = every kernel
     * of the batch takes its dt from the device clock; transfer.dt / dt_gather / grid.dt are ignored. */
} mpm_step_plan;
int mpm_enqueue_steps(const mpm_step_plan *plan, int32_t first_step, int32_t n_steps, void *stream);

/* ---- readback / aggregates ---------------------------------------------------------- */

/* ParticleStore.positions_with_ids / state readback (particles.py:466-475): all stored
 * lanes (quarantined included) in (group, lane) order as flat[n][nch] + ids[n]. */
int mpm_gather_state(const mpm_store_view *store, float *flat, int64_t *ids, void *stream);
/* positions only: pos[n][3] + ids[n] (the per-frame snapshot readback, bench.py:398-403). */
int mpm_gather_positions(const mpm_store_view *store, float *pos, int64_t *ids, void *stream);

/* total_mass / total_momentum (particles.py:477-487) and kinetic energy, accumulated in
 * float64: out[0]=mass, out[1..3]=momentum, out[4]=kinetic energy. */
int mpm_particle_aggregates(const mpm_store_view *store, double *out5, void *stream);

/* grid mass / momentum over touched blocks of raw (pipeline.py:1189-1203): out[0..3]. */
int mpm_grid_aggregates(const float *raw, const uint8_t *touched, int32_t count, int32_t deterministic,
                        double *out4, void *stream);

/* Shared-block tagging (Worker._post_barrier, pipeline.py:1147-1164; _hash_lookup_batch,
 * grid.py:161-173): peer_map[local index of code] = position in peer_codes, -1 elsewhere. */
int mpm_tag_shared(const int64_t *peer_codes, int32_t n_peer_codes, const int64_t *hkeys,
                   const int32_t *hvals, int32_t hash_cap, int32_t *peer_map, int32_t local_count,
                   void *stream);

#ifdef __cplusplus
}
#endif
#endif /* MPM_B200_H */
