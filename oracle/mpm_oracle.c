/*
 * mpm_oracle.c -- CPU restatement (float64, scalar, single thread per call) of the
 * reference MLS-MPM substep path of arxiv/paper_2111_00699 (`mpmbench`).
 *
 * THIS IS TEST INFRASTRUCTURE, NOT PRODUCT CODE.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  The product path
 * (paper_2111_00699_b200) never links or calls anything in oracle/.
 *
 * Parity status: PINNED for material kinds 0 (weakly compressible fluid) and 1 (fixed
 * corotated), see below.  Kinds 2 (snow: singular-value clamp + hardening) and 3 (sand:
 * Drucker-Prager return mapping) DO NOT EXIST IN THE REFERENCE: their
 * float64 statement below is this repository's own definition of those models --
 * "parity unpinned" -- built on the reference's SVD (orc_svd3) and transfer structure.
 *
 * Parity status of kinds 0/1: PINNED.  tests/test_oracle_golden.py checks every function here
 * bit-for-bit against arrays dumped from the reference itself
 * (tests/golden/make_golden.py, run in the build container against /root/reference)
 * and against the reference tests' own known-answer vectors.
 *
 * Each function cites the reference file:line it restates; paths are relative to
 * /root/reference/pkg/src/mpmbench/.  Data layouts are the reference's:
 *   particles  data[g][ch][lane]  f64, channels pos 0-2, vel 3-5, C 6-14, mass 15, F 16-24 | J 16
 *   grid       raw/vel[pblock][4][64] f64, slot = Morton of the low two bits per axis
 * Build: gcc -O2 -ffp-contract=off -fPIC -shared (no FMA contraction: the reference's
 * numba kernels are compiled without fastmath, so products and sums round separately).
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

typedef int64_t i64;
typedef int32_t i32;
typedef uint8_t u8;

#define CH_POS 0
#define CH_VEL 3
#define CH_C 6
#define CH_MASS 15
#define CH_DEF 16

#define C_ACCUM 0
#define C_QUARANTINE 1
#define C_DEGENERATE 2
#define C_SVD_CLAMP 3
#define C_ADDRESS_ERR 4
#define C_SUBGROUPS 5

#define MASS_SCALE 1099511627776.0 /* 2^40, pipeline.py:43 */
#define MOM_SCALE 4294967296.0     /* 2^32, pipeline.py:44 */
#define EMPTY_KEY ((i64)-1)
#define HASH_MULT ((uint64_t)0x9E3779B97F4A7C15ull)

/* ---- Morton coding: grid.py:41-70 ------------------------------------------------ */
static inline i64 part1by2(i64 v)
{
    uint64_t x = (uint64_t)v & 0x1FFFFFull;
    x = (x | (x << 32)) & 0x1F00000000FFFFull;
    x = (x | (x << 16)) & 0x1F0000FF0000FFull;
    x = (x | (x << 8)) & 0x100F00F00F00F00Full;
    x = (x | (x << 4)) & 0x10C30C30C30C30C3ull;
    x = (x | (x << 2)) & 0x1249249249249249ull;
    return (i64)x;
}
static inline i64 compact1by2(i64 v)
{
    uint64_t x = (uint64_t)v & 0x1249249249249249ull;
    x = (x ^ (x >> 2)) & 0x10C30C30C30C30C3ull;
    x = (x ^ (x >> 4)) & 0x100F00F00F00F00Full;
    x = (x ^ (x >> 8)) & 0x1F0000FF0000FFull;
    x = (x ^ (x >> 16)) & 0x1F00000000FFFFull;
    x = (x ^ (x >> 32)) & 0x1FFFFFull;
    return (i64)x;
}
i64 orc_encode_cell(i64 x, i64 y, i64 z) { return part1by2(x) | (part1by2(y) << 1) | (part1by2(z) << 2); }
void orc_decode_cell(i64 code, i64 *xyz)
{
    xyz[0] = compact1by2(code);
    xyz[1] = compact1by2(code >> 1);
    xyz[2] = compact1by2(code >> 2);
}

/* particles.py:52-58 + grid.py:92-107.  cell = floor(pos/dx - 0.5) + bias (DIVISION).
 * Returns -1, or the index of the first particle outside [0, 2^21). */
i64 orc_particle_codes(const double *pos, i64 n, double dx, i64 bias, i64 *codes)
{
    i64 bad = -1;
    for (i64 i = 0; i < n; ++i) {
        i64 c[3];
        for (int a = 0; a < 3; ++a) {
            c[a] = (i64)floor(pos[3 * i + a] / dx - 0.5) + bias;
            if ((c[a] < 0 || c[a] >= (1 << 21)) && bad < 0) bad = i;
        }
        codes[i] = orc_encode_cell(c[0], c[1], c[2]);
    }
    return bad;
}

/* ---- hash table: grid.py:130-173 -------------------------------------------------- */
static inline i64 hash_slot(i64 key, i64 shift, i64 mask)
{
    /* signed multiply wraps, arithmetic shift, then mask (grid.py:132) */
    i64 prod = (i64)((uint64_t)key * HASH_MULT);
    return (prod >> shift) & mask;
}
void orc_hash_insert_batch(i64 *keys, i64 *vals, i64 shift, i64 mask, const i64 *codes, i64 n,
                           i64 *out_idx, i64 *count_box)
{
    for (i64 i = 0; i < n; ++i) {
        i64 code = codes[i];
        i64 j = hash_slot(code, shift, mask);
        for (;;) {
            i64 k = keys[j];
            if (k == code) { out_idx[i] = vals[j]; break; }
            if (k == EMPTY_KEY) {
                keys[j] = code;
                vals[j] = count_box[0];
                out_idx[i] = count_box[0];
                count_box[0] += 1;
                break;
            }
            j = (j + 1) & mask;
        }
    }
}
void orc_hash_lookup_batch(const i64 *keys, const i64 *vals, i64 shift, i64 mask, const i64 *codes,
                           i64 n, i64 *out_idx)
{
    for (i64 i = 0; i < n; ++i) {
        i64 code = codes[i];
        i64 j = hash_slot(code, shift, mask);
        for (;;) {
            i64 k = keys[j];
            if (k == code) { out_idx[i] = vals[j]; break; }
            if (k == EMPTY_KEY) { out_idx[i] = -1; break; }
            j = (j + 1) & mask;
        }
    }
}

/* grid.py:282-322.  27-neighbourhood insert in (gblock, dz, dy, dx) order. */
i64 orc_dilate_and_link(i64 *keys, i64 *vals, i64 shift, i64 mask, i64 *count_box,
                        const i64 *gcodes, i64 n_g, i64 *codes_out, i32 *neighbor_out)
{
    for (i64 g = 0; g < n_g; ++g) {
        i64 b[3];
        orc_decode_cell(gcodes[g], b);
        int slot = 0;
        for (int dz = -1; dz <= 1; ++dz)
            for (int dy = -1; dy <= 1; ++dy)
                for (int dx = -1; dx <= 1; ++dx) {
                    i64 nx = b[0] + dx, ny = b[1] + dy, nz = b[2] + dz;
                    if (nx < 0 || ny < 0 || nz < 0 || nx >= (1 << 19) || ny >= (1 << 19) ||
                        nz >= (1 << 19))
                        return g;
                    i64 ncode = orc_encode_cell(nx, ny, nz);
                    i64 j = hash_slot(ncode, shift, mask);
                    i64 idx;
                    for (;;) {
                        i64 k = keys[j];
                        if (k == ncode) { idx = vals[j]; break; }
                        if (k == EMPTY_KEY) {
                            keys[j] = ncode;
                            idx = count_box[0];
                            vals[j] = idx;
                            count_box[0] = idx + 1;
                            codes_out[idx] = ncode;
                            break;
                        }
                        j = (j + 1) & mask;
                    }
                    neighbor_out[g * 27 + slot] = (i32)idx;
                    ++slot;
                }
    }
    return -1;
}

/* ---- sorting: particles.py:66-80, 95-129, 152-173, 177-199, 235-261 --------------- */
void orc_counting_sort_perm(const i64 *keys, i64 n, i64 *counts, i64 domain, i64 *perm)
{
    memset(counts, 0, (size_t)domain * sizeof(i64));
    for (i64 i = 0; i < n; ++i) counts[keys[i]] += 1;
    i64 total = 0;
    for (i64 k = 0; k < domain; ++k) {
        i64 c = counts[k];
        counts[k] = total;
        total += c;
    }
    for (i64 i = 0; i < n; ++i) {
        i64 k = keys[i];
        perm[counts[k]] = i;
        counts[k] += 1;
    }
}

void orc_radix10_order(const i64 *keys, i64 length, i64 *order, i64 *scratch)
{
    i64 counts[32];
    memset(counts, 0, sizeof counts);
    for (i64 l = 0; l < length; ++l) order[l] = l;
    for (i64 l = 0; l < length; ++l) counts[keys[l] & 31] += 1;
    i64 total = 0;
    for (int b = 0; b < 32; ++b) { i64 c = counts[b]; counts[b] = total; total += c; }
    for (i64 l = 0; l < length; ++l) { i64 b = keys[l] & 31; scratch[counts[b]] = l; counts[b] += 1; }
    memset(counts, 0, sizeof counts);
    for (i64 j = 0; j < length; ++j) counts[(keys[scratch[j]] >> 5) & 31] += 1;
    total = 0;
    for (int b = 0; b < 32; ++b) { i64 c = counts[b]; counts[b] = total; total += c; }
    for (i64 j = 0; j < length; ++j) {
        i64 l = scratch[j];
        i64 b = (keys[l] >> 5) & 31;
        order[counts[b]] = l;
        counts[b] += 1;
    }
}

i64 orc_build_groups(const i64 *sorted_block, i64 n, i64 lane_width, i32 *group_len,
                     i32 *group_block, i64 *slot_group, i64 *slot_lane)
{
    i64 g = -1, lane = lane_width, prev = -1;
    for (i64 i = 0; i < n; ++i) {
        i64 b = sorted_block[i];
        if (b != prev || lane == lane_width) {
            ++g;
            group_block[g] = (i32)b;
            lane = 0;
            prev = b;
        }
        slot_group[i] = g;
        slot_lane[i] = lane;
        ++lane;
        group_len[g] = (i32)lane;
    }
    return g + 1;
}

i64 orc_gather_live(const double *data, i64 G, i64 nch, i64 LW, const i32 *group_len,
                    const u8 *quarantined, const i64 *orig_id, double *flat, i64 *ids)
{
    i64 n = 0;
    for (i64 g = 0; g < G; ++g)
        for (i64 l = 0; l < group_len[g]; ++l) {
            if (quarantined && quarantined[g * LW + l]) continue;
            for (i64 c = 0; c < nch; ++c) flat[n * nch + c] = data[(g * nch + c) * LW + l];
            ids[n] = orig_id[g * LW + l];
            ++n;
        }
    return n;
}

void orc_scatter_sorted(const double *flat, const i64 *ids, const i64 *perm, i64 n, i64 nch, i64 LW,
                        const i64 *slot_group, const i64 *slot_lane, double *data, i64 *orig_id)
{
    for (i64 j = 0; j < n; ++j) {
        i64 src = perm[j], g = slot_group[j], l = slot_lane[j];
        for (i64 c = 0; c < nch; ++c) data[(g * nch + c) * LW + l] = flat[src * nch + c];
        orig_id[g * LW + l] = ids[src];
    }
}

static inline i64 clamp09(i64 v) { return v < 0 ? 0 : (v > 9 ? 9 : v); }

void orc_recompute_lane_keys(const double *data, i64 G, i64 nch, i64 LW, const i32 *group_len,
                             const i32 *group_origin, double inv_dx, i64 bias, i64 *lane_key)
{
    for (i64 g = 0; g < G; ++g) {
        i64 ox = group_origin[3 * g + 0] - 4, oy = group_origin[3 * g + 1] - 4,
            oz = group_origin[3 * g + 2] - 4;
        for (i64 l = 0; l < group_len[g]; ++l) {
            const double *d = data + g * nch * LW + l;
            i64 bx = clamp09((i64)floor(d[(CH_POS + 0) * LW] * inv_dx - 0.5) + bias - ox);
            i64 by = clamp09((i64)floor(d[(CH_POS + 1) * LW] * inv_dx - 0.5) + bias - oy);
            i64 bz = clamp09((i64)floor(d[(CH_POS + 2) * LW] * inv_dx - 0.5) + bias - oz);
            lane_key[g * LW + l] = bx + 10 * (by + 10 * bz);
        }
    }
}

/* ---- constitutive math: domain.py:189-441, pipeline.py:150-156 --------------------- */
static inline double det3(const double *f)
{
    return f[0] * (f[4] * f[8] - f[5] * f[7]) - f[1] * (f[3] * f[8] - f[5] * f[6]) +
           f[2] * (f[3] * f[7] - f[4] * f[6]);
}

/* One Jacobi rotation on the symmetric 3x3 (app,aqq,apq) with the two remaining
 * off-diagonals (arp, arq) and the V columns p,q.  domain.py:232-303. */
static inline void jacobi_rotate(double *app, double *aqq, double *apq, double *arp, double *arq,
                                 double theta_num, double *vp, double *vq)
{
    double a_pq = *apq;
    double theta = 0.5 * theta_num / a_pq;
    double t = theta >= 0.0 ? 1.0 / (theta + sqrt(1.0 + theta * theta))
                            : -1.0 / (-theta + sqrt(1.0 + theta * theta));
    double c = 1.0 / sqrt(1.0 + t * t);
    double s = t * c;
    double pp = *app, qq = *aqq;
    *app = c * c * pp - 2.0 * s * c * a_pq + s * s * qq;
    *aqq = s * s * pp + 2.0 * s * c * a_pq + c * c * qq;
    *apq = 0.0;
    double rp = *arp, rq = *arq;
    *arp = c * rp - s * rq;
    *arq = s * rp + c * rq;
    for (int r = 0; r < 3; ++r) {
        double tmp = vp[3 * r];
        vp[3 * r] = c * tmp - s * vq[3 * r];
        vq[3 * r] = s * tmp + c * vq[3 * r];
    }
}

/* domain.py:195-379.  f, u, v row-major 3x3; s[3]. */
void orc_svd3(const double *f, double *u, double *s, double *v)
{
    double a00 = f[0] * f[0] + f[3] * f[3] + f[6] * f[6];
    double a01 = f[0] * f[1] + f[3] * f[4] + f[6] * f[7];
    double a02 = f[0] * f[2] + f[3] * f[5] + f[6] * f[8];
    double a11 = f[1] * f[1] + f[4] * f[4] + f[7] * f[7];
    double a12 = f[1] * f[2] + f[4] * f[5] + f[7] * f[8];
    double a22 = f[2] * f[2] + f[5] * f[5] + f[8] * f[8];
    v[0] = 1; v[1] = 0; v[2] = 0; v[3] = 0; v[4] = 1; v[5] = 0; v[6] = 0; v[7] = 0; v[8] = 1;
    for (int it = 0; it < 30; ++it) {
        double m01 = fabs(a01), m02 = fabs(a02), m12 = fabs(a12);
        double big = m01;
        int pair = 0;
        if (m02 > big) { big = m02; pair = 1; }
        if (m12 > big) { big = m12; pair = 2; }
        if (big <= 1e-15 * (fabs(a00) + fabs(a11) + fabs(a22)) + 1e-300) break;
        if (pair == 0)      /* p=0 q=1 r=2: arp=a02 arq=a12 */
            jacobi_rotate(&a00, &a11, &a01, &a02, &a12, a11 - a00, v + 0, v + 1);
        else if (pair == 1) /* p=0 q=2 r=1: arp=a01 arq=a12 */
            jacobi_rotate(&a00, &a22, &a02, &a01, &a12, a22 - a00, v + 0, v + 2);
        else                /* p=1 q=2 r=0: arp=a01 arq=a02 */
            jacobi_rotate(&a11, &a22, &a12, &a01, &a02, a22 - a11, v + 1, v + 2);
    }
    double w0 = a00, w1 = a11, w2 = a22, tmp;
#define SWAPCOL(p, q) \
    for (int r = 0; r < 3; ++r) { tmp = v[3 * r + p]; v[3 * r + p] = v[3 * r + q]; v[3 * r + q] = tmp; }
    if (w0 < w1) { tmp = w0; w0 = w1; w1 = tmp; SWAPCOL(0, 1) }
    if (w1 < w2) { tmp = w1; w1 = w2; w2 = tmp; SWAPCOL(1, 2) }
    if (w0 < w1) { tmp = w0; w0 = w1; w1 = tmp; SWAPCOL(0, 1) }
#undef SWAPCOL
    if (det3(v) < 0.0) { v[2] = -v[2]; v[5] = -v[5]; v[8] = -v[8]; }
    double s0 = w0 > 0.0 ? sqrt(w0) : 0.0;
    double s1 = w1 > 0.0 ? sqrt(w1) : 0.0;
    double s2 = w2 > 0.0 ? sqrt(w2) : 0.0;
    double u00 = f[0] * v[0] + f[1] * v[3] + f[2] * v[6];
    double u10 = f[3] * v[0] + f[4] * v[3] + f[5] * v[6];
    double u20 = f[6] * v[0] + f[7] * v[3] + f[8] * v[6];
    double n = sqrt(u00 * u00 + u10 * u10 + u20 * u20);
    if (n < 1e-30) { u00 = 1.0; u10 = 0.0; u20 = 0.0; }
    else { u00 /= n; u10 /= n; u20 /= n; }
    double u01 = f[0] * v[1] + f[1] * v[4] + f[2] * v[7];
    double u11 = f[3] * v[1] + f[4] * v[4] + f[5] * v[7];
    double u21 = f[6] * v[1] + f[7] * v[4] + f[8] * v[7];
    double d = u01 * u00 + u11 * u10 + u21 * u20;
    u01 -= d * u00; u11 -= d * u10; u21 -= d * u20;
    n = sqrt(u01 * u01 + u11 * u11 + u21 * u21);
    if (n < 1e-30) {
        u01 = -u10; u11 = u00; u21 = 0.0;
        double n2 = sqrt(u01 * u01 + u11 * u11);
        if (n2 < 1e-30) { u01 = 0.0; u11 = 1.0; u21 = 0.0; }
        else { u01 /= n2; u11 /= n2; }
    } else { u01 /= n; u11 /= n; u21 /= n; }
    double u02 = u10 * u21 - u20 * u11;
    double u12 = u20 * u01 - u00 * u21;
    double u22 = u00 * u11 - u10 * u01;
    double fv0 = f[0] * v[2] + f[1] * v[5] + f[2] * v[8];
    double fv1 = f[3] * v[2] + f[4] * v[5] + f[5] * v[8];
    double fv2 = f[6] * v[2] + f[7] * v[5] + f[8] * v[8];
    if (fv0 * u02 + fv1 * u12 + fv2 * u22 < 0.0) s2 = -s2;
    u[0] = u00; u[1] = u01; u[2] = u02; u[3] = u10; u[4] = u11; u[5] = u12;
    u[6] = u20; u[7] = u21; u[8] = u22;
    s[0] = s0; s[1] = s1; s[2] = s2;
}

/* domain.py:383-441.  tau = 2 mu (F - R) F^T + lam (J-1) J I; returns clamp flag. */
int orc_corotated_tau(const double *f, double mu, double lam, double *t)
{
    double J = det3(f), u[9], s[3], v[9];
    orc_svd3(f, u, s, v);
    int clamped = 0;
    if (J <= 1e-10) {
        for (int k = 0; k < 3; ++k) if (s[k] < 1e-4) s[k] = 1e-4;
        J = s[0] * s[1] * s[2];
        clamped = 1;
    }
    double w[9], r[9], dm[9];
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) {
            w[3 * a + b] = s[0] * u[3 * a] * v[3 * b] + s[1] * u[3 * a + 1] * v[3 * b + 1] +
                           s[2] * u[3 * a + 2] * v[3 * b + 2];
            r[3 * a + b] = u[3 * a] * v[3 * b] + u[3 * a + 1] * v[3 * b + 1] +
                           u[3 * a + 2] * v[3 * b + 2];
            dm[3 * a + b] = w[3 * a + b] - r[3 * a + b];
        }
    double two_mu = 2.0 * mu;
    double diag = lam * (J - 1.0) * J;
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) {
            double acc = two_mu * (dm[3 * a] * w[3 * b] + dm[3 * a + 1] * w[3 * b + 1] +
                                   dm[3 * a + 2] * w[3 * b + 2]);
            t[3 * a + b] = (a == b) ? acc + diag : acc;
        }
    return clamped;
}

double orc_fluid_tau(double J, double kappa, double gamma, int clamp_tension)
{
    double p = kappa * (pow(J, -gamma) - 1.0);
    if (clamp_tension && p < 0.0) p = 0.0;
    return -p;
}

/* pipeline.py:136-147 */
static inline void axis_weights(double p, double inv_dx, i64 *b, double *w, double *f)
{
    double bb = floor(p * inv_dx - 0.5);
    double ff = p * inv_dx - bb;
    *b = (i64)bb;
    w[0] = 0.5 * ((1.5 - ff) * (1.5 - ff));
    w[1] = 0.75 - (ff - 1.0) * (ff - 1.0);
    w[2] = 0.5 * ((ff - 0.5) * (ff - 0.5));
    *f = ff;
}
static inline i64 node_slot(i64 cx, i64 cy, i64 cz)
{
    return (cx & 1) | ((cy & 1) << 1) | ((cz & 1) << 2) | ((cx & 2) << 2) | ((cy & 2) << 3) |
           ((cz & 2) << 4);
}

typedef struct {
    i64 lane_width;
    i64 nch;
    i64 mat_kind; /* 0 fluid, 1 fixed corotated */
    double mu, lam, kappa, gamma;
    i64 clamp_tension;
    double density, dx;
    i64 det, do_lane_sort;
    /* plastic kinds only (not in the reference) */
    double theta_c, theta_s, hardening, sand_alpha;
    /* particle sink (not in the reference): lanes whose advected position lies in [sink_lo, sink_hi)
     * are removed by the gather that moved them there -- mass 0, quarantined = 2, out_stats[2] += 1 */
    i64 sink_enabled;
    double sink_lo[3], sink_hi[3];
} OrcTransferParams;

#define CH_PLASTIC 25

/* ---- plastic models (kinds 2, 3): this repository's float64 definition, unpinned ---------
 * Snow (Stomakhin et al. 2013): F_trial = U S V^T, S' = clamp(S, 1-theta_c, 1+theta_s),
 *   F_E = U S' V^T, Jp <- clamp(Jp * prod(S) / prod(S'), 0.1, 10);
 *   stress = fixed-corotated on F_E with mu, lam scaled by exp(hardening * (1 - Jp)).
 * Sand (Klar et al. 2016, Drucker-Prager): e = log|S|, tr = sum e, dev = e - tr/3;
 *   tr > 0 -> S' = I (tip of the cone; the plastic scalar accumulates tr);
 *   dg = |dev| + (3 lam + 2 mu) / (2 mu) * tr * alpha; dg <= 0 -> S' = S;
 *   else S' = exp(e - dg dev / |dev|).  Stress = U (2 mu e' + lam tr(e') I) U^T, e' = log S'.
 *   (Klar's Algorithm 2 sends |dev| == 0 to the tip before it evaluates dg; for tr <= 0 that makes
 *   the map discontinuous at isotropic compression, which lies INSIDE the cone: dg = (..) tr alpha
 *   <= 0.  Here |dev| == 0, tr <= 0 falls under dg <= 0, so the projection is continuous and a
 *   float32 evaluation can be held to it; dg > 0 with tr <= 0 implies |dev| > 0.)
 * Pinned against numpy's LAPACK SVD + the published closed forms: tests/golden/make_plastic_golden.py,
 * tests/golden/plastic.npz, tests/test_oracle_golden.py::test_plastic_models_against_numpy_pin. */
void orc_snow_project(double *F, double *Jp, double theta_c, double theta_s)
{
    double u[9], s[3], v[9], sc[3];
    orc_svd3(F, u, s, v);
    double num = s[0] * s[1] * s[2], den = 1.0;
    for (int k = 0; k < 3; ++k) {
        double c = s[k];
        if (c < 1.0 - theta_c) c = 1.0 - theta_c;
        if (c > 1.0 + theta_s) c = 1.0 + theta_s;
        sc[k] = c;
        den *= c;
    }
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b)
            F[3 * a + b] = sc[0] * u[3 * a] * v[3 * b] + sc[1] * u[3 * a + 1] * v[3 * b + 1] +
                           sc[2] * u[3 * a + 2] * v[3 * b + 2];
    double j = *Jp * num / den;
    if (!(j > 0.1)) j = 0.1;
    if (j > 10.0) j = 10.0;
    *Jp = j;
}

void orc_sand_project(double *F, double *vc, double mu, double lam, double alpha)
{
    double u[9], s[3], v[9], e[3], sc[3];
    orc_svd3(F, u, s, v);
    for (int k = 0; k < 3; ++k) {
        double a = fabs(s[k]);
        e[k] = log(a > 1e-6 ? a : 1e-6);
    }
    double tr = e[0] + e[1] + e[2];
    double d0 = e[0] - tr / 3.0, d1 = e[1] - tr / 3.0, d2 = e[2] - tr / 3.0;
    double dn = sqrt(d0 * d0 + d1 * d1 + d2 * d2);
    if (tr > 0.0) {
        sc[0] = sc[1] = sc[2] = 1.0;
        *vc += tr;
    } else {
        double dg = dn + (3.0 * lam + 2.0 * mu) / (2.0 * mu) * tr * alpha;
        if (dg <= 0.0) { sc[0] = fabs(s[0]); sc[1] = fabs(s[1]); sc[2] = fabs(s[2]); if (sc[0] < 1e-6) sc[0] = 1e-6; if (sc[1] < 1e-6) sc[1] = 1e-6; if (sc[2] < 1e-6) sc[2] = 1e-6; }
        else {
            sc[0] = exp(e[0] - dg * d0 / dn);
            sc[1] = exp(e[1] - dg * d1 / dn);
            sc[2] = exp(e[2] - dg * d2 / dn);
        }
    }
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b)
            F[3 * a + b] = sc[0] * u[3 * a] * v[3 * b] + sc[1] * u[3 * a + 1] * v[3 * b + 1] +
                           sc[2] * u[3 * a + 2] * v[3 * b + 2];
}

void orc_sand_tau(const double *F, double mu, double lam, double *t)
{
    double u[9], s[3], v[9], e[3], d[3];
    orc_svd3(F, u, s, v);
    for (int k = 0; k < 3; ++k) {
        double a = fabs(s[k]);
        e[k] = log(a > 1e-6 ? a : 1e-6);
    }
    double tr = e[0] + e[1] + e[2];
    for (int k = 0; k < 3; ++k) d[k] = 2.0 * mu * e[k] + lam * tr;
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b)
            t[3 * a + b] = d[0] * u[3 * a] * u[3 * b] + d[1] * u[3 * a + 1] * u[3 * b + 1] +
                           d[2] * u[3 * a + 2] * u[3 * b + 2];
}

#define MAXLW 64
typedef struct {
    u8 valid[MAXLW];
    double wx[MAXLW][3], wy[MAXLW][3], wz[MAXLW][3];
    double fx[MAXLW], fy[MAXLW], fz[MAXLW];
    double mm[MAXLW], mvx[MAXLW], mvy[MAXLW], mvz[MAXLW];
    double Q[MAXLW][9];
    i64 order[MAXLW], scr[MAXLW];
} Scratch;

/* pipeline.py:160-238 (merged arm: stress evaluated in place) */
static void scatter_prep(double *data, u8 *quarantined, i64 g, i64 L, const OrcTransferParams *P,
                         double inv_dx, double dt, Scratch *S, i64 *counters)
{
    const i64 LW = P->lane_width, nch = P->nch;
    double coeff_base = -4.0 * dt * inv_dx * inv_dx / P->density;
    double *dg = data + g * nch * LW;
    for (i64 l = 0; l < L; ++l) {
        S->valid[l] = 0;
        if (quarantined[g * LW + l]) continue;
        double m = dg[CH_MASS * LW + l];
        if (m <= 0.0) continue;
        double px = dg[(CH_POS + 0) * LW + l], py = dg[(CH_POS + 1) * LW + l],
               pz = dg[(CH_POS + 2) * LW + l];
        double vx = dg[(CH_VEL + 0) * LW + l], vy = dg[(CH_VEL + 1) * LW + l],
               vz = dg[(CH_VEL + 2) * LW + l];
        if (!(isfinite(px) && isfinite(py) && isfinite(pz) && isfinite(vx) && isfinite(vy) &&
              isfinite(vz))) {
            quarantined[g * LW + l] = 1;
            dg[CH_MASS * LW + l] = 0.0;
            counters[C_QUARANTINE] += 1;
            continue;
        }
        i64 b;
        axis_weights(px, inv_dx, &b, S->wx[l], &S->fx[l]);
        axis_weights(py, inv_dx, &b, S->wy[l], &S->fy[l]);
        axis_weights(pz, inv_dx, &b, S->wz[l], &S->fz[l]);
        S->mm[l] = m;
        S->mvx[l] = m * vx;
        S->mvy[l] = m * vy;
        S->mvz[l] = m * vz;
        double coeff = coeff_base * m;
        if (P->mat_kind == 0) {
            double J = dg[CH_DEF * LW + l], tau;
            if (J <= 0.0) { counters[C_DEGENERATE] += 1; tau = 0.0; }
            else tau = orc_fluid_tau(J, P->kappa, P->gamma, (int)P->clamp_tension);
            for (int r = 0; r < 9; ++r) S->Q[l][r] = m * dg[(CH_C + r) * LW + l];
            S->Q[l][0] += coeff * tau;
            S->Q[l][4] += coeff * tau;
            S->Q[l][8] += coeff * tau;
        } else if (P->mat_kind == 1) {
            double F[9], t[9];
            for (int r = 0; r < 9; ++r) F[r] = dg[(CH_DEF + r) * LW + l];
            if (orc_corotated_tau(F, P->mu, P->lam, t)) counters[C_SVD_CLAMP] += 1;
            for (int r = 0; r < 9; ++r) S->Q[l][r] = m * dg[(CH_C + r) * LW + l] + coeff * t[r];
        } else {
            double F[9], t[9];
            for (int r = 0; r < 9; ++r) F[r] = dg[(CH_DEF + r) * LW + l];
            if (P->mat_kind == 2) {
                double h = exp(P->hardening * (1.0 - dg[CH_PLASTIC * LW + l]));
                if (orc_corotated_tau(F, P->mu * h, P->lam * h, t)) counters[C_SVD_CLAMP] += 1;
            } else {
                orc_sand_tau(F, P->mu, P->lam, t);
            }
            for (int r = 0; r < 9; ++r) S->Q[l][r] = m * dg[(CH_C + r) * LW + l] + coeff * t[r];
        }
        S->valid[l] = 1;
    }
}

/* pipeline.py:242-312 */
static void subgroup_scatter(const i64 *lane_key, i64 L, i64 g, const i32 *group_origin,
                             const i32 *nrow, double *raw, u8 *touched,
                             const OrcTransferParams *P, Scratch *S, i64 *counters)
{
    const i64 LW = P->lane_width;
    const double dx = P->dx;
    i64 ox = group_origin[3 * g], oy = group_origin[3 * g + 1], oz = group_origin[3 * g + 2];
    i64 bcx = ox >> 2, bcy = oy >> 2, bcz = oz >> 2;
    const i64 *lk = lane_key + g * LW;
    i64 s0 = 0;
    while (s0 < L) {
        i64 key = lk[S->order[s0]];
        i64 s1 = s0 + 1;
        while (s1 < L && lk[S->order[s1]] == key) ++s1;
        counters[C_SUBGROUPS] += 1;
        i64 basex = ox - 4 + key % 10, basey = oy - 4 + (key / 10) % 10, basez = oz - 4 + key / 100;
        for (int i = 0; i < 3; ++i) {
            i64 cx = basex + i, rx = (cx >> 2) - bcx + 1;
            for (int j = 0; j < 3; ++j) {
                i64 cy = basey + j, ry = (cy >> 2) - bcy + 1;
                for (int k = 0; k < 3; ++k) {
                    i64 cz = basez + k, rz = (cz >> 2) - bcz + 1;
                    if (rx < 0 || rx > 2 || ry < 0 || ry > 2 || rz < 0 || rz > 2) {
                        counters[C_ADDRESS_ERR] += 1;
                        continue;
                    }
                    i64 nb = nrow[(rz * 3 + ry) * 3 + rx];
                    if (nb < 0) { counters[C_ADDRESS_ERR] += 1; continue; }
                    i64 slot = node_slot(cx, cy, cz);
                    double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
                    for (i64 t = s0; t < s1; ++t) {
                        i64 l = S->order[t];
                        if (!S->valid[l]) continue;
                        double w = S->wx[l][i] * S->wy[l][j] * S->wz[l][k];
                        double dpx = ((double)i - S->fx[l]) * dx;
                        double dpy = ((double)j - S->fy[l]) * dx;
                        double dpz = ((double)k - S->fz[l]) * dx;
                        const double *Q = S->Q[l];
                        double c0 = w * S->mm[l];
                        double c1 = w * (S->mvx[l] + Q[0] * dpx + Q[1] * dpy + Q[2] * dpz);
                        double c2 = w * (S->mvy[l] + Q[3] * dpx + Q[4] * dpy + Q[5] * dpz);
                        double c3 = w * (S->mvz[l] + Q[6] * dpx + Q[7] * dpy + Q[8] * dpz);
                        if (P->det) {
                            c0 = rint(c0 * MASS_SCALE);
                            c1 = rint(c1 * MOM_SCALE);
                            c2 = rint(c2 * MOM_SCALE);
                            c3 = rint(c3 * MOM_SCALE);
                        }
                        a0 += c0; a1 += c1; a2 += c2; a3 += c3;
                    }
                    double *node = raw + nb * 256 + slot;
                    node[0] += a0;
                    node[64] += a1;
                    node[128] += a2;
                    node[192] += a3;
                    touched[nb] = 1;
                    counters[C_ACCUM] += 1;
                }
            }
        }
        s0 = s1;
    }
}

static void scatter_group(double *data, const i64 *lane_key, u8 *quarantined, i64 g, i64 L,
                          const i32 *group_block, const i32 *group_origin, const i32 *neighbor,
                          double *raw, u8 *touched, const OrcTransferParams *P, double inv_dx,
                          double dt, Scratch *S, i64 *counters)
{
    scatter_prep(data, quarantined, g, L, P, inv_dx, dt, S, counters);
    if (P->do_lane_sort) orc_radix10_order(lane_key + g * P->lane_width, L, S->order, S->scr);
    else for (i64 l = 0; l < L; ++l) S->order[l] = l;
    subgroup_scatter(lane_key, L, g, group_origin, neighbor + 27 * (i64)group_block[g], raw,
                     touched, P, S, counters);
}

/* pipeline.py:316-356 */
void orc_p2g(double *data, const i64 *lane_key, u8 *quarantined, const i32 *group_len,
             const i32 *group_block, const i32 *group_origin, i64 G, const i32 *neighbor,
             double *raw, u8 *touched, const OrcTransferParams *P, double dt, i64 *counters)
{
    Scratch S;
    double inv_dx = 1.0 / P->dx;
    for (i64 g = 0; g < G; ++g) {
        i64 L = group_len[g];
        if (L == 0) continue;
        scatter_group(data, lane_key, quarantined, g, L, group_block, group_origin, neighbor, raw,
                      touched, P, inv_dx, dt, &S, counters);
    }
}

/* pipeline.py:400-600, groups [g_lo, g_hi) */
void orc_gather_advect(double *data, i64 *lane_key, u8 *quarantined, const i32 *group_len,
                       const i32 *group_block, const i32 *group_origin, const i32 *neighbor,
                       const double *vel, const double *vel_old, double flip_blend,
                       const OrcTransferParams *P, double dt, i64 bias, double margin_lo,
                       double margin_hi, i64 g_lo, i64 g_hi, double *out_stats, i64 *counters)
{
    const i64 LW = P->lane_width, nch = P->nch;
    const double dx = P->dx;
    double inv_dx = 1.0 / dx;
    double d_inv = 4.0 * inv_dx * inv_dx;
    int use_flip = flip_blend > 0.0;
    for (i64 g = g_lo; g < g_hi; ++g) {
        i64 L = group_len[g];
        if (L == 0) continue;
        const i32 *nrow = neighbor + 27 * (i64)group_block[g];
        i64 ox = group_origin[3 * g], oy = group_origin[3 * g + 1], oz = group_origin[3 * g + 2];
        i64 bcx = ox >> 2, bcy = oy >> 2, bcz = oz >> 2;
        double zx0 = ((double)(ox - bias) - margin_lo) * dx;
        double zy0 = ((double)(oy - bias) - margin_lo) * dx;
        double zz0 = ((double)(oz - bias) - margin_lo) * dx;
        double zx1 = ((double)(ox - bias) + 4.0 + margin_hi) * dx;
        double zy1 = ((double)(oy - bias) + 4.0 + margin_hi) * dx;
        double zz1 = ((double)(oz - bias) + 4.0 + margin_hi) * dx;
        double *dg = data + g * nch * LW;
        for (i64 l = 0; l < L; ++l) {
            if (quarantined[g * LW + l] || dg[CH_MASS * LW + l] <= 0.0) continue;
            double px = dg[(CH_POS + 0) * LW + l], py = dg[(CH_POS + 1) * LW + l],
                   pz = dg[(CH_POS + 2) * LW + l];
            i64 bxl, byl, bzl;
            double wx[3], wy[3], wz[3], fxl, fyl, fzl;
            axis_weights(px, inv_dx, &bxl, wx, &fxl);
            axis_weights(py, inv_dx, &byl, wy, &fyl);
            axis_weights(pz, inv_dx, &bzl, wz, &fzl);
            bxl += bias; byl += bias; bzl += bias;
            double vx = 0, vy = 0, vz = 0, dvx = 0, dvy = 0, dvz = 0;
            double b00 = 0, b01 = 0, b02 = 0, b10 = 0, b11 = 0, b12 = 0, b20 = 0, b21 = 0, b22 = 0;
            for (int i = 0; i < 3; ++i) {
                i64 cx = bxl + i, rx = (cx >> 2) - bcx + 1;
                double dpx = ((double)i - fxl) * dx;
                for (int j = 0; j < 3; ++j) {
                    i64 cy = byl + j, ry = (cy >> 2) - bcy + 1;
                    double dpy = ((double)j - fyl) * dx;
                    for (int k = 0; k < 3; ++k) {
                        i64 cz = bzl + k, rz = (cz >> 2) - bcz + 1;
                        if (rx < 0 || rx > 2 || ry < 0 || ry > 2 || rz < 0 || rz > 2) {
                            counters[C_ADDRESS_ERR] += 1;
                            continue;
                        }
                        i64 nb = nrow[(rz * 3 + ry) * 3 + rx];
                        if (nb < 0) { counters[C_ADDRESS_ERR] += 1; continue; }
                        i64 slot = node_slot(cx, cy, cz);
                        double w = wx[i] * wy[j] * wz[k];
                        const double *node = vel + nb * 256 + slot;
                        double vnx = node[64], vny = node[128], vnz = node[192];
                        double dpz = ((double)k - fzl) * dx;
                        vx += w * vnx; vy += w * vny; vz += w * vnz;
                        if (use_flip) {
                            const double *old = vel_old + nb * 192 + slot;
                            dvx += w * (vnx - old[0]);
                            dvy += w * (vny - old[64]);
                            dvz += w * (vnz - old[128]);
                        }
                        b00 += w * vnx * dpx; b01 += w * vnx * dpy; b02 += w * vnx * dpz;
                        b10 += w * vny * dpx; b11 += w * vny * dpy; b12 += w * vny * dpz;
                        b20 += w * vnz * dpx; b21 += w * vnz * dpy; b22 += w * vnz * dpz;
                    }
                }
            }
            double c[9] = {d_inv * b00, d_inv * b01, d_inv * b02, d_inv * b10, d_inv * b11,
                           d_inv * b12, d_inv * b20, d_inv * b21, d_inv * b22};
            double nvx, nvy, nvz;
            if (use_flip) {
                double ovx = dg[(CH_VEL + 0) * LW + l], ovy = dg[(CH_VEL + 1) * LW + l],
                       ovz = dg[(CH_VEL + 2) * LW + l];
                nvx = (1.0 - flip_blend) * vx + flip_blend * (ovx + dvx);
                nvy = (1.0 - flip_blend) * vy + flip_blend * (ovy + dvy);
                nvz = (1.0 - flip_blend) * vz + flip_blend * (ovz + dvz);
            } else { nvx = vx; nvy = vy; nvz = vz; }
            double npx = px + dt * nvx, npy = py + dt * nvy, npz = pz + dt * nvz;
            if (!(isfinite(npx) && isfinite(npy) && isfinite(npz) && isfinite(nvx) &&
                  isfinite(nvy) && isfinite(nvz))) {
                quarantined[g * LW + l] = 1;
                dg[CH_MASS * LW + l] = 0.0;
                counters[C_QUARANTINE] += 1;
                continue;
            }
            if (P->sink_enabled && npx >= P->sink_lo[0] && npx < P->sink_hi[0] && npy >= P->sink_lo[1] &&
                npy < P->sink_hi[1] && npz >= P->sink_lo[2] && npz < P->sink_hi[2]) {
                /* the particle arrives in the sink box and leaves the simulation: skipped from here
                 * on like a quarantined lane, dropped at the next rebuild */
                quarantined[g * LW + l] = 2;
                dg[(CH_POS + 0) * LW + l] = npx; dg[(CH_POS + 1) * LW + l] = npy;
                dg[(CH_POS + 2) * LW + l] = npz;
                dg[CH_MASS * LW + l] = 0.0;
                out_stats[2] += 1.0;
                continue;
            }
            dg[(CH_POS + 0) * LW + l] = npx; dg[(CH_POS + 1) * LW + l] = npy;
            dg[(CH_POS + 2) * LW + l] = npz;
            dg[(CH_VEL + 0) * LW + l] = nvx; dg[(CH_VEL + 1) * LW + l] = nvy;
            dg[(CH_VEL + 2) * LW + l] = nvz;
            for (int r = 0; r < 9; ++r) dg[(CH_C + r) * LW + l] = c[r];
            if (P->mat_kind == 0) {
                dg[CH_DEF * LW + l] *= 1.0 + dt * (c[0] + c[4] + c[8]);
            } else {
                double F[9], A[9];
                for (int r = 0; r < 9; ++r) F[r] = dg[(CH_DEF + r) * LW + l];
                for (int r = 0; r < 9; ++r) A[r] = dt * c[r];
                A[0] = 1.0 + dt * c[0]; A[4] = 1.0 + dt * c[4]; A[8] = 1.0 + dt * c[8];
                double Fn[9];
                for (int a = 0; a < 3; ++a)
                    for (int b = 0; b < 3; ++b)
                        Fn[3 * a + b] = A[3 * a] * F[b] + A[3 * a + 1] * F[3 + b] + A[3 * a + 2] * F[6 + b];
                if (P->mat_kind == 2) {
                    double jp = dg[CH_PLASTIC * LW + l];
                    orc_snow_project(Fn, &jp, P->theta_c, P->theta_s);
                    dg[CH_PLASTIC * LW + l] = jp;
                } else if (P->mat_kind == 3) {
                    double vc = dg[CH_PLASTIC * LW + l];
                    orc_sand_project(Fn, &vc, P->mu, P->lam, P->sand_alpha);
                    dg[CH_PLASTIC * LW + l] = vc;
                }
                for (int r = 0; r < 9; ++r) dg[(CH_DEF + r) * LW + l] = Fn[r];
            }
            if (npx < zx0 || npx >= zx1 || npy < zy0 || npy >= zy1 || npz < zz0 || npz >= zz1)
                out_stats[0] = 1.0;
            double sp = nvx * nvx + nvy * nvy + nvz * nvz;
            if (sp > out_stats[1]) out_stats[1] = sp;
            i64 kx = clamp09((i64)floor(npx * inv_dx - 0.5) + bias - (ox - 4));
            i64 ky = clamp09((i64)floor(npy * inv_dx - 0.5) + bias - (oy - 4));
            i64 kz = clamp09((i64)floor(npz * inv_dx - 0.5) + bias - (oz - 4));
            lane_key[g * LW + l] = kx + 10 * (ky + 10 * kz);
        }
    }
}

/* pipeline.py:604-653 */
void orc_g2p2g(double *data, i64 *lane_key, u8 *quarantined, const i32 *group_len,
               const i32 *group_block, const i32 *group_origin, i64 G, const i32 *neighbor,
               const double *vel, const double *vel_old, double flip_blend, double *raw,
               u8 *touched, const OrcTransferParams *P, double dt_prev, double dt, i64 bias,
               double margin_lo, double margin_hi, double *out_stats, i64 *counters)
{
    Scratch S;
    double inv_dx = 1.0 / P->dx;
    for (i64 g = 0; g < G; ++g) {
        i64 L = group_len[g];
        if (L == 0) continue;
        orc_gather_advect(data, lane_key, quarantined, group_len, group_block, group_origin,
                          neighbor, vel, vel_old, flip_blend, P, dt_prev, bias, margin_lo,
                          margin_hi, g, g + 1, out_stats, counters);
        scatter_group(data, lane_key, quarantined, g, L, group_block, group_origin, neighbor, raw,
                      touched, P, inv_dx, dt, &S, counters);
    }
}

/* pipeline.py:660-722 */
void orc_grid_finalize(double *vel, const i64 *touched_idx, i64 n_touched, const i64 *codes,
                       i64 det, double dt, const double *gravity, const double *blo,
                       const double *bhi, i64 bc_sticky, i64 apply_bc, double dx, i64 bias,
                       double *vel_old, i64 save_old)
{
    const double inv_sm = 1.0 / MASS_SCALE, inv_sp = 1.0 / MOM_SCALE;
    for (i64 t = 0; t < n_touched; ++t) {
        i64 b = touched_idx[t];
        i64 code = codes[b];
        i64 x0 = 4 * compact1by2(code) - bias;
        i64 y0 = 4 * compact1by2(code >> 1) - bias;
        i64 z0 = 4 * compact1by2(code >> 2) - bias;
        double *nb = vel + b * 256;
        for (i64 slot = 0; slot < 64; ++slot) {
            double m = nb[slot];
            if (m <= 0.0) {
                nb[slot] = 0.0; nb[64 + slot] = 0.0; nb[128 + slot] = 0.0; nb[192 + slot] = 0.0;
                continue;
            }
            double mass, vx, vy, vz;
            if (det) {
                mass = m * inv_sm;
                vx = nb[64 + slot] * inv_sp / mass;
                vy = nb[128 + slot] * inv_sp / mass;
                vz = nb[192 + slot] * inv_sp / mass;
            } else {
                mass = m;
                vx = nb[64 + slot] / m;
                vy = nb[128 + slot] / m;
                vz = nb[192 + slot] / m;
            }
            if (save_old) {
                vel_old[b * 192 + slot] = vx;
                vel_old[b * 192 + 64 + slot] = vy;
                vel_old[b * 192 + 128 + slot] = vz;
            }
            vx += dt * gravity[0]; vy += dt * gravity[1]; vz += dt * gravity[2];
            if (apply_bc) {
                i64 sx = (slot & 1) | ((slot >> 2) & 2);
                i64 sy = ((slot >> 1) & 1) | ((slot >> 3) & 2);
                i64 sz = ((slot >> 2) & 1) | ((slot >> 4) & 2);
                double px = (double)(x0 + sx) * dx, py = (double)(y0 + sy) * dx,
                       pz = (double)(z0 + sz) * dx;
                if (bc_sticky) {
                    if (px <= blo[0] || px >= bhi[0] || py <= blo[1] || py >= bhi[1] ||
                        pz <= blo[2] || pz >= bhi[2]) { vx = 0.0; vy = 0.0; vz = 0.0; }
                } else {
                    if ((px <= blo[0] && vx < 0.0) || (px >= bhi[0] && vx > 0.0)) vx = 0.0;
                    if ((py <= blo[1] && vy < 0.0) || (py >= bhi[1] && vy > 0.0)) vy = 0.0;
                    if ((pz <= blo[2] && vz < 0.0) || (pz >= bhi[2] && vz > 0.0)) vz = 0.0;
                }
            }
            nb[slot] = mass; nb[64 + slot] = vx; nb[128 + slot] = vy; nb[192 + slot] = vz;
        }
    }
}

/* pipeline.py:1172-1188: vel[t] = raw[t] (+ peer raw rows for shared, peer-touched blocks).
 * peer_map[b] = peer's index of local block b, or -1. */
void orc_copy_rows(double *vel, const double *raw, const i64 *touched_idx, i64 n_touched)
{
    for (i64 t = 0; t < n_touched; ++t)
        memcpy(vel + touched_idx[t] * 256, raw + touched_idx[t] * 256, 256 * sizeof(double));
}
void orc_add_peer_rows(double *vel, const i64 *touched_idx, i64 n_touched, const i64 *peer_map,
                       const double *peer_raw, const u8 *peer_touched)
{
    for (i64 t = 0; t < n_touched; ++t) {
        i64 b = touched_idx[t], q = peer_map[b];
        if (q < 0 || peer_touched[q] != 1) continue;
        double *dst = vel + b * 256;
        const double *src = peer_raw + q * 256;
        for (int k = 0; k < 256; ++k) dst[k] += src[k];
    }
}
