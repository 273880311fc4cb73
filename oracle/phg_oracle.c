/*
 * phg_oracle.c -- CPU restatement of the reference PHG trace (TEST INFRASTRUCTURE).
 *
 * This file is the CHECKER, not the product.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load it.  The product
 * path (paper_2604_05794_b200/) never links or calls it.
 *
 * It restates, in scalar IEEE-754 binary64 arithmetic with no contraction
 * (built with -ffp-contract=off), the numpy algorithm of
 *   strandkit.phg.trace_batch              /root/reference/pkg/src/strandkit/phg.py:67-163
 *   strandkit.volume.sample_orientation_batch  .../volume.py:183-224
 *   strandkit.volume.OOVolume.voxel_of/in_bounds/centers  .../volume.py:42-53
 *   strandkit.geom.normalize                .../geom.py:6-10
 * operation by operation, in the same evaluation order numpy uses, so that its
 * output is bit-identical to the reference (pinned against tests/golden/ fixtures,
 * which were produced by running the reference itself; see
 * tests/golden/make_golden.py).  Evaluation-order facts it relies on (measured
 * with numpy 2.3.5 in the build container):
 *   np.linalg.norm(v, axis=1)   == sqrt((x*x + y*y) + z*z)
 *   np.einsum("ij,ij->i", a, b) == (a0*b0 + a2*b2) + a1*b1
 *
 * Strands are independent except in strict mode (phg.py:136-155), where all
 * strands advance in lockstep and commit to live_counts after every step; the
 * strict path here is therefore a step-major double loop.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct {
    double step_mm;
    double min_support;
    double steer;
    int32_t max_vertices;
    int32_t probe_steps;
    int32_t coast_steps;
    int32_t strict;
    double turn_cos; /* opt-in angle stop (our extension, not the reference): -2 = off */
} oracle_params;

typedef struct {
    const float *ori;      /* (nx,ny,nz,3) f32, C order */
    const uint8_t *occ;    /* (nx,ny,nz) bool */
    const uint8_t *at_cap; /* (nx,ny,nz) bool or NULL */
    const int64_t *near;   /* (nx,ny,nz,3) int64 or NULL */
    uint16_t *counts;      /* strict mode live counts or NULL */
    int64_t nx, ny, nz;
    double ox, oy, oz, vs;
} oracle_field;

/* numpy: np.linalg.norm(v, axis=1) for a 3-vector */
static inline double norm3(double x, double y, double z) { return sqrt((x * x + y * y) + z * z); }

/* numpy: np.einsum("ij,ij->i") for 3-vectors (pairing measured, see header) */
static inline double dot3(double a0, double a1, double a2, double b0, double b1, double b2) {
    return (a0 * b0 + a2 * b2) + a1 * b1;
}

/* geom.normalize (geom.py:6-10): v / np.maximum(|v|, 1e-12); NaN propagates */
static inline void normalize3(double *x, double *y, double *z) {
    double n = norm3(*x, *y, *z);
    double d = (n < 1e-12) ? 1e-12 : n;
    *x = *x / d;
    *y = *y / d;
    *z = *z / d;
}

static inline int64_t floor_to_i64(double g) {
    double f = floor(g);
    /* numpy casts out-of-range / NaN floats to INT64_MIN on x86 */
    if (!(f >= -9.2e18 && f <= 9.2e18)) return INT64_MIN;
    return (int64_t)f;
}

/* volume.sample_orientation_batch for one point (volume.py:190-224) */
static void sample(const oracle_field *F, double px, double py, double pz, double qx, double qy,
                   double qz, double *rx, double *ry, double *rz, int *has, double *sup) {
    double gx = (px - F->ox) / F->vs - 0.5;
    double gy = (py - F->oy) / F->vs - 0.5;
    double gz = (pz - F->oz) / F->vs - 0.5;
    int64_t bx = floor_to_i64(gx), by = floor_to_i64(gy), bz = floor_to_i64(gz);
    double fx = gx - (double)bx, fy = gy - (double)by, fz = gz - (double)bz;
    double ax = 0.0, ay = 0.0, az = 0.0, ws = 0.0;
    for (int dx = 0; dx < 2; ++dx) {
        for (int dy = 0; dy < 2; ++dy) {
            for (int dz = 0; dz < 2; ++dz) {
                int64_t ix = bx + dx, iy = by + dy, iz = bz + dz;
                int inb = ix >= 0 && ix < F->nx && iy >= 0 && iy < F->ny && iz >= 0 && iz < F->nz;
                int64_t cx = ix < 0 ? 0 : (ix >= F->nx ? F->nx - 1 : ix);
                int64_t cy = iy < 0 ? 0 : (iy >= F->ny ? F->ny - 1 : iy);
                int64_t cz = iz < 0 ? 0 : (iz >= F->nz ? F->nz - 1 : iz);
                int64_t lin = (cx * F->ny + cy) * F->nz + cz;
                int occ = F->occ[lin] && inb;
                double w = ((dx ? fx : 1 - fx) * (dy ? fy : 1 - fy)) * (dz ? fz : 1 - fz);
                if (!occ) w = 0.0;
                double o0 = (double)F->ori[3 * lin + 0];
                double o1 = (double)F->ori[3 * lin + 1];
                double o2 = (double)F->ori[3 * lin + 2];
                double s = dot3(o0, o1, o2, qx, qy, qz) < 0 ? -1.0 : 1.0;
                double k = w * s;
                ax = ax + k * o0;
                ay = ay + k * o1;
                az = az + k * o2;
                ws = ws + w;
            }
        }
    }
    int h = ws > 0;
    if (h && norm3(ax, ay, az) < 1e-9) {
        ax = qx;
        ay = qy;
        az = qz;
    }
    normalize3(&ax, &ay, &az);
    if (!h) ax = ay = az = 0.0;
    *rx = ax;
    *ry = ay;
    *rz = az;
    *has = h;
    *sup = ws;
}

typedef struct {
    double px, py, pz, dx, dy, dz;
    int64_t probe_left, coast, nverts, last_sup;
    int64_t lvx, lvy, lvz;
    int entered, active;
} strand_state;

static void init_state(strand_state *s, const double *sp, const double *sd, const oracle_params *P) {
    s->px = sp[0];
    s->py = sp[1];
    s->pz = sp[2];
    s->dx = sd[0];
    s->dy = sd[1];
    s->dz = sd[2];
    normalize3(&s->dx, &s->dy, &s->dz);
    s->probe_left = P->probe_steps;
    s->coast = 0;
    s->nverts = 1;
    s->last_sup = 1;
    s->lvx = s->lvy = s->lvz = -1000000000LL;
    s->entered = 0;
    s->active = 1;
}

/* One iteration of the trace_batch loop body for one active strand
 * (phg.py:99-156).  Returns 1 if the strand appended a vertex.  The strict
 * commit (phg.py:150-154) is done by the caller through *commit_vox. */
static int step_one(const oracle_field *F, const oracle_params *P, strand_state *s, double *out3,
                    int64_t *commit_vox) {
    double ox, oy, oz, sup;
    int has;
    sample(F, s->px, s->py, s->pz, s->dx, s->dy, s->dz, &ox, &oy, &oz, &has, &sup);
    int supported = sup >= P->min_support;
    double sx = (has && supported) ? ox : s->dx;
    double sy = (has && supported) ? oy : s->dy;
    double sz = (has && supported) ? oz : s->dz;
    double half = 0.5 * P->step_mm;
    double mx = s->px + half * sx, my = s->py + half * sy, mz = s->pz + half * sz;
    double o2x, o2y, o2z, sup2;
    int has2;
    sample(F, mx, my, mz, sx, sy, sz, &o2x, &o2y, &o2z, &has2, &sup2);
    if (has2 && sup2 >= P->min_support) {
        sx = o2x;
        sy = o2y;
        sz = o2z;
    }
    if (F->near && P->steer > 0 && !supported) { /* phg.py:108-117 */
        int64_t vx = floor_to_i64((s->px - F->ox) / F->vs);
        int64_t vy = floor_to_i64((s->py - F->oy) / F->vs);
        int64_t vz = floor_to_i64((s->pz - F->oz) / F->vs);
        vx = vx < 0 ? 0 : (vx > F->nx - 1 ? F->nx - 1 : vx);
        vy = vy < 0 ? 0 : (vy > F->ny - 1 ? F->ny - 1 : vy);
        vz = vz < 0 ? 0 : (vz > F->nz - 1 ? F->nz - 1 : vz);
        const int64_t *t = F->near + 3 * ((vx * F->ny + vy) * F->nz + vz);
        double tx = F->ox + ((double)t[0] + 0.5) * F->vs;
        double ty = F->oy + ((double)t[1] + 0.5) * F->vs;
        double tz = F->oz + ((double)t[2] + 0.5) * F->vs;
        double ux = tx - s->px, uy = ty - s->py, uz = tz - s->pz;
        normalize3(&ux, &uy, &uz);
        int ahead = dot3(ux, uy, uz, sx, sy, sz) > -0.2;
        double bx = sx + P->steer * ux, by = sy + P->steer * uy, bz = sz + P->steer * uz;
        normalize3(&bx, &by, &bz);
        if (ahead) {
            sx = bx;
            sy = by;
            sz = bz;
        }
    }
    int die = 0;
    int still_probe = !s->entered && !supported;
    if (still_probe) {
        s->probe_left -= 1;
        die = s->probe_left < 0;
    }
    int lost = s->entered && !supported;
    if (lost) s->coast += 1;
    if (s->entered && supported) s->coast = 0;
    if (lost && s->coast > P->coast_steps) die = 1;
    if (supported) {
        s->entered = 1;
        s->last_sup = s->nverts;
    }
    double tx = s->px + P->step_mm * sx, ty = s->py + P->step_mm * sy, tz = s->pz + P->step_mm * sz;
    int64_t vx = floor_to_i64((tx - F->ox) / F->vs);
    int64_t vy = floor_to_i64((ty - F->oy) / F->vs);
    int64_t vz = floor_to_i64((tz - F->oz) / F->vs);
    int inb = vx >= 0 && vx < F->nx && vy >= 0 && vy < F->ny && vz >= 0 && vz < F->nz;
    if (!inb) die = 1;
    /* opt-in angle stop (PHG_FLAG_TURN_STOP; the reference has none) */
    if (dot3(s->dx, s->dy, s->dz, sx, sy, sz) < P->turn_cos) die = 1;
    int new_vox = vx != s->lvx || vy != s->lvy || vz != s->lvz;
    int full = 0;
    if (inb) {
        int64_t lin = (vx * F->ny + vy) * F->nz + vz;
        if (P->strict)
            full = F->counts[lin] >= 1;
        else if (F->at_cap)
            full = F->at_cap[lin] != 0;
    }
    if (s->entered && inb && new_vox && full) die = 1;
    *commit_vox = -1;
    if (die) {
        s->active = 0;
        return 0;
    }
    out3[0] = tx;
    out3[1] = ty;
    out3[2] = tz;
    s->nverts += 1;
    s->px = tx;
    s->py = ty;
    s->pz = tz;
    s->dx = sx;
    s->dy = sy;
    s->dz = sz;
    if (new_vox) *commit_vox = (vx * F->ny + vy) * F->nz + vz;
    s->lvx = vx;
    s->lvy = vy;
    s->lvz = vz;
    return 1;
}

static inline int64_t keep_of(const strand_state *s) {
    if (s->entered) return s->last_sup > 1 ? s->last_sup : 1;
    return s->nverts;
}

/*
 * Trace n seeds.  slab: n*max_vertices*3 doubles (row i holds strand i's
 * vertices); keep[i] = number of leading vertices the reference returns
 * (phg.py:161); entered[i] = the reference's `entered` flag.
 */
int phg_oracle_trace(const float *ori, const uint8_t *occ, int64_t nx, int64_t ny, int64_t nz,
                     const double *origin, double vs, const uint8_t *at_cap, const int64_t *near,
                     uint16_t *live_counts, const oracle_params *P, const double *seed_pos,
                     const double *seed_dir, int64_t n, double *slab, int64_t *keep,
                     uint8_t *entered, int nthreads) {
    if (P->max_vertices < 1) return -1;
    oracle_field F = {ori, occ, at_cap, near, live_counts, nx, ny, nz, origin[0], origin[1], origin[2], vs};
    const int64_t mv = P->max_vertices;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
    if (!P->strict) {
#pragma omp parallel for schedule(dynamic, 64)
        for (int64_t i = 0; i < n; ++i) {
            strand_state s;
            init_state(&s, seed_pos + 3 * i, seed_dir + 3 * i, P);
            double *row = slab + (size_t)i * mv * 3;
            row[0] = s.px;
            row[1] = s.py;
            row[2] = s.pz;
            int64_t cv;
            for (int64_t it = 0; it < mv - 1 && s.active; ++it)
                step_one(&F, P, &s, row + 3 * s.nverts, &cv);
            keep[i] = keep_of(&s);
            entered[i] = (uint8_t)s.entered;
        }
        return 0;
    }
    /* strict: lockstep over all strands, counts committed after each step */
    uint16_t *own = NULL;
    if (!F.counts) {
        own = (uint16_t *)calloc((size_t)(nx * ny * nz), sizeof(uint16_t));
        if (!own) return -2;
        F.counts = own;
    }
    strand_state *st = (strand_state *)malloc(sizeof(strand_state) * (size_t)(n > 0 ? n : 1));
    int64_t *cv = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    if (!st || !cv) {
        free(st);
        free(cv);
        free(own);
        return -2;
    }
    for (int64_t i = 0; i < n; ++i) {
        init_state(&st[i], seed_pos + 3 * i, seed_dir + 3 * i, P);
        double *row = slab + (size_t)i * mv * 3;
        row[0] = st[i].px;
        row[1] = st[i].py;
        row[2] = st[i].pz;
    }
    for (int64_t it = 0; it < mv - 1; ++it) {
        int any = 0;
        for (int64_t i = 0; i < n; ++i) {
            cv[i] = -1;
            if (!st[i].active) continue;
            any = 1;
            double *row = slab + (size_t)i * mv * 3;
            step_one(&F, P, &st[i], row + 3 * st[i].nverts, &cv[i]);
        }
        if (!any) break;
        for (int64_t i = 0; i < n; ++i) /* np.add.at on uint16 wraps */
            if (cv[i] >= 0) F.counts[cv[i]] = (uint16_t)(F.counts[cv[i]] + 1);
    }
    for (int64_t i = 0; i < n; ++i) {
        keep[i] = keep_of(&st[i]);
        entered[i] = (uint8_t)st[i].entered;
    }
    free(st);
    free(cv);
    free(own);
    return 0;
}

/* sample_orientation_batch over n points (volume.py:183-224) */
void phg_oracle_sample(const float *ori, const uint8_t *occ, int64_t nx, int64_t ny, int64_t nz,
                       const double *origin, double vs, const double *pts, const double *prev, int64_t n,
                       double *dirs, uint8_t *has, double *support) {
    oracle_field F = {ori, occ, NULL, NULL, NULL, nx, ny, nz, origin[0], origin[1], origin[2], vs};
    for (int64_t i = 0; i < n; ++i) {
        int h;
        sample(&F, pts[3 * i], pts[3 * i + 1], pts[3 * i + 2], prev[3 * i], prev[3 * i + 1], prev[3 * i + 2],
               dirs + 3 * i, dirs + 3 * i + 1, dirs + 3 * i + 2, &h, support + i);
        has[i] = (uint8_t)h;
    }
}

int phg_oracle_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
