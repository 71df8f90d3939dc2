/*
 * springsim_oracle.c — TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the reference relaxation loop
 * (/root/reference/pkg/src/springsim, numba + numpy), used as the parity
 * checker by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs.  Nothing in the product path links or calls this.
 *
 * Parity is pinned against golden vectors produced by the real reference
 * (tests/golden/make_golden.py -> tests/golden/*.npz): the restatement must
 * reproduce them byte for byte (tests/test_oracle_golden.py).
 *
 * Restated functions (reference file:line):
 *   accumulate_springs_serial   _kernels.py:44-71        -> springs_serial()
 *   fill_slots / sum_slots      _kernels.py:74-155       -> springs_slots() (OpenMP,
 *        int64 atomic slot reservation, per-mass insertion sort by spring id:
 *        the "parallel-det" mode, bitwise equal to serial; without the sort:
 *        the "parallel" mode, the reference bench's default, summed in slot
 *        arrival order)
 *   Engine._rest_lengths        engine.py:250-259        -> rest_lengths()
 *   Engine.forces               engine.py:261-289        -> oracle_forces()
 *   Engine._step_euler/_verlet/_rk4  engine.py:303-354   -> step_*()
 *   Engine._restore_fixed       engine.py:297-301
 *   Engine.step/_check_finite   engine.py:366-381        -> oracle_step()
 *   build_voxel_lattice (boxes) lattice.py:89-136        -> oracle_voxel_box()
 *        (the workload builder of bench.py's reference arm, bench.py:83-89)
 * Built with -O2 -ffp-contract=off (no FMA contraction, like numba/numpy).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define DEGENERATE_LENGTH 1e-12            /* _kernels.py:23 */

typedef struct {
    int64_t n, s;
    double *x, *v, *x_prev;                 /* (n,3); x_prev may be NULL until first Verlet step */
    const double *m, *f_ext;               /* f_ext (n,3) */
    const uint8_t *fixed;                  /* (n) */
    const int64_t *si, *sj;
    const double *k, *l0;
    const int32_t *group;                  /* (s) or NULL */
    int32_t n_groups;
    const int32_t *gmode;                  /* 0 sinusoid, 1 constant-expansion */
    const double *gamp, *gfreq, *gphase;
    int32_t n_planes;
    const double *planes;                  /* 6 per plane */
    double g[3], dt, damping;
    int integrator;                        /* 0 euler, 1 verlet, 2 rk4 */
    int mode;                              /* 0 serial, 1 parallel-det (slots) */
    int threads;
    double t;
    int64_t n_steps;
    int has_prev;
    int64_t degenerate;
    /* scratch */
    double *l0_eff, *acc;
    double *slots; int64_t *slot_spring, *counter, *capacity; int64_t stride;
} oracle_engine;

/* engine.py:250-259 */
static void rest_lengths(oracle_engine *e, double t) {
    if (!e->group || e->n_groups == 0) return;
    for (int64_t q = 0; q < e->s; ++q) {
        int32_t g = e->group[q];
        if (g < 0) continue;
        double scale;
        if (e->gmode[g] == 1) scale = 1.0 + e->gamp[g];
        else scale = 1.0 + e->gamp[g] * sin(2.0 * M_PI * e->gfreq[g] * t + e->gphase[g]);
        e->l0_eff[q] = e->l0[q] * scale;
    }
}

/* _kernels.py:44-71 */
static int64_t springs_serial(const oracle_engine *e, const double *x, double *acc) {
    int64_t degenerate = 0;
    for (int64_t q = 0; q < e->s; ++q) {
        const int64_t i = e->si[q], j = e->sj[q];
        const double dx = x[3 * j] - x[3 * i], dy = x[3 * j + 1] - x[3 * i + 1],
                     dz = x[3 * j + 2] - x[3 * i + 2];
        const double len = sqrt(dx * dx + dy * dy + dz * dz);
        if (len < DEGENERATE_LENGTH) { degenerate++; continue; }
        const double c = e->k[q] * (len - e->l0_eff[q]) / len;
        const double fx = c * dx, fy = c * dy, fz = c * dz;
        acc[3 * i] += fx; acc[3 * i + 1] += fy; acc[3 * i + 2] += fz;
        acc[3 * j] -= fx; acc[3 * j + 1] -= fy; acc[3 * j + 2] -= fz;
    }
    return degenerate;
}

/* _kernels.py:74-155: phase 1 spring-parallel with atomic slot reservation,
 * phase 2 mass-parallel insertion sort by spring id + sum from 0.0. */
static int64_t springs_slots(oracle_engine *e, const double *x, double *acc) {
    int64_t degenerate = 0;
    const int64_t stride = e->stride;
#pragma omp parallel for reduction(+ : degenerate) schedule(static) num_threads(e->threads)
    for (int64_t q = 0; q < e->s; ++q) {
        const int64_t i = e->si[q], j = e->sj[q];
        const double dx = x[3 * j] - x[3 * i], dy = x[3 * j + 1] - x[3 * i + 1],
                     dz = x[3 * j + 2] - x[3 * i + 2];
        const double len = sqrt(dx * dx + dy * dy + dz * dz);
        double fx, fy, fz;
        if (len < DEGENERATE_LENGTH) { degenerate++; fx = fy = fz = 0.0; }
        else {
            const double c = e->k[q] * (len - e->l0_eff[q]) / len;
            fx = c * dx; fy = c * dy; fz = c * dz;
        }
        int64_t a = __atomic_fetch_add(&e->counter[i], 1, __ATOMIC_RELAXED);
        double *sl = e->slots + (i * stride + a) * 3;
        sl[0] = fx; sl[1] = fy; sl[2] = fz; e->slot_spring[i * stride + a] = q;
        int64_t b = __atomic_fetch_add(&e->counter[j], 1, __ATOMIC_RELAXED);
        sl = e->slots + (j * stride + b) * 3;
        sl[0] = -fx; sl[1] = -fy; sl[2] = -fz; e->slot_spring[j * stride + b] = q;
    }
#pragma omp parallel for schedule(static) num_threads(e->threads)
    for (int64_t i = 0; i < e->n; ++i) {
        const int64_t c = e->counter[i];
        int64_t *ss = e->slot_spring + i * stride;
        double *sl = e->slots + i * stride * 3;
        for (int64_t a = 1; a < c && e->mode == 1; ++a) {     /* parallel-det only: sort */
            const int64_t sid = ss[a];
            const double f0 = sl[3 * a], f1 = sl[3 * a + 1], f2 = sl[3 * a + 2];
            int64_t b = a - 1;
            while (b >= 0 && ss[b] > sid) {
                ss[b + 1] = ss[b];
                sl[3 * (b + 1)] = sl[3 * b]; sl[3 * (b + 1) + 1] = sl[3 * b + 1];
                sl[3 * (b + 1) + 2] = sl[3 * b + 2];
                b--;
            }
            ss[b + 1] = sid;
            sl[3 * (b + 1)] = f0; sl[3 * (b + 1) + 1] = f1; sl[3 * (b + 1) + 2] = f2;
        }
        double s0 = 0.0, s1 = 0.0, s2 = 0.0;
        for (int64_t a = 0; a < c; ++a) { s0 += sl[3 * a]; s1 += sl[3 * a + 1]; s2 += sl[3 * a + 2]; }
        acc[3 * i] = s0; acc[3 * i + 1] = s1; acc[3 * i + 2] = s2;
        e->counter[i] = 0;
    }
    return degenerate;
}

/* engine.py:261-289 (gemv x@normal restated as (x0*n0 + x1*n1) + x2*n2;
 * identical to BLAS for axis-aligned normals). */
static void forces(oracle_engine *e, const double *x, const double *v, double t, double *acc) {
    rest_lengths(e, t);
    if (e->mode == 0) {
        memset(acc, 0, sizeof(double) * 3 * e->n);
        e->degenerate += springs_serial(e, x, acc);
    } else {
        e->degenerate += springs_slots(e, x, acc);
    }
#pragma omp parallel for schedule(static) num_threads(e->threads) if (e->mode)
    for (int64_t i = 0; i < e->n; ++i) {
        for (int c = 0; c < 3; ++c) acc[3 * i + c] += e->m[i] * e->g[c];
        for (int c = 0; c < 3; ++c) acc[3 * i + c] += e->f_ext[3 * i + c];
    }
    for (int p = 0; p < e->n_planes; ++p) {
        const double *pl = e->planes + 6 * p;
        const double n0 = pl[0], n1 = pl[1], n2 = pl[2], off = pl[3], pen = pl[4], mu = pl[5];
        for (int64_t i = 0; i < e->n; ++i) {
            const double *xi = x + 3 * i;
            const double depth = off - ((xi[0] * n0 + xi[1] * n1) + xi[2] * n2);
            if (!(depth > 0.0)) continue;
            const double fn = pen * depth;
            acc[3 * i] += fn * n0; acc[3 * i + 1] += fn * n1; acc[3 * i + 2] += fn * n2;
            if (mu > 0.0) {
                const double *vi = v + 3 * i;
                const double vn = (vi[0] * n0 + vi[1] * n1) + vi[2] * n2;
                const double tx = vi[0] - vn * n0, ty = vi[1] - vn * n1, tz = vi[2] - vn * n2;
                const double speed = sqrt(tx * tx + ty * ty + tz * tz);
                if (speed > 1e-15) {
                    const double a = mu * fn, b = speed * e->m[i] / e->dt;
                    const double mag = a <= b ? a : b;
                    const double r = mag / speed;
                    acc[3 * i] -= r * tx; acc[3 * i + 1] -= r * ty; acc[3 * i + 2] -= r * tz;
                }
            }
        }
    }
}

static void restore_fixed(const oracle_engine *e, const double *x, const double *v,
                          double *xn, double *vn) {
    for (int64_t i = 0; i < e->n; ++i)
        if (e->fixed[i])
            for (int c = 0; c < 3; ++c) { xn[3 * i + c] = x[3 * i + c]; vn[3 * i + c] = v[3 * i + c]; }
}

/* engine.py:303-310 */
static void step_euler(oracle_engine *e, double *xn, double *vn) {
    forces(e, e->x, e->v, e->t, e->acc);
    for (int64_t i = 0; i < e->n; ++i) {
        const double dtm = e->dt / e->m[i];
        for (int c = 0; c < 3; ++c) {
            const int64_t q = 3 * i + c;
            xn[q] = e->x[q] + e->dt * e->v[q];
            vn[q] = e->v[q] + dtm * e->acc[q];
            if (e->damping != 0.0) vn[q] *= 1.0 - e->damping;
        }
    }
    restore_fixed(e, e->x, e->v, xn, vn);
}

/* engine.py:312-328 */
static void step_verlet(oracle_engine *e, double *xn, double *vn) {
    forces(e, e->x, e->v, e->t, e->acc);
    for (int64_t i = 0; i < e->n; ++i) {
        const double coef = e->dt * e->dt / e->m[i];
        for (int c = 0; c < 3; ++c) {
            const int64_t q = 3 * i + c;
            const double a = coef * e->acc[q];
            if (!e->has_prev) {
                xn[q] = e->x[q] + e->dt * e->v[q] + 0.5 * a;
                vn[q] = e->v[q];
            } else {
                if (e->damping != 0.0) xn[q] = e->x[q] + (1.0 - e->damping) * (e->x[q] - e->x_prev[q]) + a;
                else xn[q] = 2.0 * e->x[q] - e->x_prev[q] + a;
                vn[q] = (xn[q] - e->x_prev[q]) / (2.0 * e->dt);
            }
        }
    }
    restore_fixed(e, e->x, e->v, xn, vn);
}

/* engine.py:330-354 */
static void step_rk4(oracle_engine *e, double *xn, double *vn) {
    const int64_t n3 = 3 * e->n;
    const double dt = e->dt, t = e->t;
    double *a1 = malloc(sizeof(double) * n3), *a2 = malloc(sizeof(double) * n3),
           *a3 = malloc(sizeof(double) * n3), *a4 = malloc(sizeof(double) * n3),
           *x2 = malloc(sizeof(double) * n3), *v2 = malloc(sizeof(double) * n3),
           *x3 = malloc(sizeof(double) * n3), *v3 = malloc(sizeof(double) * n3),
           *x4 = malloc(sizeof(double) * n3), *v4 = malloc(sizeof(double) * n3);
    const double *x0 = e->x, *v0 = e->v;
    forces(e, x0, v0, t, a1);
    for (int64_t q = 0; q < n3; ++q) a1[q] = a1[q] / e->m[q / 3];
    for (int64_t q = 0; q < n3; ++q) { x2[q] = x0[q] + (0.5 * dt) * v0[q]; v2[q] = v0[q] + (0.5 * dt) * a1[q]; }
    restore_fixed(e, x0, v0, x2, v2);
    forces(e, x2, v2, t + 0.5 * dt, a2);
    for (int64_t q = 0; q < n3; ++q) a2[q] = a2[q] / e->m[q / 3];
    for (int64_t q = 0; q < n3; ++q) { x3[q] = x0[q] + (0.5 * dt) * v2[q]; v3[q] = v0[q] + (0.5 * dt) * a2[q]; }
    restore_fixed(e, x0, v0, x3, v3);
    forces(e, x3, v3, t + 0.5 * dt, a3);
    for (int64_t q = 0; q < n3; ++q) a3[q] = a3[q] / e->m[q / 3];
    for (int64_t q = 0; q < n3; ++q) { x4[q] = x0[q] + dt * v3[q]; v4[q] = v0[q] + dt * a3[q]; }
    restore_fixed(e, x0, v0, x4, v4);
    forces(e, x4, v4, t + dt, a4);
    for (int64_t q = 0; q < n3; ++q) a4[q] = a4[q] / e->m[q / 3];
    for (int64_t q = 0; q < n3; ++q) {
        xn[q] = x0[q] + (dt / 6.0) * (v0[q] + 2.0 * v2[q] + 2.0 * v3[q] + v4[q]);
        vn[q] = v0[q] + (dt / 6.0) * (a1[q] + 2.0 * a2[q] + 2.0 * a3[q] + a4[q]);
        if (e->damping != 0.0) vn[q] *= 1.0 - e->damping;
    }
    restore_fixed(e, x0, v0, xn, vn);
    free(a1); free(a2); free(a3); free(a4); free(x2); free(v2); free(x3); free(v3); free(x4); free(v4);
}

/* ------------------------------------------------------------ public API */

oracle_engine *oracle_create(int64_t n, int64_t s, const double *x, const double *v,
                             const double *m, const double *f_ext, const uint8_t *fixed,
                             const int64_t *si, const int64_t *sj, const double *k,
                             const double *l0, const int32_t *group, int32_t n_groups,
                             const int32_t *gmode, const double *gamp, const double *gfreq,
                             const double *gphase, int32_t n_planes, const double *planes,
                             const double *g, double dt, double damping, int integrator,
                             int mode, int threads) {
    oracle_engine *e = calloc(1, sizeof *e);
    e->n = n; e->s = s;
    e->x = malloc(sizeof(double) * 3 * n); memcpy(e->x, x, sizeof(double) * 3 * n);
    e->v = malloc(sizeof(double) * 3 * n); memcpy(e->v, v, sizeof(double) * 3 * n);
    e->x_prev = malloc(sizeof(double) * 3 * n);
    e->m = m; e->f_ext = f_ext; e->fixed = fixed; e->si = si; e->sj = sj; e->k = k; e->l0 = l0;
    e->group = group; e->n_groups = n_groups; e->gmode = gmode; e->gamp = gamp; e->gfreq = gfreq;
    e->gphase = gphase; e->n_planes = n_planes; e->planes = planes;
    e->g[0] = g[0]; e->g[1] = g[1]; e->g[2] = g[2];
    e->dt = dt; e->damping = damping; e->integrator = integrator; e->mode = mode;
    e->threads = threads > 0 ? threads : 1;
    e->l0_eff = malloc(sizeof(double) * (s ? s : 1)); memcpy(e->l0_eff, l0, sizeof(double) * s);
    e->acc = malloc(sizeof(double) * 3 * n);
    if (mode) {
        int64_t *deg = calloc(n, sizeof(int64_t));
        for (int64_t q = 0; q < s; ++q) { deg[si[q]]++; deg[sj[q]]++; }
        int64_t mx = 0;
        for (int64_t i = 0; i < n; ++i) if (deg[i] + 4 > mx) mx = deg[i] + 4;   /* EXTRA_SLOTS, engine.py:39-41 */
        e->stride = mx;
        e->slots = malloc(sizeof(double) * 3 * n * mx);
        e->slot_spring = malloc(sizeof(int64_t) * n * mx);
        e->counter = calloc(n, sizeof(int64_t));
        free(deg);
    }
    return e;
}

void oracle_destroy(oracle_engine *e) {
    if (!e) return;
    free(e->x); free(e->v); free(e->x_prev); free(e->l0_eff); free(e->acc);
    free(e->slots); free(e->slot_spring); free(e->counter);
    free(e);
}

/* engine.py:366-381.  Returns 0, or the 1-based count of steps done when a
 * step diverged (then *bad_mass is the lowest non-finite mass). */
int64_t oracle_step(oracle_engine *e, int64_t count, int64_t *bad_mass) {
    double *xn = malloc(sizeof(double) * 3 * e->n), *vn = malloc(sizeof(double) * 3 * e->n);
    *bad_mass = -1;
    for (int64_t s = 0; s < count; ++s) {
        if (e->integrator == 0) step_euler(e, xn, vn);
        else if (e->integrator == 1) step_verlet(e, xn, vn);
        else step_rk4(e, xn, vn);
        if (e->integrator == 1) {            /* x_prev <- x, x <- x_new */
            double *old_prev = e->x_prev;
            e->x_prev = e->x; e->x = xn; xn = old_prev;
            e->has_prev = 1;
        } else {
            double *ox = e->x; e->x = xn; xn = ox;
        }
        double *ov = e->v; e->v = vn; vn = ov;
        e->n_steps += 1;
        e->t = (double)e->n_steps * e->dt;
        for (int64_t i = 0; i < e->n; ++i) {
            int ok = 1;
            for (int c = 0; c < 3; ++c) ok &= isfinite(e->x[3 * i + c]) && isfinite(e->v[3 * i + c]);
            if (!ok) { *bad_mass = i; free(xn); free(vn); return s + 1; }
        }
    }
    free(xn); free(vn);
    return 0;
}

void oracle_forces(oracle_engine *e, const double *x, const double *v, double t, double *acc) {
    forces(e, x, v, t, acc);
}

void oracle_get(const oracle_engine *e, double *x, double *v, double *x_prev, int *has_prev,
                double *t, int64_t *n, int64_t *degenerate) {
    if (x) memcpy(x, e->x, sizeof(double) * 3 * e->n);
    if (v) memcpy(v, e->v, sizeof(double) * 3 * e->n);
    if (x_prev && e->has_prev) memcpy(x_prev, e->x_prev, sizeof(double) * 3 * e->n);
    if (has_prev) *has_prev = e->has_prev;
    if (t) *t = e->t;
    if (n) *n = e->n_steps;
    if (degenerate) *degenerate = e->degenerate;
}

void oracle_set(oracle_engine *e, const double *x, const double *v, const double *x_prev) {
    if (x) memcpy(e->x, x, sizeof(double) * 3 * e->n);
    if (v) memcpy(e->v, v, sizeof(double) * 3 * e->n);
    if (x_prev) { memcpy(e->x_prev, x_prev, sizeof(double) * 3 * e->n); e->has_prev = 1; }
}

void oracle_set_params(oracle_engine *e, double damping, const double *g) {
    e->damping = damping;
    if (g) { e->g[0] = g[0]; e->g[1] = g[1]; e->g[2] = g[2]; }
}

void oracle_set_f_ext(oracle_engine *e, const double *f_ext) { e->f_ext = f_ext; }

/* ------------------------------------------------------ workload builder
 *
 * build_voxel_lattice(box_mesh(lo, hi), LatticeSpec(dim=dim), Material(k0, l_ref))
 * (lattice.py:89-136) for a box, restated so that the reference arm of
 * bench.py can build its cube without the product library:
 *   counts = floor((hi - lo)/dim + 1e-9) + 1                 lattice.py:104-107
 *   every grid node is kept (a box contains all its grid nodes, mesh.py:75-132
 *   counts on-surface points as inside); ids in (i,j,k) lexicographic order,
 *   x = lo + idx*dim                                         lattice.py:109-119
 *   the 28 corner pairs of every cell, each sorted, de-duplicated and listed in
 *   (lower id, upper id) order                               lattice.py:121-134
 *   -- here grouped by the lower endpoint a: the corners b > a of the cells that
 *   contain a, sorted and de-duplicated (the same set and order as np.unique);
 *   l0 = np.linalg.norm(x_b - x_a) (lattice.py:84), i.e. OpenBLAS ddot
 *   = sqrt(fma(dz, dz, fma(dy, dy, dx*dx)));
 *   k = (k0 * l_ref) / l0                                    model.py:87-92
 * Call with x == NULL for the sizes only.  Returns the spring count. */
static int cmp_i64(const void *a, const void *b) {
    const int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
    return (x > y) - (x < y);
}

static int upper_partners(int64_t a, const int64_t c[3], int64_t *out) {
    const int64_t nz = c[2], ny = c[1];
    const int64_t i = a / (ny * nz), j = (a / nz) % ny, k = a % nz;
    int64_t buf[64];
    int n = 0;
    for (int64_t ci = i - 1; ci <= i; ++ci)
        for (int64_t cj = j - 1; cj <= j; ++cj)
            for (int64_t ck = k - 1; ck <= k; ++ck) {
                if (ci < 0 || cj < 0 || ck < 0 || ci > c[0] - 2 || cj > ny - 2 || ck > nz - 2) continue;
                for (int q = 0; q < 8; ++q) {            /* corners of cell (ci, cj, ck) */
                    const int64_t b = ((ci + (q >> 2)) * ny + (cj + ((q >> 1) & 1))) * nz + (ck + (q & 1));
                    if (b > a) buf[n++] = b;
                }
            }
    qsort(buf, (size_t)n, sizeof(int64_t), cmp_i64);
    int u = 0;
    for (int q = 0; q < n; ++q)
        if (u == 0 || buf[q] != out[u - 1]) out[u++] = buf[q];
    return u;
}

int64_t oracle_voxel_box(const double lo[3], const double hi[3], double dim, double k0, double l_ref,
                         int64_t counts[3], int64_t *n_masses, double *x, int64_t *si, int64_t *sj,
                         double *k, double *l0) {
    int64_t c[3];
    for (int d = 0; d < 3; ++d) c[d] = (int64_t)floor((hi[d] - lo[d]) / dim + 1e-9) + 1;
    const int64_t n = c[0] * c[1] * c[2];
    if (counts) { counts[0] = c[0]; counts[1] = c[1]; counts[2] = c[2]; }
    if (n_masses) *n_masses = n;
    int64_t *first = malloc(sizeof(int64_t) * (size_t)(n + 1));
    first[0] = 0;
#pragma omp parallel for schedule(static)
    for (int64_t a = 0; a < n; ++a) {
        int64_t tmp[32];
        first[a + 1] = upper_partners(a, c, tmp);
    }
    for (int64_t a = 0; a < n; ++a) first[a + 1] += first[a];
    const int64_t s = first[n];
    if (x) {
#pragma omp parallel for schedule(static)
        for (int64_t a = 0; a < n; ++a) {
            const int64_t idx[3] = {a / (c[1] * c[2]), (a / c[2]) % c[1], a % c[2]};
            for (int d = 0; d < 3; ++d) x[3 * a + d] = lo[d] + (double)idx[d] * dim;
        }
#pragma omp parallel for schedule(static)
        for (int64_t a = 0; a < n; ++a) {
            int64_t part[32];
            const int u = upper_partners(a, c, part);
            for (int q = 0; q < u; ++q) {
                const int64_t w = first[a] + q, b = part[q];
                const double dx = x[3 * b] - x[3 * a], dy = x[3 * b + 1] - x[3 * a + 1],
                             dz = x[3 * b + 2] - x[3 * a + 2];
                si[w] = a;
                sj[w] = b;
                l0[w] = sqrt(fma(dz, dz, fma(dy, dy, dx * dx)));
                k[w] = (k0 * l_ref) / l0[w];
            }
        }
    }
    free(first);
    return s;
}

int oracle_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
