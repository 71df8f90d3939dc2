// Resident kernel for small scenes ("small scenes").
//
// A scene of at most kResidentMaxCtas tiles (the walker, a few dozen
// robots, the cantilever) is stepped by ONE CTA -- or, in fp32, one
// thread-block cluster with one tile per CTA -- for a whole batch:
// positions live in shared memory, double-buffered by step parity; every
// mass's incidence list and a dictionary of distinct spring records are
// staged once per launch; each lane group keeps its mass's velocity and
// history (x_prev / u) in registers.  A step is: copy this CTA's halo
// positions from their owner CTAs through distributed shared memory (one
// read per halo mass), a pass over the CTA's own shared memory, and one
// barrier (__syncthreads for a lone CTA, the cluster barrier otherwise) --
// no launch, no grid barrier, no global-memory round trip: "many small-dt
// substeps batched into a persistent kernel" (north_star) for scenes whose
// step is a few microseconds of work.
//
// Arithmetic is that of the multi-CTA kernels: fp64 sums each mass's
// springs in ascending spring id with the reference's op order
// (_kernels.py:51-70, engine.py:273-328), so results are bitwise those of
// step_kernel and of the reference; fp32 uses the displacement form
// d = D + (r_o - r_m) of tile_f32.cuh.
#pragma once

#include <cooperative_groups.h>

#include "kernels.cuh"
#include "tile_f32.cuh"
#include "tile_f64.cuh"

namespace ss {

constexpr int kResidentSlots = 256;         // slots per CTA (one tile)
constexpr int kResidentMaxCtas = 16;        // cluster size (above 8: non-portable, B200 allows 16)
constexpr int kResidentMaxGroups = 64;      // actuation groups staged in shared memory

// add_external (kernels.cuh) with f_ext from registers: same op order.
template <bool F32>
__device__ __forceinline__ V3<typename Prec<F32>::T>
add_external_fe(const Params<typename Prec<F32>::T> &p, V3<typename Prec<F32>::T> a, V3<typename Prec<F32>::T> x,
                const typename Prec<F32>::T4 &v4, typename Prec<F32>::T mass, const typename Prec<F32>::T *fe) {
    using T = typename Prec<F32>::T;
    a.x = a.x + mass * p.g[0];
    a.y = a.y + mass * p.g[1];
    a.z = a.z + mass * p.g[2];
    if (p.F) {
        a.x = a.x + fe[0];
        a.y = a.y + fe[1];
        a.z = a.z + fe[2];
    }
    for (int q = 0; q < p.n_planes; ++q) {
        const T n0 = p.pn[q][0], n1 = p.pn[q][1], n2 = p.pn[q][2];
        const T depth = p.poff[q] - ((x.x * n0 + x.y * n1) + x.z * n2);
        if (!(depth > (T)0)) continue;
        const T fn = p.ppen[q] * depth;
        a.x = a.x + fn * n0;
        a.y = a.y + fn * n1;
        a.z = a.z + fn * n2;
        if (p.pfric[q] > (T)0) {
            const T vn = (v4.x * n0 + v4.y * n1) + v4.z * n2;
            const T tx = v4.x - vn * n0, ty = v4.y - vn * n1, tz = v4.z - vn * n2;
            const T speed = sqrt((tx * tx + ty * ty) + tz * tz);
            if (speed > (T)1e-15) {
                const T mag = fmin(p.pfric[q] * fn, (speed * mass) / p.dt);
                const T r = mag / speed;
                a.x = a.x - r * tx;
                a.y = a.y - r * ty;
                a.z = a.z - r * tz;
            }
        }
    }
    return a;
}

// CTA r of the cluster owns device slots [256 r, 256 r + 256).  Incidence
// word: partner (bits 0-11: a local position slot -- 0..255 own, 256 + k the
// k-th entry of this CTA's halo) | counts a degenerate spring (bit 12: this
// endpoint is the spring's lower caller id) | dictionary index << 13.
// Record image (engine.cu setup_resident), copied to shared memory:
//   shared part at 0: dict (fp64 double2 (k, l0); fp32 float4 (k, k*l0, Dx,
//     Dy), float4 (Dz, group bits, 0, 0)) [n_dict], then fp64 int32 groups
//   per CTA, at seg[r]: u32 n_halo, 3 x u32 pad, row u32 [257] (padded to
//     16 B), halo u32 [n_halo] (global device slots, padded), inc u32 [...]
// Shared memory of a CTA: positions T4 [2][pslots] (own 256, then halo) |
// dict | its segment.
struct ResidentArgs {
    const unsigned char *image;   // the record image
    const unsigned *seg;          // n_ctas + 1 segment byte offsets (multiples of 16)
    unsigned dict_bytes;          // shared part (dict + groups), multiple of 16
    int nd;                       // device slots
    int pslots;                   // position slots per CTA and parity (256 + max halo)
    int cur0;                     // X buffer holding the positions at the start
    long long count, step0;
    int bootstrap0;               // Verlet without x_prev at the first step
    int G;                        // actuation groups (scale row stride)
    unsigned off_dict, off_grp, off_seg;   // shared-memory byte offsets
};

// Spring sum of mass m by a group of G lanes (lane j = 0..G-1 of the group):
// round r evaluates incidences r*G + j side by side.  fp64: the group leader
// adds the G forces of a round in list order -- the serial spring-id order,
// bitwise -- skipping degenerate springs exactly like the reference; fp32:
// every lane sums its own incidences and the group reduces in a fixed order.
// The sum is returned to every lane of the group.
template <bool F32, int G>
__device__ __forceinline__ V3<typename Prec<F32>::T>
resident_spring_sum(const ResidentArgs &a, const unsigned char *smem, const uint32_t *row, const uint32_t *inc,
                    const typename Prec<F32>::T4 *xs, int m,   // m: local slot
                    const typename Prec<F32>::T4 &x4, const typename Prec<F32>::T *scale, int lane, unsigned gmask,
                    int leader, unsigned &deg) {
    using T = typename Prec<F32>::T;
    V3<T> s = {(T)0, (T)0, (T)0};
    const int q0 = (int)row[m], n = (int)row[m + 1] - q0;
    if constexpr (F32 && G == 1) {
        // one lane per mass: four partial sums (incidences q = 0, 1, 2, 3
        // mod 4) for instruction-level parallelism, combined in a fixed order
        const float4 *dict = reinterpret_cast<const float4 *>(smem + a.off_dict);
        V3<float> ps[4] = {{0.f, 0.f, 0.f}, {0.f, 0.f, 0.f}, {0.f, 0.f, 0.f}, {0.f, 0.f, 0.f}};
        auto term = [&](int q, V3<float> &acc) {
            const uint32_t e = inc[q0 + q];
            const float4 kd = dict[2 * (e >> 13)], ez = dict[2 * (e >> 13) + 1];
            float kl0 = kd.y;
            if (scale) {
                const int g = __float_as_int(ez.y);
                if (g >= 0) kl0 = kl0 * scale[g];
            }
            const float4 ro = xs[e & 0xfffu];
            const float dx = kd.z + (ro.x - x4.x), dy = kd.w + (ro.y - x4.y), dz = ez.x + (ro.z - x4.z);
            float d2;
            const float c = spring_c(dx, dy, dz, kd.x, kl0, d2);
            if (d2 < 1e-24f && (e & 0x1000u)) ++deg;
            acc.x = __fmaf_rn(c, dx, acc.x);
            acc.y = __fmaf_rn(c, dy, acc.y);
            acc.z = __fmaf_rn(c, dz, acc.z);
        };
        int q = 0;
        for (; q + 4 <= n; q += 4) {
#pragma unroll
            for (int u = 0; u < 4; ++u) term(q + u, ps[u]);
        }
        for (int u = 0; q < n; ++q, ++u) term(q, ps[u]);
        s.x = (ps[0].x + ps[1].x) + (ps[2].x + ps[3].x);
        s.y = (ps[0].y + ps[1].y) + (ps[2].y + ps[3].y);
        s.z = (ps[0].z + ps[1].z) + (ps[2].z + ps[3].z);
    } else if constexpr (F32) {
        const float4 *dict = reinterpret_cast<const float4 *>(smem + a.off_dict);
        for (int q = lane; q < n; q += G) {
            const uint32_t e = inc[q0 + q];
            const float4 kd = dict[2 * (e >> 13)], ez = dict[2 * (e >> 13) + 1];
            float kl0 = kd.y;
            if (scale) {
                const int g = __float_as_int(ez.y);
                if (g >= 0) kl0 = kl0 * scale[g];
            }
            const float4 ro = xs[e & 0xfffu];
            const float dx = kd.z + (ro.x - x4.x), dy = kd.w + (ro.y - x4.y), dz = ez.x + (ro.z - x4.z);
            float d2;
            const float c = spring_c(dx, dy, dz, kd.x, kl0, d2);
            if (d2 < 1e-24f && (e & 0x1000u)) ++deg;
            s.x = __fmaf_rn(c, dx, s.x);
            s.y = __fmaf_rn(c, dy, s.y);
            s.z = __fmaf_rn(c, dz, s.z);
        }
#pragma unroll
        for (int w = G / 2; w > 0; w >>= 1) {               // fixed-order tree over the group
            s.x = s.x + __shfl_down_sync(gmask, s.x, w, G);
            s.y = s.y + __shfl_down_sync(gmask, s.y, w, G);
            s.z = s.z + __shfl_down_sync(gmask, s.z, w, G);
        }
    } else if constexpr (G == 1) {
        // fp64, one lane per mass: the list in order, two incidences in
        // flight through tile_f64.cuh's branch-free IEEE fast paths; any
        // incidence outside them (or degenerate) redoes the mass with the
        // library operators, exactly as tile_f64_kernel does
        const double2 *dict = reinterpret_cast<const double2 *>(smem + a.off_dict);
        const int *dg = reinterpret_cast<const int *>(smem + a.off_grp);
        auto term = [&](uint32_t e, double &c, double &dx, double &dy, double &dz) -> bool {
            const double2 kl = dict[e >> 13];
            double l0 = kl.y;
            if (scale) {
                const int g = dg[e >> 13];
                if (g >= 0) l0 = l0 * scale[g];
            }
            const double4 xo = xs[e & 0xfffu];
            dx = xo.x - x4.x;
            dy = xo.y - x4.y;
            dz = xo.z - x4.z;
            bool ok_s, ok_d;
            const double len = sqrt_rn_fast((dx * dx + dy * dy) + dz * dz, ok_s);
            const double num = kl.x * (len - l0);
            c = div_rn_fast(num, len, ok_d);          // (a zero quotient's sign cannot reach the sum, tile_f64.cuh)
            const bool zero = (__double2hiint(num) & 0x7fffffff) == 0 && __double2loint(num) == 0;
            return ok_s && (ok_d || zero) && __double2hiint(len) > kDegenerateHi;
        };
        // kFly incidences in flight: a lone CTA per SM has the registers, and
        // the step's latency is this one lane's chain over its list
        constexpr int kFly = 4;
        bool ok = true;
        int q = 0;
        for (; q + kFly <= n; q += kFly) {
            double c[kFly], dx[kFly], dy[kFly], dz[kFly];
#pragma unroll
            for (int u = 0; u < kFly; ++u) ok &= term(inc[q0 + q + u], c[u], dx[u], dy[u], dz[u]);
#pragma unroll
            for (int u = 0; u < kFly; ++u) {
                s.x = s.x + c[u] * dx[u];
                s.y = s.y + c[u] * dy[u];
                s.z = s.z + c[u] * dz[u];
            }
        }
        for (; q < n; ++q) {
            double c0, x0, y0, z0;
            ok &= term(inc[q0 + q], c0, x0, y0, z0);
            s.x = s.x + c0 * x0;
            s.y = s.y + c0 * y0;
            s.z = s.z + c0 * z0;
        }
        if (!ok) {                                              // the exact loop (_kernels.py:51-70)
            s = {0.0, 0.0, 0.0};
            for (q = 0; q < n; ++q) {
                const uint32_t e = inc[q0 + q];
                const double2 kl = dict[e >> 13];
                double l0 = kl.y;
                if (scale) {
                    const int g = dg[e >> 13];
                    if (g >= 0) l0 = l0 * scale[g];
                }
                const double4 xo = xs[e & 0xfffu];
                const double dx = xo.x - x4.x, dy = xo.y - x4.y, dz = xo.z - x4.z;
                const double len = sqrt((dx * dx + dy * dy) + dz * dz);
                if (len < 1e-12) {
                    if (e & 0x1000u) ++deg;
                    continue;
                }
                const double c = spring_c64(kl.x, len, l0);
                s.x = s.x + c * dx;
                s.y = s.y + c * dy;
                s.z = s.z + c * dz;
            }
        }
        return s;
    } else {
        const double2 *dict = reinterpret_cast<const double2 *>(smem + a.off_dict);
        const int *dg = reinterpret_cast<const int *>(smem + a.off_grp);
        for (int r0 = 0; r0 < n; r0 += G) {
            const int q = r0 + lane;
            double fx = 0.0, fy = 0.0, fz = 0.0;
            bool add = false;
            if (q < n) {
                const uint32_t e = inc[q0 + q], di = e >> 13;
                const double2 kl = dict[di];
                double l0 = kl.y;
                if (scale) {
                    const int g = dg[di];
                    if (g >= 0) l0 = l0 * scale[g];
                }
                const double4 xo = xs[e & 0xfffu];
                const double dx = xo.x - x4.x, dy = xo.y - x4.y, dz = xo.z - x4.z;
                const double d2 = (dx * dx + dy * dy) + dz * dz;
                // the branch-free IEEE fast paths (tile_f64.cuh); a term outside
                // them is redone with the library operators -- terms are
                // independent, so the redo is per incidence
                bool ok_s, ok_d;
                const double lf = sqrt_rn_fast(d2, ok_s);
                const double num = kl.x * (lf - l0);
                double c = div_rn_fast(num, lf, ok_d);
                const bool zero = (__double2hiint(num) & 0x7fffffff) == 0 && __double2loint(num) == 0;
                add = ok_s && (ok_d || zero) && __double2hiint(lf) > kDegenerateHi;
                if (!add) {
                    const double len = sqrt(d2);
                    if (len < 1e-12) {                      // skipped and counted (_kernels.py:58-60)
                        if (e & 0x1000u) ++deg;
                    } else {
                        c = spring_c64(kl.x, len, l0);
                        add = true;
                    }
                }
                if (add) {
                    fx = c * dx;
                    fy = c * dy;
                    fz = c * dz;
                }
            }
            const unsigned ballot = __ballot_sync(gmask, add) >> leader;
#pragma unroll
            for (int i = 0; i < G; ++i) {                   // list order: s = s + f (the serial loop)
                const double gx = __shfl_sync(gmask, fx, i, G);
                const double gy = __shfl_sync(gmask, fy, i, G);
                const double gz = __shfl_sync(gmask, fz, i, G);
                if ((ballot >> i) & 1u) {
                    s.x = s.x + gx;
                    s.y = s.y + gy;
                    s.z = s.z + gz;
                }
            }
        }
    }
    s.x = __shfl_sync(gmask, s.x, 0, G);
    s.y = __shfl_sync(gmask, s.y, 0, G);
    s.z = __shfl_sync(gmask, s.z, 0, G);
    return s;
}

// INTEG: 0 Euler, 1 Verlet.  G lanes per mass slot: slot m = tid / G.
template <bool F32, int INTEG, int G>
__global__ void __launch_bounds__(G == 1 ? 256 : G == 2 ? 512 : 1024, 1) resident_kernel(Params<typename Prec<F32>::T> p,
                                                                        ResidentArgs a) {
    using T = typename Prec<F32>::T;
    using T4 = typename Prec<F32>::T4;
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    extern __shared__ __align__(16) unsigned char smem[];
    // divergence flag of each step, triple-buffered by step (mod 3): step s
    // sets flag[s%3] (in every CTA of the cluster) before its closing barrier,
    // every thread reads it after that barrier, and flag[(s+1)%3] is cleared
    // during step s -- after everyone has read it at step s-2, before anyone
    // can set it at step s+1 -- so all threads leave the loop at the same step
    __shared__ int diverged[3];
    __shared__ T sscale[2][kResidentMaxGroups];            // this and the next step's actuation scales
    T4 *const xsb = reinterpret_cast<T4 *>(smem);          // positions: [c * pslots + slot], c = step parity
    const unsigned rank = cl.block_rank(), n_ctas = cl.num_blocks();
    const int tid = threadIdx.x, bs = blockDim.x;
    const int l = tid / G, lane = tid % G;
    const int m = (int)rank * kResidentSlots + l;           // device slot
    const int leader = (tid & 31) & ~(G - 1);               // group's first lane within the warp
    const unsigned gmask = (G == 32 ? 0xffffffffu : ((1u << G) - 1u)) << leader;
    if (*p.div_step <= a.step0) return;                     // an earlier batch on the stream diverged (uniform)
    // stage the shared dictionary and this CTA's segment (16-byte copies)
    {
        uint4 *dst = reinterpret_cast<uint4 *>(smem + a.off_dict);
        const uint4 *src = reinterpret_cast<const uint4 *>(a.image);
        for (unsigned i = tid; i < a.dict_bytes / 16u; i += bs) dst[i] = __ldg(src + i);
        const unsigned s0 = __ldg(a.seg + rank), s1 = __ldg(a.seg + rank + 1);
        dst = reinterpret_cast<uint4 *>(smem + a.off_seg);
        src = reinterpret_cast<const uint4 *>(a.image + s0);
        for (unsigned i = tid; i < (s1 - s0) / 16u; i += bs) dst[i] = __ldg(src + i);
    }
    const T4 *X0 = a.cur0 ? p.Xout : p.X;                   // (host passes X[0] as X, X[1] as Xout)
    const bool in = l < kResidentSlots && m < a.nd;
    const bool act = in && (!p.orig_of || p.orig_of[m] >= 0);
    T4 x{}, v{}, hst{}, pb{};
    if (in) {
        x = X0[m];
        if (lane == 0) xsb[l] = x;
    }
    if (act) {
        v = p.V[m];
        if (INTEG == 1 && !a.bootstrap0) hst = p.Xprev[m];  // fp64: x_prev; fp32: u
        if constexpr (F32) pb = p.P[m];
    }
    if (tid < 3) diverged[tid] = 0;
    if (tid < a.G) sscale[0][tid] = p.scale[tid];
    T fe[3] = {(T)0, (T)0, (T)0};                           // f_ext is constant over a batch
    if (act && p.F) {
        const T4 f4 = p.F[m];
        fe[0] = f4.x;
        fe[1] = f4.y;
        fe[2] = f4.z;
    }
    if (n_ctas > 1) cl.sync();                              // every CTA's start positions and records staged
    else __syncthreads();
    const uint32_t *seg = reinterpret_cast<const uint32_t *>(smem + a.off_seg);
    const uint32_t n_halo = seg[0];
    const uint32_t *halo = seg + 4 + 260;                   // global device slots of this CTA's halo
    const uint32_t *srow = seg + 4;                         // rows, then incidences after the halo list
    const uint32_t *sinc = halo + ((n_halo + 3u) & ~3u);
    unsigned deg = 0;
    int c = 0;
    long long done = 0;
    int ph = 0;                                             // s % 3
    for (long long s = 0; s < a.count; ++s) {
        if (tid == 0) diverged[ph == 2 ? 0 : ph + 1] = 0;   // the next step's flag
        if (n_ctas > 1) {                                   // halo positions from their owners (DSMEM)
            T4 *cur = xsb + (c ? a.pslots : 0);
            for (uint32_t k = tid; k < n_halo; k += bs) {
                const uint32_t g = halo[k];
                cur[kResidentSlots + k] = *cl.map_shared_rank(cur + (g % kResidentSlots), g / kResidentSlots);
            }
            __syncthreads();
        }
        const T *scale = a.G ? sscale[s & 1] : nullptr;
        // the next step's scales, fetched now and published by this step's barrier
        T next_scale = (T)0;
        if (tid < a.G && s + 1 < a.count) next_scale = p.scale[(size_t)(s + 1) * a.G + tid];
        const bool boot = INTEG == 1 && s == 0 && a.bootstrap0;
        if (act) {                                          // (uniform within a group)
            const T4 x4 = x;
            const T mass = F32 ? (T)fabsf((float)x4.w) : (T)fabs((double)x4.w);
            const bool fixed = signbit(x4.w);
            const V3<T> sp = resident_spring_sum<F32, G>(a, smem, srow, sinc, xsb + (c ? a.pslots : 0), l, x4, scale,
                                                         lane, gmask, leader, deg);
            V3<T> xa = {x4.x, x4.y, x4.z};                  // absolute position (contact)
            if constexpr (F32) { xa.x = pb.x + xa.x; xa.y = pb.y + xa.y; xa.z = pb.z + xa.z; }
            const V3<T> f = add_external_fe<F32>(p, sp, xa, v, mass, fe);   // engine.py:273-288
            T xn[3], vn[3], un[3] = {(T)0, (T)0, (T)0};
            const T xc[3] = {x4.x, x4.y, x4.z};
            const T vc[3] = {v.x, v.y, v.z};
            const T fcv[3] = {f.x, f.y, f.z};
            if constexpr (INTEG == 0) {                     // engine.py:303-310
                const T dtm = p.dt / mass;
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    xn[k] = xc[k] + p.dt * vc[k];
                    vn[k] = vc[k] + dtm * fcv[k];
                    if (p.damped) vn[k] = vn[k] * p.one_minus_d;
                }
            } else {                                        // engine.py:312-328
                const T coef = p.dt2_over / mass;
                if constexpr (F32) {                        // increment form (kernels.cuh verlet_u)
                    const float u[3] = {hst.x, hst.y, hst.z};
#pragma unroll
                    for (int k = 0; k < 3; ++k) {
                        const float acc = coef * fcv[k];
                        if (boot) {
                            un[k] = p.dt * vc[k] + 0.5f * acc;
                            vn[k] = vc[k];
                        } else {
                            un[k] = (p.damped ? p.one_minus_d * u[k] : u[k]) + acc;
                            vn[k] = (un[k] + u[k]) / p.two_dt;
                        }
                        xn[k] = xc[k] + un[k];
                    }
                } else if (boot) {
#pragma unroll
                    for (int k = 0; k < 3; ++k) {
                        xn[k] = (xc[k] + p.dt * vc[k]) + (T)0.5 * (coef * fcv[k]);
                        vn[k] = vc[k];
                    }
                } else {
                    const T xp[3] = {hst.x, hst.y, hst.z};
#pragma unroll
                    for (int k = 0; k < 3; ++k) {
                        const T acc = coef * fcv[k];
                        if (p.damped) xn[k] = (xc[k] + p.one_minus_d * (xc[k] - xp[k])) + acc;
                        else          xn[k] = ((T)2 * xc[k] - xp[k]) + acc;
                        vn[k] = (xn[k] - xp[k]) / p.two_dt;
                    }
                }
            }
            if (fixed) {
#pragma unroll
                for (int k = 0; k < 3; ++k) { xn[k] = xc[k]; vn[k] = vc[k]; un[k] = (T)0; }
            }
            if constexpr (INTEG == 1) {
                if constexpr (F32) hst = T4{un[0], un[1], un[2], (T)0};
                else hst = x4;                              // x_prev of the next step
            }
            x.x = xn[0];
            x.y = xn[1];
            x.z = xn[2];
            v.x = vn[0];
            v.y = vn[1];
            v.z = vn[2];
            if (lane == 0) {
                xsb[(c ? 0 : a.pslots) + l] = x;
                if (!(finite3<F32>(xn[0], xn[1], xn[2]) && finite3<F32>(vn[0], vn[1], vn[2]))) {
                    for (unsigned r = 0; r < n_ctas; ++r) *cl.map_shared_rank(&diverged[ph], r) = 1;   // rare
                    atomicMin(p.div_mass, p.orig_of ? p.orig_of[m] : m);
                }
            }
        }
        if (tid < a.G) sscale[(s + 1) & 1][tid] = next_scale;
        if (n_ctas > 1) cl.sync();                          // this step's writes before the next step's reads
        else __syncthreads();
        c ^= 1;
        done = s + 1;
        if (diverged[ph]) {                                 // committed; the reference raises here
            if (tid == 0 && rank == 0) atomicMin(p.div_step, a.step0 + s + 1);
            break;
        }
        ph = ph == 2 ? 0 : ph + 1;
    }
    // write back: x into the buffer the host will call current, history,
    // velocities; padding slots keep their zeros
    if (act && lane == 0) {
        T4 *Xc = (a.cur0 ^ (int)(done & 1)) ? p.Xout : const_cast<T4 *>(p.X);
        T4 *Xo = (a.cur0 ^ (int)(done & 1)) ? const_cast<T4 *>(p.X) : p.Xout;
        Xc[m] = x;
        p.Vout[m] = v;
        if constexpr (INTEG == 1) {
            if constexpr (F32) p.U[m] = hst;
            else Xo[m] = hst;
        }
    }
    flush_degenerate(p.degenerate, deg);
}

}  // namespace ss
