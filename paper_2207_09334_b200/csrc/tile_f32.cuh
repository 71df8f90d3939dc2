// fp32 production-mode tile kernels (Euler / Verlet).  DESIGN.md §4.
//
// tile_lean_kernel: one tile (256 masses) per CTA of 256 threads; the tile
// blob is TMA-bulk-copied into shared memory while the own states load and
// the halo positions are gathered once as tile-local y = (P - A) + r; then
//
//   compact format (tiles.h, the default): each thread walks its mass's
//     incidence list (partner slot, dictionary index) and sums
//     c*d, c = k - (k l0)/L, evaluating each spring from both endpoints --
//     no barrier, no written state, 2 B per incidence streamed;
//   explicit format (fallback when a tile has > 64 distinct records):
//     spring-once passes -- owner pass (c written over the record's k),
//     foreign pass over the copies of cross-tile springs, barrier, reference
//     pass adding c * (y_owner - y_me);
//
// then the fused epilogue: external forces, Verlet / Euler, restore fixed,
// finiteness (integrate_store).
//
// Positions are staged as tile-local y = (P - A) + r (kernels.cuh
// stage_tile): both endpoints of a spring see the same c and exactly
// opposite d, so Newton's third law holds bitwise; the summation order is
// fixed by the layout, so results are deterministic.
//
// Record format of fp32 tile builds (tiles_f32.cpp): k and k*l0 in fp32
// (planar), so c = k (L - l0)/L = fma(-(k l0), 1/L, k): one FFMA after the
// reciprocal square root (same rounding sensitivity as k (L - l0)/L: both
// are limited by the fp32 ulp of L).
#pragma once

#include "kernels.cuh"

namespace ss {

// --------------------------------------------------------------- primitives

__device__ __forceinline__ void cp_async16(void *dst, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
// arrive on an mbarrier when all of this thread's prior cp.async have landed
// (counts as one of the barrier's expected arrivals)
__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t *bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void named_sync(int id, int count) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void named_arrive(int id, int count) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// SS_PROF phase timing: thread `who` adds the cycles since `t0` to slot i.
__device__ __forceinline__ long long prof_clock() { return clock64(); }
__device__ __forceinline__ void prof_add(const Params<float> &p, bool who, int i, long long &t0) {
    if (p.prof && who) {
        const long long t1 = clock64();
        atomicAdd(p.prof + i, (unsigned long long)(t1 - t0));
        t0 = t1;
    }
}

__device__ __forceinline__ float rsqrt_ftz(float x) {
    float r;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// c = k - (k l0) / L for endpoint offset d: rsqrt + one Newton step.
// Degenerate springs (L < 1e-12, _kernels.py:58-60) give c = 0; NaN
// propagates like the reference's arithmetic.  d2 is returned for the
// caller's degenerate bookkeeping.
__device__ __forceinline__ float spring_c(float dx, float dy, float dz, float k, float kl0, float &d2) {
    d2 = __fmaf_rn(dz, dz, __fmaf_rn(dy, dy, __fmul_rn(dx, dx)));
    float inv = rsqrt_ftz(d2);
    inv = __fmul_rn(inv, __fmaf_rn(__fmul_rn(-0.5f, d2), __fmul_rn(inv, inv), 1.5f));
    const float c = __fmaf_rn(-kl0, inv, k);
    return d2 < 1e-24f ? 0.0f : c;
}

// External forces + Euler/Verlet update + restore fixed + store + finiteness
// check of device mass m (engine.py:273-328, 297-301, 375-381).
template <int INTEG>
__device__ __forceinline__ void integrate_store(const Params<float> &p, int m, V3<float> sum, float4 x4,
                                                float4 p4, float4 v4, float4 xp4, bool need_prev) {
    const float mass = fabsf(x4.w);
    const bool fixed = signbit(x4.w);
    const V3<float> xa = {p4.x + x4.x, p4.y + x4.y, p4.z + x4.z};
    const V3<float> f = add_external<true>(p, m, sum, xa, v4, mass);
    float xn[3], vn[3];
    const float x[3] = {x4.x, x4.y, x4.z};
    const float v[3] = {v4.x, v4.y, v4.z};
    const float fc[3] = {f.x, f.y, f.z};
    if constexpr (INTEG == 0) {
        const float dtm = p.dt / mass;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            xn[c] = x[c] + p.dt * v[c];
            vn[c] = v[c] + dtm * fc[c];
            if (p.damped) vn[c] = vn[c] * p.one_minus_d;
        }
    } else {
        const float coef = p.dt2_over / mass;
        if (!need_prev) {
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                xn[c] = (x[c] + p.dt * v[c]) + 0.5f * (coef * fc[c]);
                vn[c] = v[c];
            }
        } else {
            const float xp[3] = {xp4.x, xp4.y, xp4.z};
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const float acc = coef * fc[c];
                if (p.damped) xn[c] = (x[c] + p.one_minus_d * (x[c] - xp[c])) + acc;
                else          xn[c] = (2.f * x[c] - xp[c]) + acc;
                vn[c] = (xn[c] - xp[c]) / p.two_dt;
            }
        }
    }
    if (fixed) {
#pragma unroll
        for (int c = 0; c < 3; ++c) { xn[c] = x[c]; vn[c] = v[c]; }
    }
    p.Xout[m] = make_float4(xn[0], xn[1], xn[2], x4.w);
    p.Vout[m] = make_float4(vn[0], vn[1], vn[2], 0.f);
    if (!(finite3<true>(xn[0], xn[1], xn[2]) && finite3<true>(vn[0], vn[1], vn[2])))
        flag_divergence<true>(p, m);
}

// ------------------------------------------------------------ tile passes

struct TileView {
    unsigned char *bl;           // the tile blob in shared memory
    const TileHdr *h;
    const float4 *sY;            // staged y: [0, 256) own masses, [256, ...) halo
};

__device__ __forceinline__ TileView tile_view(unsigned char *bl, const float4 *sY) {
    return TileView{bl, reinterpret_cast<const TileHdr *>(bl), sY};
}

__device__ __forceinline__ void acc3(V3<float> &s, float c, float dx, float dy, float dz) {
    s.x = __fmaf_rn(c, dx, s.x);
    s.y = __fmaf_rn(c, dy, s.y);
    s.z = __fmaf_rn(c, dz, s.z);
}

// ------------------------------------------------- explicit format passes

// Owner pass of tile mass l: its own records (slot q*256 + l).
// Accumulates c*d, writes c over k (the in-tile partners read it in
// ref_pass), and returns the number of degenerate own springs (counted once
// per spring per evaluation, by the owner, like _kernels.py:58-60).
template <bool GROUPS>
__device__ __forceinline__ unsigned owner_pass(const Params<float> &p, const TileView &v, int l, const float4 &y,
                                               int n_own, V3<float> &s) {
    const uint16_t *oo = reinterpret_cast<const uint16_t *>(v.bl + v.h->off_oo) + l;
    float *ok = reinterpret_cast<float *>(v.bl + v.h->off_okl) + l;
    const float *okl0 = ok + (v.h->W << 8);
    const int8_t *og = GROUPS && v.h->off_og ? reinterpret_cast<const int8_t *>(v.bl + v.h->off_og) + l : nullptr;
    float dmin = INFINITY;
    auto body = [&](int q) {
        const float k = ok[q << 8];
        float kl0 = okl0[q << 8];
        if constexpr (GROUPS) {
            if (og) {
                const int g = og[q << 8];
                if (g >= 0) kl0 = kl0 * p.scale[g];
            }
        }
        const float4 yo = v.sY[oo[q << 8]];
        const float dx = yo.x - y.x, dy = yo.y - y.y, dz = yo.z - y.z;
        float d2;
        const float c = spring_c(dx, dy, dz, k, kl0, d2);
        dmin = fminf(dmin, d2);
        acc3(s, c, dx, dy, dz);
        ok[q << 8] = c;
    };
    int q = 0;
#pragma unroll 1
    for (; q + 3 < n_own; q += 4) {
        body(q);
        body(q + 1);
        body(q + 2);
        body(q + 3);
    }
#pragma unroll 1
    for (; q < n_own; ++q) body(q);
    unsigned deg = 0;
    if (dmin < 1e-24f) {                                    // rare: count the degenerate ones
        for (int r = 0; r < n_own; ++r) {
            const float4 yo = v.sY[oo[r << 8]];
            const float dx = yo.x - y.x, dy = yo.y - y.y, dz = yo.z - y.z;
            const float d2 = __fmaf_rn(dz, dz, __fmaf_rn(dy, dy, __fmul_rn(dx, dx)));
            deg += d2 < 1e-24f ? 1u : 0u;
        }
    }
    return deg;
}

// Foreign copies, thread per record (f = i0, i0 + stride, ...): c of the
// springs whose owner lies in another tile, written over the copy's k.
template <bool GROUPS>
__device__ __forceinline__ void foreign_pass(const Params<float> &p, const TileView &v, int i0, int stride) {
    const int nf = (int)v.h->n_foreign;
    const uint16_t *fo = reinterpret_cast<const uint16_t *>(v.bl + v.h->off_fo);
    const uint8_t *fl = v.bl + v.h->off_fl;
    float *fk = reinterpret_cast<float *>(v.bl + v.h->off_fkl);
    const float *fkl0 = fk + nf;
    const int8_t *fg = GROUPS && v.h->off_fg ? reinterpret_cast<const int8_t *>(v.bl + v.h->off_fg) : nullptr;
#pragma unroll 1
    for (int f = i0; f < nf; f += stride) {
        const float k = fk[f];
        float kl0 = fkl0[f];
        if constexpr (GROUPS) {
            if (fg) {
                const int g = fg[f];
                if (g >= 0) kl0 = kl0 * p.scale[g];
            }
        }
        const float4 ya = v.sY[fl[f]], yo = v.sY[fo[f]];
        float d2;
        fk[f] = spring_c(yo.x - ya.x, yo.y - ya.y, yo.z - ya.z, k, kl0, d2);   // counted by the owner tile
    }
}

// Reference pass of tile mass l: s += c * (y_owner - y_me), foreign
// references first (n_for of them), then in-tile ones (value = owner slot).
__device__ __forceinline__ void ref_pass(const TileView &v, int l, const float4 &y, int n_ref, V3<float> &s) {
    const uint16_t *rf = reinterpret_cast<const uint16_t *>(v.bl + v.h->off_ref) + l;
    const uint16_t *fo = reinterpret_cast<const uint16_t *>(v.bl + v.h->off_fo);
    const float *fk = reinterpret_cast<const float *>(v.bl + v.h->off_fkl);
    const float *ok = reinterpret_cast<const float *>(v.bl + v.h->off_okl);
    const int n_for = (v.bl + v.h->off_nf)[l];
    auto fbody = [&](int q) {
        const uint32_t f = rf[q << 8] & 0x7fffu;
        const float c = fk[f];
        const float4 yo = v.sY[fo[f]];
        acc3(s, c, yo.x - y.x, yo.y - y.y, yo.z - y.z);
    };
    auto ibody = [&](int q) {
        const uint32_t r = rf[q << 8];
        const float c = ok[r];
        const float4 yo = v.sY[r & 0xffu];
        acc3(s, c, yo.x - y.x, yo.y - y.y, yo.z - y.z);
    };
    int q = 0;
#pragma unroll 1
    for (; q + 3 < n_for; q += 4) {
        fbody(q);
        fbody(q + 1);
        fbody(q + 2);
        fbody(q + 3);
    }
#pragma unroll 1
    for (; q < n_for; ++q) fbody(q);
#pragma unroll 1
    for (; q + 3 < n_ref; q += 4) {
        ibody(q);
        ibody(q + 1);
        ibody(q + 2);
        ibody(q + 3);
    }
#pragma unroll 1
    for (; q < n_ref; ++q) ibody(q);
}

// -------------------------------------------------- compact format pass

// Spring sum of tile mass l over its incidence list (tiles.h compact
// format: u16 = partner slot | dictionary index << 10, own springs first).
// Each spring is evaluated from both of its endpoints; the two evaluations
// see exactly opposite d and the same c, so Newton's third law holds
// bitwise.  Returns the number of degenerate own springs.
template <bool GROUPS>
__device__ __forceinline__ unsigned incidence_sum(const Params<float> &p, const TileView &v, int l, const float4 &y,
                                                  int n_own, int n_inc, V3<float> &s) {
    const uint16_t *inc = reinterpret_cast<const uint16_t *>(v.bl + v.h->off_oo) + l;
    const float2 *dict = reinterpret_cast<const float2 *>(v.bl + v.h->off_okl);
    const int8_t *dg = GROUPS && v.h->off_og ? reinterpret_cast<const int8_t *>(v.bl + v.h->off_og) : nullptr;
    float dmin = INFINITY;
    auto body = [&](int q) {
        const uint32_t e = inc[q << 8];
        const uint32_t mi = e >> 10;
        float2 kl = dict[mi];
        if constexpr (GROUPS) {
            if (dg) {
                const int g = dg[mi];
                if (g >= 0) kl.y = kl.y * p.scale[g];
            }
        }
        const float4 yo = v.sY[e & 0x3ffu];
        const float dx = yo.x - y.x, dy = yo.y - y.y, dz = yo.z - y.z;
        float d2;
        const float c = spring_c(dx, dy, dz, kl.x, kl.y, d2);
        dmin = fminf(dmin, d2);                             // a degenerate reference is also degenerate at its owner
        acc3(s, c, dx, dy, dz);
    };
    int q = 0;
#pragma unroll 1
    for (; q + 3 < n_inc; q += 4) {
        body(q);
        body(q + 1);
        body(q + 2);
        body(q + 3);
    }
#pragma unroll 1
    for (; q < n_inc; ++q) body(q);
    unsigned deg = 0;
    if (dmin < 1e-24f) {                                    // rare: count the degenerate own springs
        for (int r = 0; r < n_own; ++r) {
            const float4 yo = v.sY[inc[r << 8] & 0x3ffu];
            const float dx = yo.x - y.x, dy = yo.y - y.y, dz = yo.z - y.z;
            const float d2 = __fmaf_rn(dz, dz, __fmaf_rn(dy, dy, __fmul_rn(dx, dx)));
            deg += d2 < 1e-24f ? 1u : 0u;
        }
    }
    return deg;
}

// Epilogue of tile mass l (device id m): the history vector the integrator
// needs (x_prev for Verlet, v otherwise) was prefetched; v is read only to
// bootstrap, for friction, or to restore a fixed mass; P only for contact.
template <int INTEG>
__device__ __forceinline__ void tile_epilogue(const Params<float> &p, int m, const V3<float> &s, const float4 &x4,
                                              const float4 &hist, bool need_prev) {
    float4 v4 = need_prev ? make_float4(0.f, 0.f, 0.f, 0.f) : hist;
    if (need_prev && (p.n_planes > 0 || signbit(x4.w))) v4 = p.V[m];
    float4 p4 = make_float4(0.f, 0.f, 0.f, 0.f);
    if (p.n_planes > 0) p4 = p.P[m];
    integrate_store<INTEG>(p, m, s, x4, p4, v4, hist, need_prev);
}

// ------------------------------------------------------------------ lean

__device__ __forceinline__ void mbar_wait_warp0(uint64_t *bar, uint32_t phase) {
    if (threadIdx.x < 32) mbar_wait(bar, phase);
    __syncthreads();
}

template <int INTEG, bool GROUPS, int FMT, int MINB = (FMT == 1 ? 5 : 3)>
__global__ void __launch_bounds__(kTile, MINB) tile_lean_kernel(Params<float> p) {
    extern __shared__ __align__(128) unsigned char smem[];
    if (*p.div_step < p.step) return;                       // grid-uniform
    const Topology<float> &t = p.topo;
    const int l = threadIdx.x;
    const int m = blockIdx.x * kTile + l;
    const int n = (int)(__ldg(t.tsplit + blockIdx.x) >> 24) + 1;
    const bool active = l < n;
    const bool need_prev = INTEG == 1 && !p.bootstrap;
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem);
    unsigned char *bl = smem + 128;
    float4 *sY = reinterpret_cast<float4 *>(bl + t.blob_smem);
    if (l == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar + 1)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (l == 0) {
        const int tb = p.debug == 2 ? 0 : blockIdx.x;       // debug 2: every CTA stages tile 0 (L2-resident)
        const unsigned long long g0 = t.toff[tb];
        const uint32_t bytes = (uint32_t)(t.toff[tb + 1] - g0);
        const uint32_t split = t.tsplit[tb] & 0xffffffu;
        bulk_copy(bl, t.blob + g0, split, bar);
        bulk_copy(bl + split, t.blob + g0 + split, bytes - split, bar + 1);
    }
    const float4 A = ldg4(p.P + blockIdx.x * kTile + (n - 1) / 2);
    float4 x4 = make_float4(0.f, 0.f, 0.f, 0.f), hist = x4;
    if (active) {
        x4 = ldg4(p.X + m);
        hist = need_prev ? ldg4(p.Xprev + m) : ldg4(p.V + m);
        const float4 pp = ldg4(p.P + m);
        sY[l] = make_float4((pp.x - A.x) + x4.x, (pp.y - A.y) + x4.y, (pp.z - A.z) + x4.z, x4.w);
    }
    mbar_wait_warp0(bar, 0);                                // header + halo ids
    const TileView v = tile_view(bl, sY);
    {
        const int *halo = reinterpret_cast<const int *>(bl + v.h->off_halo);
        const int nh = (int)v.h->n_halo;
#pragma unroll 1
        for (int i = l; i < nh; i += kTile) {
            const int gm = halo[i];
            if (gm < 0) continue;                           // hole of the bank-aware halo layout
            const float4 r = ldg4(p.X + gm), pp = ldg4(p.P + gm);
            sY[kTile + i] = make_float4((pp.x - A.x) + r.x, (pp.y - A.y) + r.y, (pp.z - A.z) + r.z, 0.f);
        }
    }
    mbar_wait_warp0(bar + 1, 0);                            // records (+ the staged states)
    V3<float> s = {0.f, 0.f, 0.f};
    if constexpr (FMT == 1) {                               // compact: one pass, no further barrier
        if (!active) return;
        if (p.debug != 1) {
            const uint16_t cnt = reinterpret_cast<const uint16_t *>(bl + v.h->off_cnt)[l];
            flush_degenerate(p.degenerate, incidence_sum<GROUPS>(p, v, l, sY[l], cnt & 0xff, cnt >> 8, s));
        }
    } else {                                                // explicit: spring-once passes
        float4 y = make_float4(0.f, 0.f, 0.f, 0.f);
        int n_ref = 0;
        if (active && p.debug != 1) {
            y = sY[l];
            const uint16_t cnt = reinterpret_cast<const uint16_t *>(bl + v.h->off_cnt)[l];
            n_ref = cnt >> 8;
            flush_degenerate(p.degenerate, owner_pass<GROUPS>(p, v, l, y, cnt & 0xff, s));
        }
        if (p.debug != 1) foreign_pass<GROUPS>(p, v, l, kTile);
        __syncthreads();                                    // every c written
        if (!active) return;
        if (p.debug != 1) ref_pass(v, l, y, n_ref, s);
    }
    tile_epilogue<INTEG>(p, m, s, x4, hist, need_prev);
}

}  // namespace ss
