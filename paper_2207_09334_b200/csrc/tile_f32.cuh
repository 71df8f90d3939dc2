// fp32 production-mode tile kernels (Euler / Verlet).  DESIGN.md §4.
//
// Both kernels evaluate every spring ONCE per tile it touches (spring-once),
// on the fp32 tile layout of tiles_f32.cpp:
//
//   owner pass      one thread per tile mass walks its own records (slot =
//                   q*256 + l): c = k - (k l0)/L, the term c*d is
//                   accumulated in registers and c is written back over the
//                   record's k in the tile's shared-memory copy;
//   foreign pass    springs whose owner lies in another tile are evaluated
//                   from the tile's copies, thread per record;
//   barrier
//   reference pass  each mass adds c * (y_owner - y_me): foreign references
//                   first, then in-tile ones, whose value IS the owner's
//                   slot -- one LDS c, one LDS.128 y, 3 FADD, 3 FFMA, no
//                   square root;
//   epilogue        external forces, Verlet / Euler, restore fixed,
//                   finiteness (integrate_store).
//
// The masses of a tile are ordered by their (foreign, own, in-tile) counts,
// so the lanes of a warp walk lists of (nearly) equal length.
//
// Positions are staged as tile-local y = (P - A) + r (kernels.cuh
// stage_tile): both endpoints of a spring see the same c and exactly
// opposite d, so Newton's third law holds bitwise; the summation order is
// fixed by the layout, so results are deterministic and identical between
// the two kernels.
//
//   tile_lean_kernel  one tile per CTA (256 threads, 3 CTAs per SM).
//   tile_ws_kernel    persistent, one CTA per SM, warp-specialized: producer
//                     warps stream tiles into a 3-stage shared-memory ring
//                     (TMA bulk copy of the records + cp.async gathers of the
//                     own and halo states), two consumer groups of 8 warps
//                     compute alternate tiles, so the record stream overlaps
//                     the arithmetic.
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

template <int INTEG, bool GROUPS>
__global__ void __launch_bounds__(kTile, 3) tile_lean_kernel(Params<float> p) {
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
            const float4 r = ldg4(p.X + gm), pp = ldg4(p.P + gm);
            sY[kTile + i] = make_float4((pp.x - A.x) + r.x, (pp.y - A.y) + r.y, (pp.z - A.z) + r.z, 0.f);
        }
    }
    mbar_wait_warp0(bar + 1, 0);                            // records (+ the staged states)
    V3<float> s = {0.f, 0.f, 0.f};
    float4 y = make_float4(0.f, 0.f, 0.f, 0.f);
    int n_ref = 0;
    if (active && p.debug != 1) {
        y = sY[l];
        const uint16_t cnt = reinterpret_cast<const uint16_t *>(bl + v.h->off_cnt)[l];
        n_ref = cnt >> 8;
        flush_degenerate(p.degenerate, owner_pass<GROUPS>(p, v, l, y, cnt & 0xff, s));
    }
    if (p.debug != 1) foreign_pass<GROUPS>(p, v, l, kTile);
    __syncthreads();                                        // every c written
    if (!active) return;
    if (p.debug != 1) ref_pass(v, l, y, n_ref, s);
    tile_epilogue<INTEG>(p, m, s, x4, hist, need_prev);
}

// ------------------------------------------------------------- persistent

constexpr int kWsProducers = 128;
constexpr int kWsStages = 3;
constexpr int kWsThreads = kWsProducers + 2 * kTile;

// Stage s of the ring: [blob (blob_smem) | X raw (256 + max_halo) | P raw
// (256 + max_halo)].  The producers' cp.async gathers land raw X and P; the
// consumers convert them in place into y (over the P slots) before use.
struct WsGeom {
    uint32_t stage_bytes, blob_smem, slots;
    __device__ __forceinline__ unsigned char *blob(unsigned char *smem, int s) const {
        return smem + 128 + (size_t)s * stage_bytes;
    }
    __device__ __forceinline__ float4 *xraw(unsigned char *smem, int s) const {
        return reinterpret_cast<float4 *>(blob(smem, s) + blob_smem);
    }
    __device__ __forceinline__ float4 *praw(unsigned char *smem, int s) const {
        return xraw(smem, s) + slots;
    }
};

__host__ __device__ inline size_t ws_stage_bytes(size_t blob_smem, size_t max_halo) {
    return (blob_smem + 2 * (kTile + max_halo) * sizeof(float4) + 127u) & ~(size_t)127u;
}

// Barriers:
//   mbarrier [3s]   header + halo ids of stage s (TMA)
//   mbarrier [3s+1] records of stage s (TMA)
//   mbarrier [3s+2] cp.async gathers of stage s: one arrival per producer thread
//   named FULL[s] = 1+s is not needed: consumers wait on the mbarriers directly
//   named EMPTY[s] = 4+s: 256 consumer arrivals + 128 producer syncs
//   named GROUP[g] = 7+g: the 256 threads of a consumer group
//   named PROD = 9: the 128 producer threads
template <int INTEG, bool GROUPS>
__global__ void __launch_bounds__(kWsThreads, 1) tile_ws_kernel(Params<float> p) {
    extern __shared__ __align__(128) unsigned char smem[];
    if (*p.div_step < p.step) return;                       // grid-uniform
    const Topology<float> &t = p.topo;
    const int tid = threadIdx.x;
    const int G = (int)gridDim.x;
    const int b = (int)blockIdx.x;
    const int n_mine = (t.n_tiles - b + G - 1) / G;
    const WsGeom geo{(uint32_t)ws_stage_bytes(t.blob_smem, t.max_halo), t.blob_smem, kTile + t.max_halo};
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem);
    if (tid == 0) {
        for (int i = 0; i < kWsStages; ++i) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar + 3 * i)));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar + 3 * i + 1)));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar + 3 * i + 2)),
                         "r"(kWsProducers));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (tid < kWsProducers) {
        // ------------------------------------------------------------ producers
        // Tile k: TMA its blob, cp.async its own states, then (header landed)
        // cp.async its halo states.  Nothing here waits for data except the
        // 1.3 KB header; the consumers wait on the three mbarriers.
        long long t0 = prof_clock();
        const bool pw = tid == 0;
        for (int k = 0; k < n_mine; ++k) {
            const int s = k % kWsStages;
            const uint32_t phase = (uint32_t)(k / kWsStages) & 1u;
            const int T = b + k * G;
            if (k >= kWsStages) named_sync(4 + s, kWsProducers + kTile);   // stage released
            prof_add(p, pw, 0, t0);                         // [0] producer: waiting for a free stage
            unsigned char *bl = geo.blob(smem, s);
            if (tid == 0) {
                const int tb = p.debug == 2 ? 0 : T;
                const unsigned long long g0 = t.toff[tb];
                const uint32_t bytes = (uint32_t)(t.toff[tb + 1] - g0);
                const uint32_t split = t.tsplit[tb] & 0xffffffu;
                bulk_copy(bl, t.blob + g0, split, bar + 3 * s);
                bulk_copy(bl + split, t.blob + g0 + split, bytes - split, bar + 3 * s + 1);
            }
            float4 *xr = geo.xraw(smem, s), *pr = geo.praw(smem, s);
            const int n = (int)(__ldg(t.tsplit + T) >> 24) + 1;
            for (int i = tid; i < n; i += kWsProducers) {   // own states: no dependency
                cp_async16(xr + i, p.X + T * kTile + i);
                cp_async16(pr + i, p.P + T * kTile + i);
            }
            prof_add(p, pw, 1, t0);                         // [1] producer: TMA + own gathers issued
            if (tid < 32) mbar_wait(bar + 3 * s, phase);   // header + halo ids
            named_sync(9, kWsProducers);
            prof_add(p, pw, 2, t0);                         // [2] producer: waiting for the header
            const TileHdr *h = reinterpret_cast<const TileHdr *>(bl);
            const int *halo = reinterpret_cast<const int *>(bl + h->off_halo);
            const int nh = (int)h->n_halo;
            for (int i = tid; i < nh; i += kWsProducers) {
                const int gm = halo[i];
                cp_async16(xr + kTile + i, p.X + gm);
                cp_async16(pr + kTile + i, p.P + gm);
            }
            cp_async_mbar_arrive(bar + 3 * s + 2);          // fires when this thread's copies land
            prof_add(p, pw, 3, t0);                         // [3] producer: halo gathers issued
        }
        // drain the releases of the last stages so no named barrier is left
        // with pending arrivals when the CTA exits
        for (int k = n_mine > kWsStages ? n_mine - kWsStages : 0; k < n_mine; ++k)
            named_sync(4 + k % kWsStages, kWsProducers + kTile);
        return;
    }

    // ---------------------------------------------------------------- consumers
    const int c = tid - kWsProducers;
    const int g = c >> 8;                                   // consumer group
    const int l = c & (kTile - 1);
    const bool need_prev = INTEG == 1 && !p.bootstrap;
    unsigned deg = 0;
    long long t0 = prof_clock();
    const bool cw = l == 0;
    for (int k = g; k < n_mine; k += 2) {
        const int s = k % kWsStages;
        const uint32_t phase = (uint32_t)(k / kWsStages) & 1u;
        const int T = b + k * G;
        const int m = T * kTile + l;
        const int n = (int)(__ldg(t.tsplit + T) >> 24) + 1;
        const bool active = l < n;
        float4 hist = make_float4(0.f, 0.f, 0.f, 0.f);     // epilogue history, prefetched
        if (active) hist = need_prev ? ldg4(p.Xprev + m) : ldg4(p.V + m);
        unsigned char *bl = geo.blob(smem, s);
        float4 *xr = geo.xraw(smem, s), *pr = geo.praw(smem, s);
        mbar_wait(bar + 3 * s + 2, phase);                  // own + halo states landed
        mbar_wait(bar + 3 * s, phase);                      // header (halo count)
        prof_add(p, cw, 4, t0);                             // [4] consumer: waiting for the states
        const TileView v0 = tile_view(bl, pr);
        {                                                   // y = (P - A) + r, in place over P
            const float4 A = pr[(n - 1) / 2];
            const int ns = kTile + (int)v0.h->n_halo;
            named_sync(7 + g, kTile);                       // A read before anyone overwrites it
            for (int i = l; i < ns; i += kTile) {
                if (i >= n && i < kTile) continue;
                const float4 r = xr[i], pp = pr[i];
                pr[i] = make_float4((pp.x - A.x) + r.x, (pp.y - A.y) + r.y, (pp.z - A.z) + r.z, r.w);
            }
        }
        const float4 x4 = active ? xr[l] : make_float4(0.f, 0.f, 0.f, 0.f);
        prof_add(p, cw, 5, t0);                             // [5] consumer: y conversion
        mbar_wait(bar + 3 * s + 1, phase);                  // records
        named_sync(7 + g, kTile);                           // every y converted
        prof_add(p, cw, 6, t0);                             // [6] consumer: waiting for records + group
        const TileView v = v0;
        V3<float> sum = {0.f, 0.f, 0.f};
        float4 y = make_float4(0.f, 0.f, 0.f, 0.f);
        int n_ref = 0;
        if (active && p.debug != 1) {
            y = v.sY[l];
            const uint16_t cnt = reinterpret_cast<const uint16_t *>(bl + v.h->off_cnt)[l];
            n_ref = cnt >> 8;
            deg += owner_pass<GROUPS>(p, v, l, y, cnt & 0xff, sum);
        }
        prof_add(p, cw, 7, t0);                             // [7] consumer: owner pass
        if (p.debug != 1) foreign_pass<GROUPS>(p, v, l, kTile);
        prof_add(p, cw, 8, t0);                             // [8] consumer: foreign pass
        named_sync(7 + g, kTile);                           // every c of the tile written
        prof_add(p, cw, 9, t0);                             // [9] consumer: group barrier
        if (active && p.debug != 1) ref_pass(v, l, y, n_ref, sum);
        prof_add(p, cw, 10, t0);                            // [10] consumer: reference pass
        // generic-proxy writes (c over k, y over P) must be ordered before the
        // next async-proxy (TMA / cp.async) writes into this stage
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        named_arrive(4 + s, kWsProducers + kTile);          // stage free for tile k + 3
        if (active) tile_epilogue<INTEG>(p, m, sum, x4, hist, need_prev);
        prof_add(p, cw, 11, t0);                            // [11] consumer: epilogue
    }
    flush_degenerate(p.degenerate, deg);
}

}  // namespace ss
