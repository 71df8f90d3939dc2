// Record-pass tile kernel (fp32 production mode, Euler / Verlet).  DESIGN.md §4.
//
// A tile of 256 masses (one CTA of 512 threads) is staged as in kernels.cuh
// (TMA bulk copy of the tile's records, halo positions gathered once into
// shared memory as tile-local y = (P - A) + r).  The springs are then
// evaluated once per tile, spring-parallel, and summed mass-parallel:
//
//   record pass  thread-per-record over the tile's own record slots
//                (slot = q*256 + owner) and its foreign record copies:
//                c = k (L - l0) / L from the two staged endpoint positions,
//                written over the record's k in shared memory.  Uniform work,
//                no per-mass divergence; padding slots point at their own
//                mass (d = 0 -> c = 0, not counted as degenerate).
//   barrier
//   mass pass    two adjacent lanes per mass split its incidence list (own
//                records, then references; an in-tile reference value is the
//                owner's slot, a foreign one indexes the copies) and combine
//                with one shuffle.  Every incidence adds c * (y_partner - y_me):
//                one LDS c, one LDS.128 y, 3 FADD, 3 FFMA, no square root.
//   then the even lane runs the fused integrator epilogue (external forces,
//   Verlet/Euler, restore fixed, finiteness); the history vector it needs
//   (x_prev or v) was streamed into shared memory by cp.async at the start.
//
// Both endpoints of a spring see the same c and exactly opposite d (the
// staged tile-local frame is shared), so Newton's third law holds bitwise.
// Summation order is fixed by the layout, so results are deterministic.
// Springs crossing a tile boundary are evaluated once in each of the two
// tiles (the foreign copies: ~30% of references on the 10M cube).
//
// Requires an fp32 tile build (tiles.h: slice_log2 == 8, padding slots
// self-pointing, foreign partners in off_fl) without self-springs.
#pragma once

#include "pipe_kernel.cuh"

namespace ss {

__device__ __forceinline__ float rsqrt_ftz(float x) {
    float r;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// c = k (L - l0) / L of one spring with endpoint offset d (d2 = |d|^2):
// rsqrt + one Newton step (L to ~1 ulp), branch-free degenerate handling.
__device__ __forceinline__ float spring_coef(float dx, float dy, float dz, float k, float l0, bool &ok) {
    const float d2 = __fmaf_rn(dz, dz, __fmaf_rn(dy, dy, __fmul_rn(dx, dx)));
    float inv = rsqrt_ftz(d2);
    inv = __fmul_rn(inv, __fmaf_rn(__fmul_rn(-0.5f, d2), __fmul_rn(inv, inv), 1.5f));
    const float len = __fmul_rn(d2, inv);
    ok = d2 >= 1e-24f;
    return ok ? __fmul_rn(__fmul_rn(k, len - l0), inv) : 0.0f;
}

template <int INTEG, bool GROUPS>
__global__ void __launch_bounds__(kPipeThreads, 3) tile_fast_kernel(Params<float> p) {
    extern __shared__ __align__(128) unsigned char smem[];
    if (*p.div_step < p.step) return;                       // grid-uniform
    const Topology<float> &t = p.topo;
    const int tid = threadIdx.x;
    const int role = tid & 1;                               // lanes 2j, 2j+1 share mass j
    const int l = tid >> 1;
    const int m = blockIdx.x * kTile + l;
    const int n = (int)(__ldg(t.tsplit + blockIdx.x) >> 24) + 1;
    const bool active = l < n;
    const bool lead = active && role == 0;
    const bool need_prev = INTEG == 1 && !p.bootstrap;
    // Verlet reads v only to bootstrap, for friction, or to restore a fixed mass;
    // the one history vector the integrator needs streams into shared memory
    // (cp.async) while the tile stages, without holding registers.
    float4 *sHist = reinterpret_cast<float4 *>(smem + 128 + t.blob_smem) + (kTile + t.max_halo);
    if (lead) cp_async16(sHist + l, need_prev ? p.Xprev + m : p.V + m);
    cp_async_commit();
    const TileCtx<true> ctx = stage_tile<true>(p, smem, m, lead, l);
    const TileHdr *h = ctx.h;
    unsigned char *bl = const_cast<unsigned char *>(ctx.blob);
    const float4 *sX = ctx.sX;
    const uint16_t *oo = reinterpret_cast<const uint16_t *>(bl + h->off_oo);
    float2 *okl = reinterpret_cast<float2 *>(bl + h->off_okl);
    const uint16_t *fo = reinterpret_cast<const uint16_t *>(bl + h->off_fo);
    float2 *fkl = reinterpret_cast<float2 *>(bl + h->off_fkl);

    // ---- record pass: c of every own record slot and foreign copy
    if (p.debug != 1) {
        unsigned deg = 0;
        const int n_slots = (int)h->W << 8;
        const int8_t *og = GROUPS && h->off_og ? reinterpret_cast<const int8_t *>(bl + h->off_og) : nullptr;
        for (int s = tid; s < n_slots; s += kPipeThreads) {
            const int a = s & (kTile - 1);
            const int o = oo[s];
            const float2 kl = okl[s];
            float l0 = kl.y;
            if constexpr (GROUPS) {
                if (og) {
                    const int g = og[s];
                    if (g >= 0) l0 = l0 * p.scale[g];
                }
            }
            const float4 ya = sX[a], yo = sX[o];
            bool ok;
            const float c = spring_coef(yo.x - ya.x, yo.y - ya.y, yo.z - ya.z, kl.x, l0, ok);
            deg += (!ok && o != a) ? 1u : 0u;
            okl[s].x = c;
        }
        const int nf = (int)h->n_foreign;
        const uint8_t *fl = bl + h->off_fl;
        const int8_t *fg = GROUPS && h->off_fg ? reinterpret_cast<const int8_t *>(bl + h->off_fg) : nullptr;
        for (int f = tid; f < nf; f += kPipeThreads) {
            const float2 kl = fkl[f];
            float l0 = kl.y;
            if constexpr (GROUPS) {
                if (fg) {
                    const int g = fg[f];
                    if (g >= 0) l0 = l0 * p.scale[g];
                }
            }
            const float4 ya = sX[fl[f]], yo = sX[fo[f]];
            bool ok;
            fkl[f].x = spring_coef(yo.x - ya.x, yo.y - ya.y, yo.z - ya.z, kl.x, l0, ok);   // counted by the owner tile
        }
        flush_degenerate(p.degenerate, deg);
    }
    cp_async_wait_all();
    __syncthreads();

    // ---- mass pass: the mass's incidences [own records..., references...],
    // alternate ones per lane of the pair, combined by one shuffle
    V3<float> s = {0.f, 0.f, 0.f};
    if (active && p.debug != 1) {
        const float4 y = sX[l];
        const uint16_t cnt = reinterpret_cast<const uint16_t *>(bl + h->off_cnt)[l];
        const int n_own = cnt & 0xff, n_ref = cnt >> 8;
        for (int q = role; q < n_own; q += 2) {
            const int slot = (q << 8) | l;
            const float c = okl[slot].x;
            const float4 yo = sX[oo[slot]];
            s.x = __fmaf_rn(c, yo.x - y.x, s.x);
            s.y = __fmaf_rn(c, yo.y - y.y, s.y);
            s.z = __fmaf_rn(c, yo.z - y.z, s.z);
        }
        const uint16_t *rf = reinterpret_cast<const uint16_t *>(bl + h->off_ref) + l;
        for (int q = role ^ (n_own & 1); q < n_ref; q += 2) {
            const uint32_t v = rf[q << 8];
            const bool foreign = (v & 0x8000u) != 0;
            const uint32_t f = v & 0x7fffu;
            const float c = foreign ? fkl[f].x : okl[v].x;
            const int o = foreign ? (int)fo[f] : (int)(v & 0xffu);
            const float4 yo = sX[o];
            s.x = __fmaf_rn(c, yo.x - y.x, s.x);
            s.y = __fmaf_rn(c, yo.y - y.y, s.y);
            s.z = __fmaf_rn(c, yo.z - y.z, s.z);
        }
    }
    // both lanes of the pair compute the same (commutative) sum
    s.x += __shfl_xor_sync(0xffffffffu, s.x, 1);
    s.y += __shfl_xor_sync(0xffffffffu, s.y, 1);
    s.z += __shfl_xor_sync(0xffffffffu, s.z, 1);
    if (lead) {
        const float4 x4 = ctx.own_x;
        const float4 hist = sHist[l];
        float4 v4 = need_prev ? make_float4(0.f, 0.f, 0.f, 0.f) : hist;
        if (need_prev && (p.n_planes > 0 || signbit(x4.w))) v4 = p.V[m];   // friction / fixed restore
        integrate_store<INTEG>(p, m, s, x4, ctx.own_p, v4, hist, need_prev);
    }
}

// ------------------------------------------------------------------ lean
// One thread per tile mass (256 threads): the owner pass accumulates the
// owner's own terms while it writes c (the spring-once scheme of
// once_kernel.cuh), foreign copies are evaluated thread-per-record, and the
// reference pass adds c * (y_owner - y_me).  Loops are kept rolled (trip
// counts ~13 per mass) so no unroll remainders are generated; only warp 0
// polls the TMA mbarriers, the other warps sleep in the CTA barrier.
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
    const uint32_t split_word = __ldg(t.tsplit + blockIdx.x);
    const int n = (int)(split_word >> 24) + 1;
    const bool active = l < n;
    const bool need_prev = INTEG == 1 && !p.bootstrap;
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem);
    unsigned char *bl = smem + 128;
    float4 *sX = reinterpret_cast<float4 *>(bl + t.blob_smem);
    float4 *sHist = sX + (kTile + t.max_halo);
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
    // own state: the history vector the integrator needs streams to shared
    // memory (cp.async); r (w = +-m) stays in registers for the epilogue
    if (active) cp_async16(sHist + l, need_prev ? p.Xprev + m : p.V + m);
    cp_async_commit();
    const float4 A = ldg4(p.P + blockIdx.x * kTile + (n - 1) / 2);
    float4 x4 = make_float4(0.f, 0.f, 0.f, 0.f);
    if (active) {
        x4 = ldg4(p.X + m);
        const float4 pp = ldg4(p.P + m);
        sX[l] = make_float4((pp.x - A.x) + x4.x, (pp.y - A.y) + x4.y, (pp.z - A.z) + x4.z, x4.w);
    }
    mbar_wait_warp0(bar, 0);                                // header + halo ids
    const TileHdr *h = reinterpret_cast<const TileHdr *>(bl);
    {
        const int *halo = reinterpret_cast<const int *>(bl + h->off_halo);
        const int nh = (int)h->n_halo;
#pragma unroll 1
        for (int i = l; i < nh; i += kTile) {
            const int gm = halo[i];
            const float4 r = ldg4(p.X + gm), pp = ldg4(p.P + gm);
            sX[kTile + i] = make_float4((pp.x - A.x) + r.x, (pp.y - A.y) + r.y, (pp.z - A.z) + r.z, 0.f);
        }
    }
    mbar_wait_warp0(bar + 1, 0);                            // records (+ halo states via the barrier)

    const uint16_t *oo = reinterpret_cast<const uint16_t *>(bl + h->off_oo);
    float2 *okl = reinterpret_cast<float2 *>(bl + h->off_okl);
    const uint16_t *fo = reinterpret_cast<const uint16_t *>(bl + h->off_fo);
    float2 *fkl = reinterpret_cast<float2 *>(bl + h->off_fkl);
    V3<float> s = {0.f, 0.f, 0.f};
    float4 y = make_float4(0.f, 0.f, 0.f, 0.f);
    int n_ref = 0;
    if (p.debug != 1) {
        unsigned deg = 0;
        if (active) {                                       // owner pass
            y = sX[l];
            const uint16_t cnt = reinterpret_cast<const uint16_t *>(bl + h->off_cnt)[l];
            const int n_own = cnt & 0xff;
            n_ref = cnt >> 8;
            const int8_t *og = GROUPS && h->off_og ? reinterpret_cast<const int8_t *>(bl + h->off_og) : nullptr;
#pragma unroll 1
            for (int q = 0; q < n_own; ++q) {
                const int slot = (q << 8) | l;
                const float2 kl = okl[slot];
                float l0 = kl.y;
                if constexpr (GROUPS) {
                    if (og) {
                        const int g = og[slot];
                        if (g >= 0) l0 = l0 * p.scale[g];
                    }
                }
                const float4 yo = sX[oo[slot]];
                const float dx = yo.x - y.x, dy = yo.y - y.y, dz = yo.z - y.z;
                bool ok;
                const float c = spring_coef(dx, dy, dz, kl.x, l0, ok);
                deg += ok ? 0u : 1u;
                s.x = __fmaf_rn(c, dx, s.x);
                s.y = __fmaf_rn(c, dy, s.y);
                s.z = __fmaf_rn(c, dz, s.z);
                okl[slot].x = c;
            }
        }
        {                                                   // foreign copies, thread per record
            const int nf = (int)h->n_foreign;
            const uint8_t *fl = bl + h->off_fl;
            const int8_t *fg = GROUPS && h->off_fg ? reinterpret_cast<const int8_t *>(bl + h->off_fg) : nullptr;
#pragma unroll 1
            for (int f = l; f < nf; f += kTile) {
                const float2 kl = fkl[f];
                float l0 = kl.y;
                if constexpr (GROUPS) {
                    if (fg) {
                        const int g = fg[f];
                        if (g >= 0) l0 = l0 * p.scale[g];
                    }
                }
                const float4 ya = sX[fl[f]], yo = sX[fo[f]];
                bool ok;
                fkl[f].x = spring_coef(yo.x - ya.x, yo.y - ya.y, yo.z - ya.z, kl.x, l0, ok);   // counted by the owner tile
            }
        }
        flush_degenerate(p.degenerate, deg);
    }
    cp_async_wait_all();
    __syncthreads();                                        // every c written
    if (!active) return;
    if (p.debug != 1) {                                     // reference pass
        const uint16_t *rf = reinterpret_cast<const uint16_t *>(bl + h->off_ref) + l;
#pragma unroll 1
        for (int q = 0; q < n_ref; ++q) {
            const uint32_t v = rf[q << 8];
            const bool foreign = (v & 0x8000u) != 0;
            const uint32_t f = v & 0x7fffu;
            const float c = foreign ? fkl[f].x : okl[v].x;
            const int o = foreign ? (int)fo[f] : (int)(v & 0xffu);
            const float4 yo = sX[o];
            s.x = __fmaf_rn(c, yo.x - y.x, s.x);
            s.y = __fmaf_rn(c, yo.y - y.y, s.y);
            s.z = __fmaf_rn(c, yo.z - y.z, s.z);
        }
    }
    const float4 hist = sHist[l];
    float4 v4 = need_prev ? make_float4(0.f, 0.f, 0.f, 0.f) : hist;
    if (need_prev && (p.n_planes > 0 || signbit(x4.w))) v4 = p.V[m];       // friction / fixed restore
    float4 p4 = make_float4(0.f, 0.f, 0.f, 0.f);
    if (p.n_planes > 0) p4 = p.P[m];                        // absolute position for contact
    integrate_store<INTEG>(p, m, s, x4, p4, v4, hist, need_prev);
}

}  // namespace ss
