// Spring-once tile kernel (fp32 production mode, Euler / Verlet).  DESIGN.md §4.
//
// The mass-centric gather of kernels.cuh evaluates every spring twice, once
// from each endpoint.  Here a spring whose two endpoints sit in the same tile
// is evaluated once, by its owner (the endpoint with the lower caller id):
//
//   phase 1  owner pass:   for each own record   c = k(L - l0)/L, s += c*d,
//                          and c is written back over the record's k in the
//                          tile's shared-memory copy of the blob;
//            foreign pass: references whose owner lies in another tile are
//                          evaluated from the tile's foreign record copies.
//   barrier
//   phase 2  in-tile refs: s += c * (y_owner - y_me)   (one LDS.32 + one LDS.128,
//                          no sqrt: the owner's c, the partner's exact -d).
//
// The partner's term is bitwise the negation of the owner's (d is exact
// in the staged tile-local frame), so momentum stays exact and the result
// equals what a per-endpoint recomputation would produce.  Two threads per
// tile mass (q = role, role + 2, ...) keep 16 warps per CTA; the two partial
// sums are combined in a fixed order, so results are deterministic.
//
// Requires an fp32 tile build: every mass canonical and a mass's foreign
// references listed before its in-tile ones (tiles.h, off_nf).
#pragma once

#include "pipe_kernel.cuh"

namespace ss {

// c and d of one spring from staged tile-local positions (spring_term_y's
// arithmetic, split so the caller can keep c).
__device__ __forceinline__ float spring_c(const float4 &yo, const V3<float> &ym, float k, float l0, float &dx,
                                          float &dy, float &dz, bool count_degenerate, unsigned &deg) {
    dx = yo.x - ym.x;
    dy = yo.y - ym.y;
    dz = yo.z - ym.z;
    const float d2 = __fmaf_rn(dz, dz, __fmaf_rn(dy, dy, __fmul_rn(dx, dx)));
    float inv = rsqrtf(d2);
    inv = __fmul_rn(inv, __fmaf_rn(__fmul_rn(-0.5f, d2), __fmul_rn(inv, inv), 1.5f));
    const float len = __fmul_rn(d2, inv);
    const bool ok = d2 >= 1e-24f;
    deg += (!ok && count_degenerate) ? 1u : 0u;
    return ok ? __fmul_rn(__fmul_rn(k, len - l0), inv) : 0.0f;
}

template <int INTEG, bool GROUPS, int MINB>
__global__ void __launch_bounds__(kPipeThreads, MINB) tile_once_kernel(Params<float> p) {
    extern __shared__ __align__(128) unsigned char smem[];
    if (*p.div_step < p.step) return;                       // grid-uniform
    const Topology<float> &t = p.topo;
    const int tid = threadIdx.x;
    const int role = tid >> 8;
    const int l = tid & (kTile - 1);
    const int m = blockIdx.x * kTile + l;
    const int n = (int)(__ldg(t.tsplit + blockIdx.x) >> 24) + 1;
    const bool active = l < n;
    const bool need_prev = INTEG == 1 && !p.bootstrap;
    // Verlet reads v only to bootstrap, for friction, or to restore a fixed mass
    const bool need_v = INTEG == 0 || !need_prev || p.n_planes > 0;
    float4 v4 = make_float4(0.f, 0.f, 0.f, 0.f), xp4 = v4;
    if (active && role == 0) {                              // epilogue streams first
        if (need_v) v4 = p.V[m];
        if (need_prev) xp4 = p.Xprev[m];
    }
    const TileCtx<true> ctx = stage_tile<true>(p, smem, m, active && role == 0);
    float4 *part = ctx.sX + (kTile + t.max_halo);
    const TileHdr *h = ctx.h;
    unsigned char *bl = const_cast<unsigned char *>(ctx.blob);
    const float4 *sX = ctx.sX;
    V3<float> s = {0.f, 0.f, 0.f};
    unsigned deg = 0;
    int n_ref = 0, n_for = 0;
    V3<float> ym = {0.f, 0.f, 0.f};
    const int Wr = (int)h->Wr;
    const uint16_t *rf = reinterpret_cast<const uint16_t *>(bl + h->off_ref) + ell_slot(l, 0, Wr, h->slice_log2);
    float2 *okl = reinterpret_cast<float2 *>(bl + h->off_okl);
    const int W = (int)h->W;
    if (active) {
        const float4 y = sX[l];
        ym = {y.x, y.y, y.z};
        const uint16_t cnt = reinterpret_cast<const uint16_t *>(bl + h->off_cnt)[l];
        const int n_own = cnt & 0xff;
        n_ref = cnt >> 8;
        n_for = reinterpret_cast<const uint8_t *>(bl + h->off_nf)[l];
        const uint16_t *oo = reinterpret_cast<const uint16_t *>(bl + h->off_oo);
        const int8_t *og = GROUPS && h->off_og ? reinterpret_cast<const int8_t *>(bl + h->off_og) : nullptr;
        const int base = ell_slot(l, 0, W, h->slice_log2);
#pragma unroll 2
        for (int q = role; q < n_own; q += 2) {            // owner pass
            const int slot = base + (q << h->slice_log2);
            const float2 kl = okl[slot];
            float l0 = kl.y;
            if constexpr (GROUPS) {
                if (og) {
                    const int g = og[slot];
                    if (g >= 0) l0 = l0 * p.scale[g];
                }
            }
            float dx, dy, dz;
            const float c = spring_c(sX[oo[slot]], ym, kl.x, l0, dx, dy, dz, true, deg);
            s.x = __fmaf_rn(c, dx, s.x);
            s.y = __fmaf_rn(c, dy, s.y);
            s.z = __fmaf_rn(c, dz, s.z);
            okl[slot].x = c;                                // k -> c for the in-tile partner
        }
        const uint16_t *fo = reinterpret_cast<const uint16_t *>(bl + h->off_fo);
        const float2 *fkl = reinterpret_cast<const float2 *>(bl + h->off_fkl);
        const int8_t *fg = GROUPS && h->off_fg ? reinterpret_cast<const int8_t *>(bl + h->off_fg) : nullptr;
#pragma unroll 2
        for (int q = role; q < n_for; q += 2) {            // foreign references
            const uint32_t idx = rf[q << h->slice_log2] & 0x7fffu;
            const float2 kl = fkl[idx];
            float l0 = kl.y;
            if constexpr (GROUPS) {
                if (fg) {
                    const int g = fg[idx];
                    if (g >= 0) l0 = l0 * p.scale[g];
                }
            }
            spring_term_y(sX[fo[idx]], ym, kl.x, l0, s, false, deg);
        }
    }
    __syncthreads();                                        // every c written
    if (active) {
#pragma unroll 2
        for (int q = n_for + role; q < n_ref; q += 2) {    // in-tile references
            const uint32_t v = rf[q << h->slice_log2];
            const uint32_t ol = v & 0xffu;
            const uint32_t slot = ell_slot(ol, v >> 8, W, h->slice_log2);
            const float c = okl[slot].x;
            const float4 yo = sX[ol];
            s.x = __fmaf_rn(c, yo.x - ym.x, s.x);
            s.y = __fmaf_rn(c, yo.y - ym.y, s.y);
            s.z = __fmaf_rn(c, yo.z - ym.z, s.z);
        }
        if (role == 1) part[l] = make_float4(s.x, s.y, s.z, 0.f);
    }
    flush_degenerate(p.degenerate, deg);
    __syncthreads();
    if (active && role == 0) {
        const float4 pr = part[l];
        s.x += pr.x;
        s.y += pr.y;
        s.z += pr.z;
        const float4 x4 = ctx.own_x;
        if (!need_v && signbit(x4.w)) v4 = p.V[m];          // fixed mass: restore its v
        integrate_store<INTEG>(p, m, s, x4, ctx.own_p, v4, xp4, need_prev);
    }
}

}  // namespace ss
