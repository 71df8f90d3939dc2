// 512-thread tile kernels (fp32 production mode, Euler / Verlet).  DESIGN.md §3.4.
//
// Two threads per tile mass: threads 0..255 sum the references of mass
// l = tid, threads 256..511 the own records of mass l = tid-256 (whole warps
// per role, no divergence).  The two partial sums are combined in a fixed
// order (refs + own), so results are deterministic and identical across
// launch shapes and shardings.  Per-incidence arithmetic is
// spring_term<true>; the integrator epilogue is step_kernel's.
//
//  tile_step2_kernel : one tile per CTA (like step_kernel<.., TILE>), 16
//                      warps per CTA -> twice the resident warps per SM.
//  tile_pipe_kernel  : persistent, one CTA per SM; TMA heads triple-buffered,
//                      TMA records and cp.async states double-buffered, so
//                      tile i+1 streams in while tile i computes (opt-in:
//                      SS_PIPE=1).
#pragma once

#include "kernels.cuh"

namespace ss {

constexpr int kPipeThreads = 2 * kTile;

__device__ __forceinline__ void cp_async16(void *dst, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Partial spring sum of tile mass l for this thread's role (0 refs, 1 own).
// `bl` is the blob base the section offsets are relative to.
template <bool CANON, bool GROUPS>
__device__ __forceinline__ V3<float> split_sum(const Params<float> &p, const TileHdr *h, const unsigned char *bl,
                                               const float4 *sX, const float4 *sP, int l, int role,
                                               float4 x4, float4 p4) {
    V3<float> sum = {0.f, 0.f, 0.f};
    unsigned deg = 0;
    const V3<float> xm = {x4.x, x4.y, x4.z}, pm = {p4.x, p4.y, p4.z};
    const int W = (int)h->W, Wr = (int)h->Wr;
    const uint16_t cnt = reinterpret_cast<const uint16_t *>(bl + h->off_cnt)[l];
    const uint16_t *oo = reinterpret_cast<const uint16_t *>(bl + h->off_oo);
    const float2 *okl = reinterpret_cast<const float2 *>(bl + h->off_okl);
    const int8_t *og = h->off_og ? reinterpret_cast<const int8_t *>(bl + h->off_og) : nullptr;
    if (role == 0) {
        const int n_ref = cnt >> 8;
        const uint16_t *fo = reinterpret_cast<const uint16_t *>(bl + h->off_fo);
        const float2 *fkl = reinterpret_cast<const float2 *>(bl + h->off_fkl);
        const int8_t *fg = h->off_fg ? reinterpret_cast<const int8_t *>(bl + h->off_fg) : nullptr;
        const uint16_t *rf = reinterpret_cast<const uint16_t *>(bl + h->off_ref) + ell_slot(l, 0, Wr, h->slice_log2);
#pragma unroll 2
        for (int q = 0; q < n_ref; ++q) {
            const uint32_t v = rf[q << h->slice_log2];
            const bool foreign = (v & 0x8000u) != 0;
            const uint32_t ol = v & 0xffu;
            const uint32_t slot = ell_slot(ol, v >> 8, W, h->slice_log2);
            const uint32_t idx = foreign ? (v & 0x7fffu) : slot;
            const float2 kl = foreign ? fkl[idx] : okl[idx];
            int o;
            bool mine = false;
            if constexpr (CANON) {
                o = foreign ? (int)fo[idx] : (int)ol;
            } else {
                mine = !foreign && (int)ol == l;
                o = foreign ? (int)fo[idx] : (mine ? (int)oo[slot] : (int)ol);
            }
            float l0 = kl.y;
            if constexpr (GROUPS) {
                if (og) {
                    const int g = foreign ? fg[idx] : og[idx];
                    if (g >= 0) l0 = l0 * p.scale[g];
                }
            }
            spring_term<true>(sX[o], sP[o], xm, pm, kl.x, l0, sum, mine, deg);
        }
    } else {
        const int n_own = cnt & 0xff;
        const int base = ell_slot(l, 0, W, h->slice_log2);
#pragma unroll 2
        for (int q = 0; q < n_own; ++q) {
            const int slot = base + (q << h->slice_log2);
            const int o = oo[slot];
            const float2 kl = okl[slot];
            float l0 = kl.y;
            if constexpr (GROUPS) {
                if (og) {
                    const int g = og[slot];
                    if (g >= 0) l0 = l0 * p.scale[g];
                }
            }
            spring_term<true>(sX[o], sP[o], xm, pm, kl.x, l0, sum, true, deg);
        }
    }
    flush_degenerate(p.degenerate, deg);
    return sum;
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

// --------------------------------------------------- one tile per CTA, 512 threads

// Role-split partial spring sum of tile mass l from the staged tile-local
// positions y (stage_tile<true>): role 0 the references, role 1 the own records.
template <bool CANON, bool GROUPS>
__device__ __forceinline__ V3<float> split_sum_y(const Params<float> &p, const TileCtx<true> &c, int l,
                                                 int role) {
    V3<float> sum = {0.f, 0.f, 0.f};
    unsigned deg = 0;
    const TileHdr *h = c.h;
    const unsigned char *bl = c.blob;
    const float4 y = c.sX[l];
    const V3<float> ym = {y.x, y.y, y.z};
    const int W = (int)h->W, Wr = (int)h->Wr;
    const uint16_t cnt = reinterpret_cast<const uint16_t *>(bl + h->off_cnt)[l];
    const uint16_t *oo = reinterpret_cast<const uint16_t *>(bl + h->off_oo);
    const float2 *okl = reinterpret_cast<const float2 *>(bl + h->off_okl);
    const int8_t *og = h->off_og ? reinterpret_cast<const int8_t *>(bl + h->off_og) : nullptr;
    if (role == 0) {
        const int n_ref = cnt >> 8;
        const uint16_t *fo = reinterpret_cast<const uint16_t *>(bl + h->off_fo);
        const float2 *fkl = reinterpret_cast<const float2 *>(bl + h->off_fkl);
        const int8_t *fg = h->off_fg ? reinterpret_cast<const int8_t *>(bl + h->off_fg) : nullptr;
        const uint16_t *rf = reinterpret_cast<const uint16_t *>(bl + h->off_ref) + ell_slot(l, 0, Wr, h->slice_log2);
#pragma unroll 2
        for (int q = 0; q < n_ref; ++q) {
            const uint32_t v = rf[q << h->slice_log2];
            const bool foreign = (v & 0x8000u) != 0;
            const uint32_t ol = v & 0xffu;
            const uint32_t slot = ell_slot(ol, v >> 8, W, h->slice_log2);
            const uint32_t idx = foreign ? (v & 0x7fffu) : slot;
            const float2 kl = foreign ? fkl[idx] : okl[idx];
            int o;
            bool mine = false;
            if constexpr (CANON) {
                o = foreign ? (int)fo[idx] : (int)ol;
            } else {
                mine = !foreign && (int)ol == l;
                o = foreign ? (int)fo[idx] : (mine ? (int)oo[slot] : (int)ol);
            }
            float l0 = kl.y;
            if constexpr (GROUPS) {
                if (og) {
                    const int g = foreign ? fg[idx] : og[idx];
                    if (g >= 0) l0 = l0 * p.scale[g];
                }
            }
            spring_term_y(c.sX[o], ym, kl.x, l0, sum, mine, deg);
        }
    } else {
        const int n_own = cnt & 0xff;
        const int base = ell_slot(l, 0, W, h->slice_log2);
#pragma unroll 2
        for (int q = 0; q < n_own; ++q) {
            const int slot = base + (q << h->slice_log2);
            const float2 kl = okl[slot];
            float l0 = kl.y;
            if constexpr (GROUPS) {
                if (og) {
                    const int g = og[slot];
                    if (g >= 0) l0 = l0 * p.scale[g];
                }
            }
            spring_term_y(c.sX[oo[slot]], ym, kl.x, l0, sum, true, deg);
        }
    }
    flush_degenerate(p.degenerate, deg);
    return sum;
}

template <int INTEG, bool CANON, bool GROUPS>
__global__ void __launch_bounds__(kPipeThreads, 3) tile_step2_kernel(Params<float> p) {
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
    // the epilogue thread (role 0) prefetches V and x_prev before the staging
    float4 v4 = make_float4(0.f, 0.f, 0.f, 0.f), xp4 = v4;
    if (active && role == 0) {
        v4 = p.V[m];
        if (need_prev) xp4 = p.Xprev[m];
    }
    const TileCtx<true> ctx = stage_tile<true>(p, smem, m, active && role == 0);
    float4 *part = ctx.sX + (kTile + t.max_halo);
    V3<float> sum = {0.f, 0.f, 0.f};
    if (active) {
        if (p.debug != 1) sum = split_sum_y<CANON, GROUPS>(p, ctx, l, role);
        if (role == 1) part[l] = make_float4(sum.x, sum.y, sum.z, 0.f);
    }
    __syncthreads();
    if (active && role == 0) {
        const float4 pr = part[l];
        sum.x += pr.x;
        sum.y += pr.y;
        sum.z += pr.z;
        integrate_store<INTEG>(p, m, sum, ctx.own_x, ctx.own_p, v4, xp4, need_prev);
    }
}

// ------------------------------------------------------- persistent, pipelined

// Shared-memory carve-up (pointers derived arithmetically from the extern
// __shared__ base so the compiler emits LDS/STS):
// [barriers | 3 heads | 2 record buffers | 2 x state | partials]
struct PipeGeom {
    uint32_t head, rest, slots;
    __device__ __forceinline__ unsigned char *head_buf(unsigned char *smem, int k) const {
        return smem + 128 + k * head;
    }
    __device__ __forceinline__ unsigned char *rest_buf(unsigned char *smem, int k) const {
        return smem + 128 + 3 * head + k * rest;
    }
    __device__ __forceinline__ float4 *state(unsigned char *smem, int k) const {
        return reinterpret_cast<float4 *>(smem + 128 + 3 * head + 2 * rest) + k * (2 * slots + 2 * kTile);
    }
    __device__ __forceinline__ float4 *part(unsigned char *smem) const {
        return reinterpret_cast<float4 *>(smem + 128 + 3 * head + 2 * rest) + 2 * (2 * slots + 2 * kTile);
    }
};

__device__ __forceinline__ uint32_t tile_split(const Topology<float> &t, int tile) {
    return t.tsplit[tile] & 0xffffffu;
}

__device__ __forceinline__ void pipe_issue_head(const Topology<float> &t, int tile, unsigned char *dst,
                                                uint64_t *bar) {
    bulk_copy(dst, t.blob + t.toff[tile], tile_split(t, tile), bar);
}
__device__ __forceinline__ void pipe_issue_rest(const Topology<float> &t, int tile, unsigned char *dst,
                                                uint64_t *bar) {
    const unsigned long long g0 = t.toff[tile];
    const uint32_t split = tile_split(t, tile);
    bulk_copy(dst, t.blob + g0 + split, (uint32_t)(t.toff[tile + 1] - g0) - split, bar);
}

// cp.async gather of tile `tile`'s own (X, P, V, Xprev) and halo (X, P) states.
template <int INTEG>
__device__ __forceinline__ void pipe_gather_state(const Params<float> &p, int tile, const unsigned char *head,
                                                  float4 *sX, float4 *sP, float4 *sV, float4 *sXp,
                                                  bool need_prev) {
    const TileHdr *h = reinterpret_cast<const TileHdr *>(head);
    const int n = (int)h->n, nh = (int)h->n_halo;
    const int tid = threadIdx.x;
    const int l = tid & (kTile - 1);
    if (l < n) {
        const int m = tile * kTile + l;
        if (tid < kTile) {
            cp_async16(sX + l, p.X + m);
            cp_async16(sV + l, p.V + m);
        } else {
            cp_async16(sP + l, p.P + m);
            if (INTEG == 1 && need_prev) cp_async16(sXp + l, p.Xprev + m);
        }
    }
    const int *halo = reinterpret_cast<const int *>(head + h->off_halo);
    for (int i = tid; i < nh; i += kPipeThreads) {
        const int g = halo[i];
        cp_async16(sX + kTile + i, p.X + g);
        cp_async16(sP + kTile + i, p.P + g);
    }
    cp_async_commit();
}

template <int INTEG, bool CANON, bool GROUPS>
__global__ void __launch_bounds__(kPipeThreads, 1) tile_pipe_kernel(Params<float> p) {
    extern __shared__ __align__(128) unsigned char smem[];
    if (*p.div_step < p.step) return;                       // grid-uniform
    const Topology<float> &t = p.topo;
    const int tid = threadIdx.x;
    const int role = tid >> 8;
    const int l = tid & (kTile - 1);
    uint64_t *hbar = reinterpret_cast<uint64_t *>(smem);    // 3 head barriers
    uint64_t *rbar = hbar + 3;                              // 2 record barriers
    const int stride = (int)gridDim.x;
    const int n_mine = (t.n_tiles - (int)blockIdx.x + stride - 1) / stride;
    if (n_mine <= 0) return;
    const PipeGeom G{t.head_smem, t.rest_smem, kTile + t.max_halo};
    float4 *part = G.part(smem);
    const bool need_prev = INTEG == 1 && !p.bootstrap;

    if (tid == 0) {
        for (int b = 0; b < 5; ++b)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(hbar + b)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tid == 0) {
        for (int k = 0; k < 2 && k < n_mine; ++k) {
            const int tile = blockIdx.x + k * stride;
            pipe_issue_head(t, tile, G.head_buf(smem, k), hbar + k);
            pipe_issue_rest(t, tile, G.rest_buf(smem, k), rbar + k);
        }
    }
    mbar_wait(hbar, 0);
    {
        float4 *st0 = G.state(smem, 0);
        pipe_gather_state<INTEG>(p, blockIdx.x, G.head_buf(smem, 0), st0, st0 + G.slots, st0 + 2 * G.slots,
                                 st0 + 2 * G.slots + kTile, need_prev);
    }
    cp_async_wait_all();
    __syncthreads();

    for (int i = 0; i < n_mine; ++i) {
        const int b2 = i & 1, b3 = i % 3;
        const int tile = blockIdx.x + i * stride;
        if (tid == 0 && i + 2 < n_mine)                     // head of tile i+2, two iterations ahead
            pipe_issue_head(t, tile + 2 * stride, G.head_buf(smem, (i + 2) % 3), hbar + (i + 2) % 3);
        if (i + 1 < n_mine) {                               // state of tile i+1 (its head landed)
            const int n3 = (i + 1) % 3, n2 = (i + 1) & 1;
            mbar_wait(hbar + n3, (uint32_t)((i + 1) / 3) & 1u);
            float4 *stn = G.state(smem, n2);
            pipe_gather_state<INTEG>(p, tile + stride, G.head_buf(smem, n3), stn, stn + G.slots,
                                     stn + 2 * G.slots, stn + 2 * G.slots + kTile, need_prev);
        }
        mbar_wait(rbar + b2, (uint32_t)(i >> 1) & 1u);      // records of tile i
        const TileHdr *h = reinterpret_cast<const TileHdr *>(G.head_buf(smem, b3));
        const unsigned char *bl = G.rest_buf(smem, b2) - tile_split(t, tile);   // offsets are blob-relative
        const float4 *sX = G.state(smem, b2), *sP = sX + G.slots;
        const float4 *sV = sX + 2 * G.slots, *sXp = sX + 2 * G.slots + kTile;
        const int n = (int)h->n;
        V3<float> sum = {0.f, 0.f, 0.f};
        float4 x4 = make_float4(0.f, 0.f, 0.f, 0.f), p4 = x4;
        if (l < n) {
            x4 = sX[l];
            p4 = sP[l];
            sum = split_sum<CANON, GROUPS>(p, h, bl, sX, sP, l, role, x4, p4);
            if (role == 1) part[l] = make_float4(sum.x, sum.y, sum.z, 0.f);
        }
        __syncthreads();
        if (role == 0 && l < n) {
            const float4 pr = part[l];
            sum.x += pr.x;
            sum.y += pr.y;
            sum.z += pr.z;
            integrate_store<INTEG>(p, tile * kTile + l, sum, x4, p4, sV[l], sXp[l], need_prev);
        }
        cp_async_wait_all();                                // tile i+1's state landed
        __syncthreads();                                    // stage i free
        if (tid == 0 && i + 2 < n_mine)
            pipe_issue_rest(t, tile + 2 * stride, G.rest_buf(smem, b2), rbar + b2);
    }
}

}  // namespace ss
