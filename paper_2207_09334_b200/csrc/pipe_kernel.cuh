// Persistent, software-pipelined tile kernel (fp32 production mode, Euler /
// Verlet).  DESIGN.md §3.4.
//
// One 512-thread CTA per SM walks its tiles t = blockIdx.x + i*gridDim.x.
// Each tile blob is fetched by the TMA engine in two pieces: the small head
// (header + halo id list, triple-buffered, issued two tiles ahead) and the
// records (double-buffered, issued one tile ahead).  While tile i is being
// computed, tile i+1's records stream in and cp.async gathers tile i+1's own
// and halo states (its head landed an iteration earlier), so DRAM streaming,
// L2 gathers and arithmetic overlap instead of alternating.
//
// Threads 0..255 sum the references of mass l = tid, threads 256..511 the own
// records of mass l = tid-256 (whole warps per role, no divergence); the two
// partial sums are combined in a fixed order (refs + own): deterministic.
// Per-incidence arithmetic is spring_term<true>; the integrator epilogue uses
// the same expressions as step_kernel.
#pragma once

#include "kernels.cuh"

namespace ss {

constexpr int kPipeThreads = 2 * kTile;

__device__ __forceinline__ void cp_async16(void *dst, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Shared-memory carve-up (all pointers derived arithmetically from the
// extern __shared__ base, so the compiler keeps them in the shared window
// and emits LDS/STS): [barriers | 3 heads | 2 record buffers | 2 x state | partials]
struct PipeGeom {
    uint32_t head, rest, slots;       // bytes per head / records buffer, state slots
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

// thread 0: TMA of tile `tile`'s head (header + halo ids) / records
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
    const int role = tid >> 8;                              // 0 refs + epilogue, 1 own records
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
        // ---- forces from shared memory
        const unsigned char *head = G.head_buf(smem, b3);
        const TileHdr *h = reinterpret_cast<const TileHdr *>(head);
        const unsigned char *bl = G.rest_buf(smem, b2) - tile_split(t, tile);   // offsets are blob-relative
        const float4 *sX = G.state(smem, b2), *sP = sX + G.slots;
        const float4 *sV = sX + 2 * G.slots, *sXp = sX + 2 * G.slots + kTile;
        const int n = (int)h->n;
        const int W = (int)h->W, Wr = (int)h->Wr;
        V3<float> sum = {0.f, 0.f, 0.f};
        unsigned deg = 0;
        float4 x4 = make_float4(0.f, 0.f, 0.f, 0.f), p4 = x4;
        if (l < n) {
            x4 = sX[l];
            p4 = sP[l];
            const V3<float> xm = {x4.x, x4.y, x4.z}, pm = {p4.x, p4.y, p4.z};
            const uint16_t cnt = reinterpret_cast<const uint16_t *>(bl + h->off_cnt)[l];
            const uint16_t *oo = reinterpret_cast<const uint16_t *>(bl + h->off_oo);
            const float2 *okl = reinterpret_cast<const float2 *>(bl + h->off_okl);
            const int8_t *og = h->off_og ? reinterpret_cast<const int8_t *>(bl + h->off_og) : nullptr;
            if (role == 0) {
                const int n_ref = cnt >> 8;
                const uint16_t *fo = reinterpret_cast<const uint16_t *>(bl + h->off_fo);
                const float2 *fkl = reinterpret_cast<const float2 *>(bl + h->off_fkl);
                const int8_t *fg = h->off_fg ? reinterpret_cast<const int8_t *>(bl + h->off_fg) : nullptr;
                const uint16_t *rf =
                    reinterpret_cast<const uint16_t *>(bl + h->off_ref) + (l >> 5) * Wr * 32 + (l & 31);
#pragma unroll 2
                for (int q = 0; q < n_ref; ++q) {
                    const uint32_t v = rf[q * 32];
                    const bool foreign = (v & 0x8000u) != 0;
                    const uint32_t ol = v & 0xffu;
                    const uint32_t slot = ((ol >> 5) * W + (v >> 8)) * 32 + (ol & 31u);
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
                const int base = (l >> 5) * W * 32 + (l & 31);
#pragma unroll 2
                for (int q = 0; q < n_own; ++q) {
                    const int slot = base + q * 32;
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
                part[l] = make_float4(sum.x, sum.y, sum.z, 0.f);
            }
        }
        flush_degenerate(p.degenerate, deg);
        __syncthreads();                                    // own-record partials visible
        // ---- epilogue (role 0): combine, external forces, integrate
        if (role == 0 && l < n) {
            const float4 pr = part[l];
            sum.x += pr.x;
            sum.y += pr.y;
            sum.z += pr.z;
            const int m = tile * kTile + l;
            const float mass = fabsf(x4.w);
            const bool fixed = signbit(x4.w);
            const float4 v4 = sV[l];
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
                    const float4 xp4 = sXp[l];
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
        cp_async_wait_all();                                // tile i+1's state landed
        __syncthreads();                                    // stage i free
        if (tid == 0 && i + 2 < n_mine)                     // records of tile i+2 into the freed buffer
            pipe_issue_rest(t, tile + 2 * stride, G.rest_buf(smem, b2), rbar + b2);
    }
}

}  // namespace ss
