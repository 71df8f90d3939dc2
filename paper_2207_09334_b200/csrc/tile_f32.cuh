// fp32 production-mode tile kernels (Euler / Verlet).  DESIGN.md §4.
//
// tile_lean_kernel: one tile (256 masses) per CTA of 256 threads, on the
// compact fp32 tile format (tiles.h).  The tile blob is TMA-bulk-copied into
// shared memory while every thread loads its own state; the displacement
// r = x - X0 of the tile's own and halo masses is staged once; then each
// thread walks its mass's incidence list (partner slot, dictionary index)
// and sums c*d with
//
//   d = D + (r_partner - r_me)         D = fp32 rest vector (dictionary)
//   c = k - (k l0) / |d|               rsqrt + one Newton step
//
// evaluating each spring from both endpoints (exactly opposite d, the same
// c: Newton's third law holds bitwise) -- no barrier after staging, nothing
// written to shared memory, 2 B per incidence streamed.  The fused epilogue
// applies external forces, Verlet / Euler, restore fixed and the finiteness
// check (integrate_store).  The summation order is fixed by the layout, so
// results are deterministic.
//
// Precision: r differences between neighbours are small, so the strain
// resolution is that of |r|, not of the absolute coordinates or of the
// tile extent; c = fma(-(k l0), 1/L, k) has the rounding sensitivity of
// k (L - l0)/L (both limited by the fp32 ulp of L).
#pragma once

#include "kernels.cuh"

namespace ss {

// --------------------------------------------------------------- primitives

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
// RK4 stage STAGE (1-4) of device mass m at the trial state (x4, vs4):
// kernels.cuh rk4_kernel's stage update (engine.py:330-354), on the lean
// kernel's spring sum.  X0/V0 step start, SV/SA running sums.
template <int STAGE>
__device__ __forceinline__ void rk4_store(const Params<float> &p, int m, V3<float> sum, const float4 &x4,
                                          const float4 &p4, const float4 &vs4, int tile) {
    const float4 x04 = p.X0[m];
    const float mass = fabsf(x04.w);
    const bool fixed = signbit(x04.w);
    const V3<float> xa = {p4.x + x4.x, p4.y + x4.y, p4.z + x4.z};
    const V3<float> f = add_external<true>(p, m, sum, xa, vs4, mass);
    const float a[3] = {f.x / mass, f.y / mass, f.z / mass};
    const float4 v04 = p.V0[m];
    const float x0[3] = {x04.x, x04.y, x04.z};
    const float v0[3] = {v04.x, v04.y, v04.z};
    const float vs[3] = {vs4.x, vs4.y, vs4.z};
    float xn[3], vn[3], sv[3], sa[3];
    if constexpr (STAGE == 1) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            xn[c] = x0[c] + p.half_dt * v0[c];
            vn[c] = v0[c] + p.half_dt * a[c];
            sa[c] = a[c];
        }
    } else if constexpr (STAGE == 2 || STAGE == 3) {
        const float4 sv4 = p.SV[m], sa4 = p.SA[m];
        const float h = (STAGE == 2) ? p.half_dt : p.dt;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            xn[c] = x0[c] + h * vs[c];
            vn[c] = v0[c] + h * a[c];
            const float svp = (STAGE == 2) ? v0[c] : (&sv4.x)[c];
            sv[c] = svp + 2.0f * vs[c];
            sa[c] = (&sa4.x)[c] + 2.0f * a[c];
        }
    } else {
        const float4 sv4 = p.SV[m], sa4 = p.SA[m];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const float svf = (&sv4.x)[c] + vs[c];
            const float saf = (&sa4.x)[c] + a[c];
            xn[c] = x0[c] + p.dt6 * svf;
            vn[c] = v0[c] + p.dt6 * saf;
            if (p.damped) vn[c] = vn[c] * p.one_minus_d;
        }
    }
    if (fixed) {
#pragma unroll
        for (int c = 0; c < 3; ++c) { xn[c] = x0[c]; vn[c] = v0[c]; }
    }
    const float4 xo = make_float4(xn[0], xn[1], xn[2], x04.w);
    if (!xchg_store(p, m, xo, tile)) return;                // a ghost: its neighbour writes this stage's trial x
    p.Xout[m] = xo;
    p.Vout[m] = make_float4(vn[0], vn[1], vn[2], 0.f);
    if constexpr (STAGE == 1) {
        p.SA[m] = make_float4(sa[0], sa[1], sa[2], 0.f);
    } else if constexpr (STAGE < 4) {
        p.SV[m] = make_float4(sv[0], sv[1], sv[2], 0.f);
        p.SA[m] = make_float4(sa[0], sa[1], sa[2], 0.f);
    } else {
        if (!(finite3<true>(xn[0], xn[1], xn[2]) && finite3<true>(vn[0], vn[1], vn[2])))
            flag_divergence<true>(p, m);
    }
}

// INTEG: 0 Euler, 1 Verlet, 2-5 RK4 stages 1-4 (rk4_store).
template <int INTEG>
__device__ __forceinline__ void integrate_store(const Params<float> &p, int m, V3<float> sum, float4 x4,
                                                float4 p4, float4 v4, float4 xp4, bool need_prev,
                                                int tile = blockIdx.x) {
    if constexpr (INTEG >= 2) {
        rk4_store<INTEG - 1>(p, m, sum, x4, p4, v4, tile);
        return;
    }
    const float mass = fabsf(x4.w);
    const bool fixed = signbit(x4.w);
    const V3<float> xa = {p4.x + x4.x, p4.y + x4.y, p4.z + x4.z};
    const V3<float> f = add_external<true>(p, m, sum, xa, v4, mass);
    float xn[3], vn[3], un[3] = {0.f, 0.f, 0.f};
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
    } else {                                                // increment-form Verlet (kernels.cuh verlet_u)
        verlet_u(p, x, v, fc, p.dt2_over / mass, xp4, xn, vn, un);
    }
    if (fixed) {
#pragma unroll
        for (int c = 0; c < 3; ++c) { xn[c] = x[c]; vn[c] = v[c]; un[c] = 0.f; }
    }
    const float4 xo = make_float4(xn[0], xn[1], xn[2], x4.w);
    if (!xchg_store(p, m, xo, tile)) return;                // a ghost: its neighbour writes it
    p.Xout[m] = xo;
    p.Vout[m] = make_float4(vn[0], vn[1], vn[2], 0.f);
    if constexpr (INTEG == 1) p.U[m] = make_float4(un[0], un[1], un[2], 0.f);
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

// -------------------------------------------------- compact format pass

// Spring sum of tile mass l over its incidence list (own springs first),
// from the staged displacements sR.  Returns the number of degenerate own
// springs.
// LANES > 1: this thread takes incidences lane, lane + LANES, ... and the
// caller combines the lanes' sums; dmin_out gets the smallest d^2 seen (the
// degenerate recount, by lane 0, covers all own springs).
// (k, k*l0, Dx, Dy), Dz and group of incidence q (entry e): the tile's
// dictionary, or (REC 1, general graphs) this mass's column of the inline
// (k, k*l0) records in global memory (tiles.h), streamed, with
// D = fp32(X0_partner - X0_me) from the fp64 rest positions staged in shared
// memory (sX0: x, y, z planes of ns slots) -- the dictionary's value.
// REC 0: the dictionary (rest vector stored); 1: inline records (general
// graphs); 2: the dictionary of (k, k*l0, group) with the rest vector from
// the staged X0 (scenes whose positions are off a lattice -- jittered robot
// populations -- where a D-keyed dictionary overflows but the materials do not)
template <int REC>
struct F32Rec {
    const float4 *dict;          // dictionary (2 float4 per entry)
    const float2 *kk;            // inline (k, k*l0) + column
    const int8_t *g;             // inline groups + column (null: none)
    const double *sX0;           // inline: staged X0 planes
    int ns;                      //   plane stride
    double mx, my, mz;           //   X0 of this mass
    __device__ __forceinline__ float2 load(int q) const { return __ldcs(kk + (q << 8)); }
    __device__ __forceinline__ void get(uint32_t e, int q, float4 &kd, float &dz_, int &grp) const {
        get(e, q, REC == 1 ? load(q) : make_float2(0.f, 0.f), kd, dz_, grp);
    }
    // k2: the inline (k, k*l0) of incidence q, already loaded
    __device__ __forceinline__ void get(uint32_t e, int q, float2 k2, float4 &kd, float &dz_, int &grp) const {
        if constexpr (REC == 1) {
            const uint32_t sl = e & 0x3ffu;
            kd = make_float4(k2.x, k2.y, __double2float_rn(__dsub_rn(sX0[sl], mx)),
                             __double2float_rn(__dsub_rn(sX0[ns + sl], my)));
            dz_ = __double2float_rn(__dsub_rn(sX0[2 * ns + sl], mz));
            grp = g ? g[q << 8] : -1;
        } else if constexpr (REC == 2) {
            const float4 *ent = dict + 2 * (e >> 10);
            const float4 k4 = ent[0];
            const uint32_t sl = e & 0x3ffu;
            kd = make_float4(k4.x, k4.y, __double2float_rn(__dsub_rn(sX0[sl], mx)),
                             __double2float_rn(__dsub_rn(sX0[ns + sl], my)));
            dz_ = __double2float_rn(__dsub_rn(sX0[2 * ns + sl], mz));
            grp = __float_as_int(ent[1].y);
        } else {
            const float4 *ent = dict + 2 * (e >> 10);
            kd = ent[0];
            const float4 ez = ent[1];                       // (Dz, group bits, -, -)
            dz_ = ez.x;
            grp = __float_as_int(ez.y);
        }
    }
};

template <bool GROUPS, int LANES = 1, int REC = 0>
__device__ __forceinline__ unsigned incidence_sum(const Params<float> &p, const TileView &v, int l, const float4 &rm,
                                                  int n_own, int n_inc, V3<float> &s, int lane = 0,
                                                  float *dmin_out = nullptr, int tile = 0) {
    const uint16_t *inc = reinterpret_cast<const uint16_t *>(v.bl + v.h->off_oo) + l;
    F32Rec<REC> rec;
    if constexpr (REC == 1) {
        const unsigned long long b0 = p.topo.kl_off[tile] + (unsigned long long)l;
        rec.kk = p.topo.kd_inline + b0;
        rec.g = p.topo.g_inline ? p.topo.g_inline + b0 : nullptr;
    } else {
        rec.dict = reinterpret_cast<const float4 *>(v.bl + v.h->off_okl);
    }
    if constexpr (REC != 0) {                               // the staged X0 planes
        rec.ns = kTile + (int)p.topo.max_halo;
        rec.sX0 = reinterpret_cast<const double *>(v.sY + rec.ns);
        rec.mx = rec.sX0[l];
        rec.my = rec.sX0[rec.ns + l];
        rec.mz = rec.sX0[2 * rec.ns + l];
    }
    float dmin = INFINITY;
    auto body = [&](int q, float2 k2) {
        const uint32_t e = inc[q << 8];
        float4 kd;                                          // (k, k*l0, Dx, Dy)
        float dzr;
        int g;
        rec.get(e, q, k2, kd, dzr, g);
        float kl0 = kd.y;
        if constexpr (GROUPS) {
            if (g >= 0) kl0 = kl0 * p.scale[g];
        }
        const float4 ro = v.sY[e & 0x3ffu];
        const float dx = kd.z + (ro.x - rm.x), dy = kd.w + (ro.y - rm.y), dz_ = dzr + (ro.z - rm.z);
        float d2;
        const float c = spring_c(dx, dy, dz_, kd.x, kl0, d2);
        dmin = fminf(dmin, d2);                             // a degenerate reference is also degenerate at its owner
        acc3(s, c, dx, dy, dz_);
    };
    if constexpr (REC == 1) {
        // records streamed from HBM, software pipelined: the next group's
        // loads are in flight while this group computes
        constexpr int P = 4;
        float2 kc[P];
#pragma unroll
        for (int j = 0; j < P; ++j) kc[j] = j < n_inc ? rec.load(j) : make_float2(0.f, 0.f);
#pragma unroll 1
        for (int q = 0; q < n_inc; q += P) {
            float2 kn[P];
#pragma unroll
            for (int j = 0; j < P; ++j) kn[j] = q + P + j < n_inc ? rec.load(q + P + j) : make_float2(0.f, 0.f);
#pragma unroll
            for (int j = 0; j < P; ++j)
                if (q + j < n_inc) body(q + j, kc[j]);
#pragma unroll
            for (int j = 0; j < P; ++j) kc[j] = kn[j];
        }
    } else {
        const float2 none = make_float2(0.f, 0.f);
        int q = lane;
#pragma unroll 1
        for (; q + 3 * LANES < n_inc; q += 4 * LANES) {
            body(q, none);
            body(q + LANES, none);
            body(q + 2 * LANES, none);
            body(q + 3 * LANES, none);
        }
#pragma unroll 1
        for (; q < n_inc; q += LANES) body(q, none);
    }
    unsigned deg = 0;
    if (dmin_out) {
        *dmin_out = dmin;
        return 0;
    }
    if (dmin < 1e-24f) {                                    // rare: count the degenerate own springs
        for (int r = 0; r < n_own; ++r) {
            const uint32_t e = inc[r << 8];
            float4 kd;
            float dzr;
            int g;
            rec.get(e, r, kd, dzr, g);
            const float4 ro = v.sY[e & 0x3ffu];
            const float dx = kd.z + (ro.x - rm.x), dy = kd.w + (ro.y - rm.y), dz_ = dzr + (ro.z - rm.z);
            const float d2 = __fmaf_rn(dz_, dz_, __fmaf_rn(dy, dy, __fmul_rn(dx, dx)));
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
                                              const float4 &hist, bool need_prev, int tile) {
    float4 v4 = need_prev ? make_float4(0.f, 0.f, 0.f, 0.f) : hist;
    if (need_prev && (p.n_planes > 0 || signbit(x4.w))) v4 = p.V[m];
    float4 p4 = make_float4(0.f, 0.f, 0.f, 0.f);
    if (p.n_planes > 0) p4 = p.P[m];
    integrate_store<INTEG>(p, m, s, x4, p4, v4, hist, need_prev, tile);
}

// The tile of this CTA: sharded slabs run their boundary tiles first
// (ORDERED, kernels.cuh xchg_*), so the neighbours' flags publish early.
template <bool ORDERED>
__device__ __forceinline__ int lean_tile(const Params<float> &p) {
    if constexpr (ORDERED) return __ldg(p.tile_order + blockIdx.x);
    else return (int)blockIdx.x;
}

// ------------------------------------------------------------------ lean

__device__ __forceinline__ void mbar_wait_warp0(uint64_t *bar, uint32_t phase) {
    if (threadIdx.x < 32) mbar_wait(bar, phase);
    __syncthreads();
}

// Launched with programmatic dependent launch (engine.cu launch_tile_f32):
// every CTA lets the next substep's grid launch as soon as it has started,
// so the next grid's CTAs fill the SM slots freed during this grid's tail and
// stream their (step-independent) record blobs by TMA before they wait for
// this grid's positions (griddepcontrol.wait).
// LANES = 2 (scenes with few tiles): 512 threads per tile; thread t works on
// mass l = t mod 256 with lane t / 256 taking every other incidence, and the
// lanes' sums meet in shared memory in a fixed order -- twice the warps for
// the same tiles, for scenes too small to fill the GPU.
template <int INTEG, bool GROUPS, int LANES = 1, bool ORDERED = false, int REC = 0>
__device__ __forceinline__ void lean_body(const Params<float> &p, unsigned char *smem) {
    static_assert(!(REC != 0 && LANES > 1), "records with the staged X0 step with one lane per mass");
    const Topology<float> &t = p.topo;
    const int tid = threadIdx.x;
    const int l = tid % kTile, lane = tid / kTile;
    const int tile = lean_tile<ORDERED>(p);
    const int m = tile * kTile + l;
    const int n = (int)(__ldg(t.tsplit + tile) >> 24) + 1;
    const bool active = l < n;
    const bool need_prev = INTEG == 1 && !p.bootstrap;
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem);
    unsigned char *bl = smem + 128;
    float4 *sR = reinterpret_cast<float4 *>(bl + t.blob_smem);
    if (tid == 0) {
        if (p.reinit) {                                     // persistent kernel: re-arm completed barriers
            asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)));
            asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(bar + 1)));
        }
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar + 1)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tid == 0) {
        const int tb = p.debug == 2 ? 0 : tile;             // debug 2: every CTA stages tile 0 (L2-resident)
        const unsigned long long g0 = t.toff[tb];
        const uint32_t bytes = (uint32_t)(t.toff[tb + 1] - g0);
        const uint32_t split = t.tsplit[tb] & 0xffffffu;
        bulk_copy(bl, t.blob + g0, split, bar);
        bulk_copy(bl + split, t.blob + g0 + split, bytes - split, bar + 1);
    }
    // REC != 0: the fp64 rest positions X0 of own and halo slots, as x, y, z
    // planes behind the staged displacements (rest vectors formed per
    // incidence); step-independent, so staged before the grid dependency
    const int ns = kTile + (int)t.max_halo;
    double *sX0 = reinterpret_cast<double *>(sR + ns);
    if constexpr (REC != 0) {
        if (active) {
            sX0[l] = __ldg(t.x0 + 3 * (long long)m);
            sX0[ns + l] = __ldg(t.x0 + 3 * (long long)m + 1);
            sX0[2 * ns + l] = __ldg(t.x0 + 3 * (long long)m + 2);
        }
        mbar_wait_warp0(bar, 0);                            // halo ids
        const int *halo = reinterpret_cast<const int *>(bl + reinterpret_cast<const TileHdr *>(bl)->off_halo);
        const int nh = (int)reinterpret_cast<const TileHdr *>(bl)->n_halo;
#pragma unroll 1
        for (int i = tid; i < nh; i += kTile) {
            const int gm = halo[i];
            if (gm >= 0) {
                sX0[kTile + i] = __ldg(t.x0 + 3 * (long long)gm);
                sX0[ns + kTile + i] = __ldg(t.x0 + 3 * (long long)gm + 1);
                sX0[2 * ns + kTile + i] = __ldg(t.x0 + 3 * (long long)gm + 2);
            }
        }
    }
    // everything below reads the previous substep's state
    asm volatile("griddepcontrol.wait;" ::: "memory");
    xchg_wait(p, tile);
    if (*p.div_step < step_of(p)) {                             // grid-uniform (an earlier step diverged):
        if (tid == 0) {                                     // retire only once the bulk copies have landed
            mbar_wait(bar, 0);
            mbar_wait(bar + 1, 0);
        }
        return;
    }
    float4 x4 = make_float4(0.f, 0.f, 0.f, 0.f), hist = x4;
    if (active && lane == 0) {
        x4 = ldg4(p.X + m);                                 // r = x - X0, w = +-m
        hist = need_prev ? ldg4(p.Xprev + m) : ldg4(p.V + m);
        sR[l] = x4;
    }
    mbar_wait_warp0(bar, 0);                                // header + halo ids
    const TileView v = tile_view(bl, sR);
    {
        const int *halo = reinterpret_cast<const int *>(bl + v.h->off_halo);
        const int nh = (int)v.h->n_halo;
        // up to 3 x 256 halo slots (compact format): all loads in flight
        // before the first store, one memory latency instead of three
        constexpr int J = (3 + LANES - 1) / LANES;
        float4 hv[J];
#pragma unroll
        for (int j = 0; j < J; ++j) {
            const int i = tid + j * kTile * LANES;
            const int gm = i < nh ? halo[i] : -1;           // -1: beyond the list or a hole
            hv[j] = gm >= 0 ? ldg4(p.X + gm) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int j = 0; j < J; ++j) {
            const int i = tid + j * kTile * LANES;
            if (i < nh) sR[kTile + i] = hv[j];
        }
#pragma unroll 1
        for (int i = tid + J * kTile * LANES; i < nh; i += kTile * LANES) {   // (not reached by compact tiles)
            const int gm = halo[i];
            if (gm >= 0) sR[kTile + i] = ldg4(p.X + gm);
        }
    }
    mbar_wait_warp0(bar + 1, 0);                            // records (+ the staged states)
    V3<float> s = {0.f, 0.f, 0.f};
    if constexpr (LANES == 1) {
        if (!active) return;
        if (p.debug != 1) {
            const uint16_t cnt = reinterpret_cast<const uint16_t *>(bl + v.h->off_cnt)[l];
            flush_degenerate(p.degenerate,
                             incidence_sum<GROUPS, 1, REC>(p, v, l, x4, cnt & 0xff, cnt >> 8, s, 0, nullptr, tile));
        }
    } else {
        // lane 1's partial sums (and its smallest d^2) meet lane 0's in shared
        // memory behind the halo, in a fixed order
        float4 *part = sR + kTile + t.max_halo;
        float dmin = INFINITY;
        uint16_t cnt = 0;
        if (active) {
            if (lane) x4 = sR[l];
            cnt = reinterpret_cast<const uint16_t *>(bl + v.h->off_cnt)[l];
            if (p.debug != 1) incidence_sum<GROUPS, LANES>(p, v, l, x4, cnt & 0xff, cnt >> 8, s, lane, &dmin);
            if (lane) part[l] = make_float4(s.x, s.y, s.z, dmin);
        }
        __syncthreads();
        if (!active || lane) return;
        const float4 o = part[l];
        s.x = s.x + o.x;
        s.y = s.y + o.y;
        s.z = s.z + o.z;
        if (fminf(dmin, o.w) < 1e-24f && p.debug != 1) {  // rare: recount the degenerate own springs
            V3<float> junk = {0.f, 0.f, 0.f};
            flush_degenerate(p.degenerate, incidence_sum<GROUPS>(p, v, l, x4, cnt & 0xff, cnt & 0xff, junk));
        }
    }
    tile_epilogue<INTEG>(p, m, s, x4, hist, need_prev, tile);
}

template <int INTEG, bool GROUPS, int MINB = 6, int LANES = 1, bool ORDERED = false, int REC = 0>
__global__ void __launch_bounds__(kTile * LANES, LANES == 1 ? MINB : 3) tile_lean_kernel(Params<float> p) {
    extern __shared__ __align__(128) unsigned char smem[];
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    lean_body<INTEG, GROUPS, LANES, ORDERED, REC>(p, smem);
    xchg_finish(p, lean_tile<ORDERED>(p));
}

// Persistent cooperative variant for small scenes (kernels.cuh persist_step_kernel).
template <int INTEG, bool GROUPS>
__global__ void __launch_bounds__(kTile) persist_lean_kernel(Params<float> p, PersistArgs<float> a) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ Params<float> q;                             // this step's parameters, one copy per CTA
    for (long long s = 0; s < a.count; ++s) {
        if (threadIdx.x == 0) q = persist_params(p, a, s);
        __syncthreads();
        lean_body<INTEG, GROUPS>(q, smem);
        grid_barrier();
        if (*p.div_step <= a.step0 + s + 1) return;         // this or an earlier step diverged
    }
}

}  // namespace ss
