// On-device sampling for simulate / RunResult (engine.py:476-565) and the
// energy breakdown (engine.py:148-170, energy_breakdown):
//
//   EPE = 1/2 sum_s k_s (|x_j - x_i| - l0_eff_s)^2
//   GPE = sum_m m |g| (x_m . up - datum),  up = -g/|g|  (0 without gravity)
//   KE  = 1/2 sum_m m |v_m|^2
//
// evaluated at a sampled state (Verlet: x_prev paired with the lagged central
// difference v, like the reference's simulate) and summed in caller order by
// numpy's pairwise summation (below), so an fp64 engine's energies are
// bitwise the reference's.  Traced positions are gathered into a row
// buffer; rows stay on the device until the run segment ends.
#pragma once

#include <cuda_runtime.h>

#include "kernels.cuh"

namespace ss {

constexpr int kSampleThreads = 256;

struct SampleArgs {
    const void *X;               // positions at the sample (T4; fp32: displacement r)
    const void *Usub;            // fp32 Verlet x_prev samples: u subtracted from X (null: none)
    const void *V;               // velocities at the sample (T4)
    const float4 *P;             // fp32 base positions (null in fp64)
    const double *mass;          // fp64 masses per device slot (0: padding)
    const double *x0;            // fp32 TILE: fp64 rest positions (x = X0 + r); null: x = P + r
    int nd;                      // device mass slots
    const int *ssi, *ssj;        // springs in device ids
    const double *sk, *sl0;      // k, l0 (caller precision: fp64)
    const int *sgrp;             // actuation group per spring (-1 passive), may be null
    const double *scale;         // group scales at the sample time
    long long n_springs;
    double g_mag, up[3], datum;
    long long n_masses;          // caller masses
    const int *dev_of;           // caller mass id -> device slot
    const int *ids;              // traced masses (device ids)
    int n_ids;
    double *pos_row;             // n_ids x 3
    double *energy_row;          // 4
};

template <bool F32>
__device__ __forceinline__ void load_pos(const SampleArgs &a, int i, double &x, double &y, double &z, double &m) {
    if constexpr (F32) {
        float4 r = reinterpret_cast<const float4 *>(a.X)[i];
        if (a.Usub) {
            const float4 u = reinterpret_cast<const float4 *>(a.Usub)[i];
            x = (double)r.x - (double)u.x;                  // exact in fp64
            y = (double)r.y - (double)u.y;
            z = (double)r.z - (double)u.z;
            if (a.x0) {
                x += a.x0[3 * i + 0];
                y += a.x0[3 * i + 1];
                z += a.x0[3 * i + 2];
            } else {
                const float4 b = a.P[i];
                x += (double)b.x;
                y += (double)b.y;
                z += (double)b.z;
            }
            m = fabs((double)r.w);
            return;
        }
        if (a.x0) {
            x = a.x0[3 * i + 0] + (double)r.x;
            y = a.x0[3 * i + 1] + (double)r.y;
            z = a.x0[3 * i + 2] + (double)r.z;
        } else {
            const float4 b = a.P[i];
            x = (double)b.x + (double)r.x;
            y = (double)b.y + (double)r.y;
            z = (double)b.z + (double)r.z;
        }
        m = fabs((double)r.w);
    } else {
        const double4 r = reinterpret_cast<const double4 *>(a.X)[i];
        x = r.x;
        y = r.y;
        z = r.z;
        m = fabs(r.w);
    }
}

template <bool F32>
__device__ __forceinline__ void load_vel(const SampleArgs &a, int i, double &x, double &y, double &z) {
    if constexpr (F32) {
        const float4 v = reinterpret_cast<const float4 *>(a.V)[i];
        x = v.x;
        y = v.y;
        z = v.z;
    } else {
        const double4 v = reinterpret_cast<const double4 *>(a.V)[i];
        x = v.x;
        y = v.y;
        z = v.z;
    }
}

// ---------------------------------------------------------------------------
// numpy's pairwise summation, restated for the device.  np.sum over a
// contiguous float64 array of n elements (numpy's pairwise_sum, the add
// reduction's inner loop) is
//   0.0 + pw(a, n)
//   pw(a, n) = sequential sum from 0.0                                  n < 8
//            = r[j] = a[j], r[j] += a[i + j] (i = 8, 16, ... < n - n%8),
//              ((r0 + r1) + (r2 + r3)) + ((r4 + r5) + (r6 + r7)),
//              then the n%8 tail added in order                         n <= 128
//            = pw(a, n2) + pw(a + n2, n - n2),  n2 = n/2 - (n/2)%8      otherwise
// (checked bitwise against np.sum for n = 1..300 and up to 10^6 by
// tests/test_energy_pairwise.py).  The host builds the recursion once per n
// (PwPlan: leaves in order, internal nodes grouped by height); a leaf is
// summed by 8 lanes (lane j owns accumulator r[j]), the tree is combined
// level by level.  With the reference's per-element formulas
// (engine.py:148-170: norm = sqrt((d0^2 + d1^2) + d2^2); einsum's row dot
// (v0^2 + v2^2) + v1^2; (m |g|) (x.up - datum)) the energies are bitwise
// those of the reference's energy_breakdown at the same state.

struct PwPlanDev {
    const long long *leaf_off;   // leaf i covers [leaf_off[i], leaf_off[i] + leaf_len[i])
    const int *leaf_len;
    int n_leaves;
    const int4 *nodes;           // (left, right, out, -) value ids, grouped by height
    const int *level_start;      // n_levels + 1 offsets into nodes
    int n_levels;
    int root;                    // value id of the whole sum
};

// EPE term of caller spring s: k (L - l0_eff)^2.
template <bool F32>
__device__ __forceinline__ double spring_energy_term(const SampleArgs &a, long long s) {
    double xi, yi, zi, mi, xj, yj, zj, mj;
    load_pos<F32>(a, a.ssi[s], xi, yi, zi, mi);
    load_pos<F32>(a, a.ssj[s], xj, yj, zj, mj);
    const double dx = xj - xi, dy = yj - yi, dz = zj - zi;
    const double len = sqrt((dx * dx + dy * dy) + dz * dz);
    double l0 = a.sl0[s];
    if (a.sgrp) {
        const int g = a.sgrp[s];
        if (g >= 0) l0 = l0 * a.scale[g];
    }
    const double e = len - l0;
    return a.sk[s] * (e * e);
}

// GPE and KE terms of caller mass c.
template <bool F32>
__device__ __forceinline__ void mass_energy_terms(const SampleArgs &a, long long c, double &gpe, double &ke) {
    const int i = a.dev_of[c];
    const double m = a.mass[i];
    double x, y, z, mw, vx, vy, vz;
    load_pos<F32>(a, i, x, y, z, mw);
    load_vel<F32>(a, i, vx, vy, vz);
    gpe = a.g_mag > 0.0 ? (m * a.g_mag) * (((x * a.up[0] + y * a.up[1]) + z * a.up[2]) - a.datum) : 0.0;
    ke = m * ((vx * vx + vz * vz) + vy * vy);
}

// Element terms of one kind (SPRINGS: EPE; else GPE and KE).
template <bool F32, bool SPRINGS>
__device__ __forceinline__ void energy_terms(const SampleArgs &a, long long e, double &t0, double &t1) {
    if constexpr (SPRINGS) {
        t0 = spring_energy_term<F32>(a, e);
        t1 = 0.0;
    } else {
        mass_energy_terms<F32>(a, e, t0, t1);
    }
}

// Leaf sums: 8 lanes per leaf (4 leaves per warp).
template <bool F32, bool SPRINGS>
__global__ void __launch_bounds__(kSampleThreads) pw_leaf_kernel(SampleArgs a, PwPlanDev pl, double *v0, double *v1) {
    const long long gt = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long leaf = gt >> 3;
    const int j = (int)(gt & 7);
    const bool live = leaf < pl.n_leaves;
    const long long off = live ? pl.leaf_off[leaf] : 0;
    const int n = live ? pl.leaf_len[leaf] : 0;
    double r0 = 0.0, r1 = 0.0;
    if (live && n >= 8) {
        energy_terms<F32, SPRINGS>(a, off + j, r0, r1);
        const int body = n - (n & 7);
        for (int i = 8; i < body; i += 8) {
            double t0, t1;
            energy_terms<F32, SPRINGS>(a, off + i + j, t0, t1);
            r0 += t0;
            r1 += t1;
        }
    }
    // ((r0 + r1) + (r2 + r3)) + ((r4 + r5) + (r6 + r7)) across the 8 lanes
#pragma unroll
    for (int w = 1; w < 8; w <<= 1) {
        const double o0 = __shfl_down_sync(0xffffffffu, r0, w, 8);
        const double o1 = __shfl_down_sync(0xffffffffu, r1, w, 8);
        r0 = r0 + o0;
        r1 = r1 + o1;
    }
    if (!live || j != 0) return;
    if (n < 8) {                                            // only when the whole array is this short
        r0 = 0.0;
        r1 = 0.0;
        for (int i = 0; i < n; ++i) {
            double t0, t1;
            energy_terms<F32, SPRINGS>(a, off + i, t0, t1);
            r0 += t0;
            r1 += t1;
        }
    } else {
        for (int i = n - (n & 7); i < n; ++i) {
            double t0, t1;
            energy_terms<F32, SPRINGS>(a, off + i, t0, t1);
            r0 += t0;
            r1 += t1;
        }
    }
    v0[leaf] = r0;
    if (v1) v1[leaf] = r1;
}

// Internal nodes, one height at a time (one block).
__global__ void __launch_bounds__(1024) pw_combine_kernel(PwPlanDev pl, double *v0, double *v1) {
    for (int lv = 0; lv < pl.n_levels; ++lv) {
        for (int q = pl.level_start[lv] + threadIdx.x; q < pl.level_start[lv + 1]; q += blockDim.x) {
            const int4 nd = pl.nodes[q];
            v0[nd.z] = v0[nd.x] + v0[nd.y];
            if (v1) v1[nd.z] = v1[nd.x] + v1[nd.y];
        }
        __syncthreads();
    }
}

// (epe, gpe, ke, total) as engine.py:160-170 and :396-398 form them.
__global__ void pw_final_kernel(const double *vs, int root_s, const double *vg, const double *vk, int root_m,
                                bool has_springs, double g_mag, double *energy_row) {
    const double epe = has_springs ? 0.5 * (0.0 + vs[root_s]) : 0.0;
    const double gpe = g_mag > 0.0 ? 0.0 + vg[root_m] : 0.0;
    const double ke = 0.5 * (0.0 + vk[root_m]);
    energy_row[0] = epe;
    energy_row[1] = gpe;
    energy_row[2] = ke;
    energy_row[3] = (epe + gpe) + ke;
}

// Traced positions of one sample row.
template <bool F32>
__global__ void __launch_bounds__(kSampleThreads) sample_ids_kernel(SampleArgs a) {
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < a.n_ids; q += gridDim.x * blockDim.x) {
        double x, y, z, m;
        load_pos<F32>(a, a.ids[q], x, y, z, m);
        a.pos_row[3 * q + 0] = x;
        a.pos_row[3 * q + 1] = y;
        a.pos_row[3 * q + 2] = z;
    }
}

}  // namespace ss
