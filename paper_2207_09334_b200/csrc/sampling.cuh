// On-device sampling for simulate / RunResult (engine.py:476-565) and the
// energy breakdown (engine.py:148-170, energy_breakdown):
//
//   EPE = 1/2 sum_s k_s (|x_j - x_i| - l0_eff_s)^2
//   GPE = sum_m m |g| (x_m . up - datum),  up = -g/|g|  (0 without gravity)
//   KE  = 1/2 sum_m m |v_m|^2
//
// evaluated at a sampled state (Verlet: x_prev paired with the lagged central
// difference v, like the reference's simulate), accumulated in fp64 with a
// fixed-order block tree and a fixed-order final pass, so the numbers are
// deterministic (they differ from numpy's pairwise sums only by rounding:
// sampling, not part of the stepped state).  Traced positions are gathered
// into a row buffer; rows stay on the device until the run segment ends.
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
    const int *ids;              // traced masses (device ids)
    int n_ids;
    double *pos_row;             // n_ids x 3
    double *partial;             // gridDim.x x 3
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

// fixed-order tree over the block (blockDim.x == kSampleThreads)
__device__ __forceinline__ void block_sum3(double &a, double &b, double &c, double *sh) {
    const int t = threadIdx.x;
    sh[t] = a;
    sh[kSampleThreads + t] = b;
    sh[2 * kSampleThreads + t] = c;
    __syncthreads();
    for (int w = kSampleThreads / 2; w > 0; w >>= 1) {
        if (t < w) {
            sh[t] += sh[t + w];
            sh[kSampleThreads + t] += sh[kSampleThreads + t + w];
            sh[2 * kSampleThreads + t] += sh[2 * kSampleThreads + t + w];
        }
        __syncthreads();
    }
    a = sh[0];
    b = sh[kSampleThreads];
    c = sh[2 * kSampleThreads];
}

// Per-block partial (epe, gpe, ke) + the traced positions (block 0).
template <bool F32>
__global__ void __launch_bounds__(kSampleThreads) sample_partial_kernel(SampleArgs a) {
    __shared__ double sh[3 * kSampleThreads];
    const long long stride = (long long)gridDim.x * blockDim.x;
    const long long t0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    double epe = 0.0, gpe = 0.0, ke = 0.0;
    for (long long s = t0; s < a.n_springs; s += stride) {
        double xi, yi, zi, mi, xj, yj, zj, mj;
        load_pos<F32>(a, a.ssi[s], xi, yi, zi, mi);
        load_pos<F32>(a, a.ssj[s], xj, yj, zj, mj);
        const double dx = xj - xi, dy = yj - yi, dz = zj - zi;
        const double len = sqrt(dx * dx + dy * dy + dz * dz);
        double l0 = a.sl0[s];
        if (a.sgrp) {
            const int g = a.sgrp[s];
            if (g >= 0) l0 = l0 * a.scale[g];
        }
        const double e = len - l0;
        epe += a.sk[s] * (e * e);
    }
    for (long long i = t0; i < a.nd; i += stride) {
        double x, y, z, mw, vx, vy, vz;
        const double m = a.mass[i];                         // the caller's fp64 mass (fp32 state holds a rounded copy)
        if (m == 0.0) continue;                             // padding slot
        load_pos<F32>(a, (int)i, x, y, z, mw);
        load_vel<F32>(a, (int)i, vx, vy, vz);
        if (a.g_mag > 0.0) gpe += m * a.g_mag * ((x * a.up[0] + y * a.up[1] + z * a.up[2]) - a.datum);
        ke += m * (vx * vx + vy * vy + vz * vz);
    }
    block_sum3(epe, gpe, ke, sh);
    if (threadIdx.x == 0) {
        a.partial[3 * blockIdx.x + 0] = epe;
        a.partial[3 * blockIdx.x + 1] = gpe;
        a.partial[3 * blockIdx.x + 2] = ke;
    }
    if (blockIdx.x == 0) {
        for (int q = threadIdx.x; q < a.n_ids; q += blockDim.x) {
            double x, y, z, m;
            load_pos<F32>(a, a.ids[q], x, y, z, m);
            a.pos_row[3 * q + 0] = x;
            a.pos_row[3 * q + 1] = y;
            a.pos_row[3 * q + 2] = z;
        }
    }
}

// One block: sum the partials in block order, write (epe, gpe, ke, total).
__global__ void __launch_bounds__(kSampleThreads) sample_final_kernel(const double *partial, int nblocks,
                                                                      double *energy_row) {
    __shared__ double sh[3 * kSampleThreads];
    double epe = 0.0, gpe = 0.0, ke = 0.0;
    for (int b = threadIdx.x; b < nblocks; b += blockDim.x) {
        epe += partial[3 * b + 0];
        gpe += partial[3 * b + 1];
        ke += partial[3 * b + 2];
    }
    block_sum3(epe, gpe, ke, sh);
    if (threadIdx.x == 0) {
        const double e = 0.5 * epe, k = 0.5 * ke;
        energy_row[0] = e;
        energy_row[1] = gpe;
        energy_row[2] = k;
        energy_row[3] = (e + gpe) + k;
    }
}

}  // namespace ss
