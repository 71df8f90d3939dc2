// Halo exchange for x-slab sharding.
//
// A shard's local scene holds its owned masses plus one halo plane per
// neighbour; halo masses are marked fixed, so the step kernel leaves them in
// place, and after every substep their positions are overwritten with the
// neighbour's freshly integrated boundary plane.  Only x (fp64) / the
// displacement r (fp32; both shards hold the same base P for a mass) moves;
// the receiving side keeps its own .w (the fixed flag differs per shard).
#pragma once

#include <cuda_runtime.h>

namespace ss {

template <typename T4>
__global__ void halo_pack_kernel(const T4 *__restrict__ X, const int *__restrict__ idx, int n,
                                 T4 *__restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = X[idx[i]];
}

template <typename T4>
__global__ void halo_unpack_kernel(T4 *__restrict__ X, const int *__restrict__ idx, int n,
                                   const T4 *__restrict__ in) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        T4 v = X[idx[i]];
        const T4 r = in[i];
        v.x = r.x;
        v.y = r.y;
        v.z = r.z;
        X[idx[i]] = v;
    }
}

// Same-device neighbour (virtual shards): copy src boundary plane straight
// into dst's halo slots.
template <typename T4>
__global__ void halo_copy_kernel(const T4 *__restrict__ Xs, const int *__restrict__ sidx,
                                 T4 *__restrict__ Xd, const int *__restrict__ didx, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        const T4 r = Xs[sidx[i]];
        T4 v = Xd[didx[i]];
        v.x = r.x;
        v.y = r.y;
        v.z = r.z;
        Xd[didx[i]] = v;
    }
}

// ------------------------------------------------------ peer-memory transport
// One process per GPU, neighbours on the same node (NVLink/NVSwitch): every
// substep each shard
//  1. halo_push_kernel: stores its freshly integrated boundary planes straight
//     into the neighbours' mailboxes (CUDA-IPC-mapped device memory, i.e.
//     NVLink P2P stores); the last CTA of each side then publishes the step
//     number in the neighbour's flag word (st.release.sys);
//  2. halo_land_kernel: waits (ld.acquire.sys) until each neighbour has
//     published this step and copies the mailbox planes into its own halo
//     slots (x / r only; .w stays, the halo masses are fixed here).
// Both are ordered on the shard's stream after its step kernel, so the next
// step kernel sees complete halos; no host round trip, no NCCL.  Plane
// buffers are double-buffered by step parity: a shard pushes step n+2 into
// the buffer its neighbour read at step n only after landing step n+1, which
// the neighbour published after landing step n (transitively ordered).
//
// Mailbox (allocated by the receiving shard, exported by IPC handle):
//   [0, 256): int64 flag[2] (last step landed from the lower / upper
//             neighbour), uint32 push counters[2] (the shard's own), int32
//             error word;
//   then per side s: 2 parity buffers of n_recv[s] T4.
struct MailboxHead {
    long long flag[2];
    unsigned counter[2];
    int error;
};
constexpr size_t kMailboxHead = 256;
constexpr long long kLandTimeoutNs = 20000000000ll;   // 20 s: a lost neighbour is an error, not a hang

template <typename T4>
struct PushArgs {
    const T4 *X;                  // this shard's new state
    const int *send_idx[2];
    int n_send[2];
    T4 *peer_buf[2];              // this step's parity buffer in the neighbour's mailbox (null: no neighbour)
    long long *peer_flag[2];      // the neighbour's flag word for this side
    unsigned *counter[2];         // this shard's completion counters
    int blocks0;                  // CTAs of side 0
    long long step;
};

template <typename T4>
__global__ void __launch_bounds__(256) halo_push_kernel(PushArgs<T4> a) {
    const int s = (int)blockIdx.x < a.blocks0 ? 0 : 1;
    const int b = s ? (int)blockIdx.x - a.blocks0 : (int)blockIdx.x;
    const int i = b * blockDim.x + threadIdx.x;
    if (i < a.n_send[s]) a.peer_buf[s][i] = a.X[a.send_idx[s][i]];
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned nb = s ? gridDim.x - (unsigned)a.blocks0 : (unsigned)a.blocks0;
        if (atomicAdd(a.counter[s], 1u) == nb - 1) {        // last CTA of this side
            *a.counter[s] = 0u;
            __threadfence_system();
            asm volatile("st.release.sys.global.s64 [%0], %1;" ::"l"(a.peer_flag[s]), "l"(a.step) : "memory");
        }
    }
}

template <typename T4>
struct LandArgs {
    T4 *X;                        // this shard's new state
    const int *recv_idx[2];
    int n_recv[2];
    const T4 *buf[2];             // this step's parity buffer in the own mailbox (null: no neighbour)
    const long long *flag[2];
    int *error;
    int blocks0;
    long long step;
};

__device__ __forceinline__ float4 ld_cg(const float4 *p) { return __ldcg(p); }
__device__ __forceinline__ double4 ld_cg(const double4 *p) {
    const double2 a = __ldcg(reinterpret_cast<const double2 *>(p));
    const double2 b = __ldcg(reinterpret_cast<const double2 *>(p) + 1);
    return make_double4(a.x, a.y, b.x, b.y);
}

template <typename T4>
__global__ void __launch_bounds__(256) halo_land_kernel(LandArgs<T4> a) {
    const int s = (int)blockIdx.x < a.blocks0 ? 0 : 1;
    const int b = s ? (int)blockIdx.x - a.blocks0 : (int)blockIdx.x;
    if (threadIdx.x == 0) {
        long long seen, t0, t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        for (;;) {
            asm volatile("ld.acquire.sys.global.s64 %0, [%1];" : "=l"(seen) : "l"(a.flag[s]) : "memory");
            if (seen >= a.step) break;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            if (t - t0 > kLandTimeoutNs) {
                atomicExch(a.error, 1);
                break;
            }
            __nanosleep(256);
        }
    }
    __syncthreads();
    const int i = b * blockDim.x + threadIdx.x;
    if (i < a.n_recv[s]) {
        T4 v = a.X[a.recv_idx[s][i]];
        const T4 r = ld_cg(a.buf[s] + i);                   // written by the neighbour: bypass L1
        v.x = r.x;
        v.y = r.y;
        v.z = r.z;
        a.X[a.recv_idx[s][i]] = v;
    }
}

}  // namespace ss
