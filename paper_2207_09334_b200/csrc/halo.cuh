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
// One process per GPU, neighbours on the same node (NVLink/NVSwitch).  The
// step kernels themselves store the boundary planes into the neighbours'
// position buffers and synchronise through step flags (kernels.cuh
// xchg_wait / xchg_store / xchg_finish); this mailbox holds the flags:
//   int64 flag[2]   last step the lower / upper neighbour has completed
//                   (written by the neighbour, release, system scope)
//   uint32 counter  this shard's grid completion counter
//   int32 error     a neighbour was silent past the timeout
struct MailboxHead {
    long long flag[2];
    unsigned counter[2];
    int error;
};
constexpr size_t kMailboxHead = 256;

}  // namespace ss
