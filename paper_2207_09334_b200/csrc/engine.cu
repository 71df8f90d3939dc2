// Engine object and C ABI (include/springsim_b200.h).
//
// Host side of the relaxation loop: freezes a scene description into device
// buffers (engine.py:182-246), builds the incidence layout, and drives the
// per-step kernels of kernels.cuh on a private CUDA stream.  A batch of
// `count` steps is enqueued back-to-back with the divergence check fused
// into each step's epilogue, so a batch costs one host synchronisation, not
// one per step (engine.py:366-373 checks after every step).

#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <map>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <type_traits>
#include <utility>
#include <string>
#include <vector>

#include "common.h"
#include "kernels.cuh"
#include "tile_f32.cuh"
#include "tile_f64.cuh"
#include "sampling.cuh"
#include "layout.h"
#include "springsim_b200.h"
#include "tiles.h"
#include "halo.cuh"
#include "resident.cuh"
#include "nccl_shim.h"

using namespace ss;

#define CK(expr)                                                                         \
    do {                                                                                 \
        cudaError_t _e = (expr);                                                         \
        if (_e != cudaSuccess)                                                           \
            return ss::fail(SS_ECUDA, "%s failed: %s", #expr, cudaGetErrorString(_e));   \
    } while (0)

namespace {

constexpr int kBlock = kBlockThreads;
// fp32 inline tiles stage X0 too (tile_f32.cuh): ~57 KB per CTA on the 10M
// cube, so at most 4 CTAs per SM -- let the kernel have the registers
constexpr int kInlineMinB = 4;

struct Group {
    int mode;
    double amplitude, frequency, phase;
};

struct DevBuf {
    void *p = nullptr;
    size_t bytes = 0;
};

}  // namespace

struct ss_engine {
    int device = 0;
    cudaStream_t stream = nullptr;
    int precision = SS_F64, layout = SS_LAYOUT_CSR, integrator = SS_VERLET;
    int64_t N = 0, S = 0;
    int64_t ND = 0;                // device mass slots (TILE: padded to whole tiles)

    // host-side scalars (engine.py:190-194, 222-224)
    double dt = 1e-4, damping = 0.0, gravity[3] = {0, 0, 0};
    double gpe_datum = 0.0;        // GPE reference height (engine.py:240-242), sampling only
    std::vector<Group> groups;
    std::vector<double> planes;    // 6 per plane
    std::vector<double> m;         // masses (caller order)
    std::vector<uint8_t> fixed;    // caller order
    std::vector<int32_t> orig_of;  // device id -> caller id (empty: identity)
    std::vector<float> base;       // fp32 base positions, device order, 4 per mass
    std::vector<double> x0;        // fp32 TILE: rest positions X0 (device order, 3 per slot); state r = x - X0
    bool rx0 = false;              // fp32 TILE engines keep r = x - X0 (tiles.h), others r = x - P
    double t = 0.0;
    int64_t n = 0;
    bool has_prev = false;
    void *U = nullptr;             // fp32 Verlet: u = x - x_prev (increment form, kernels.cuh verlet_u)
    bool has_fext = false;

    // device state (device order)
    std::vector<DevBuf> bufs;
    void *X[2] = {nullptr, nullptr};
    int cur = 0;
    void *V = nullptr;
    void *P = nullptr;
    void *F = nullptr;
    void *XA = nullptr, *XB = nullptr, *VS = nullptr, *SV = nullptr, *SA = nullptr;  // RK4
    void *scale = nullptr;
    size_t scale_cap = 0;
    unsigned long long *d_degenerate = nullptr;
    void *pinned[3] = {nullptr, nullptr, nullptr};   // page-locked staging for state transfers
    // fp64 state transfers in the caller's layout ((N,3) f64, 24 B per mass):
    // two pinned chunk buffers (host memcpy into one overlaps the DMA out of
    // the other), a device staging array, and the +-m word of every slot
    void *chunk_buf[2] = {nullptr, nullptr};
    cudaEvent_t chunk_done[2] = {nullptr, nullptr};
    double *d_raw = nullptr;
    double *d_w = nullptr;
    double *d_raw2 = nullptr;                  // fp32: second caller-layout buffer (v, x_prev)
    double *d_x0dev = nullptr;                 // fp32 tiles: X0 per device slot, fp64
    size_t pinned_bytes[3] = {0, 0, 0};
    cudaEvent_t staged = nullptr;              // recorded after asynchronous uploads from `pinned`
    cudaEvent_t chunk_ev[4] = {nullptr, nullptr, nullptr, nullptr};   // chunked downloads
    bool staged_pending = false;
    // on-device sampling (ss_energy_setup / ss_step_sampled)
    int *d_ssi = nullptr, *d_ssj = nullptr, *d_sgrp = nullptr;
    double *d_sk = nullptr, *d_sl0 = nullptr, *d_smass = nullptr, *d_sx0 = nullptr;
    int64_t energy_springs = -1;               // -1: ss_energy_setup not called
    DevBuf d_sids, d_srows, d_serows, d_sscale;
    int *d_sdev_of = nullptr;                  // caller mass id -> device slot
    PwPlanDev pw_springs{}, pw_masses{};       // numpy pairwise-sum plans (sampling.cuh)
    double *d_pwv[3] = {nullptr, nullptr, nullptr};   // their node values: EPE; GPE, KE
    long long *d_div_step = nullptr;
    int *d_div_mass = nullptr;
    int *d_orig_of = nullptr;
    void *d_acc = nullptr;
    void *d_tmp[2] = {nullptr, nullptr};

    // topology
    Layout lay;
    TileLayout tl;
    void *k = nullptr, *l0 = nullptr, *e_k = nullptr, *e_l0 = nullptr;
    int *row = nullptr, *grp = nullptr, *e_other = nullptr, *e_grp = nullptr, *r_pos = nullptr,
        *cnt = nullptr;
    int2 *inc = nullptr;
    unsigned char *d_blob = nullptr;
    double2 *d_kl_inline = nullptr;            // fp64 inline tile format (tiles.h)
    float2 *d_kd_inline = nullptr;             // fp32 inline tile format (+ d_x0dev)
    int8_t *d_g_inline = nullptr;
    unsigned long long *d_kl_off = nullptr;
    unsigned long long *d_toff = nullptr;
    unsigned int *d_tsplit = nullptr;
    uint32_t blob_smem = 0, max_halo = 0;
    size_t smem_bytes = 0;
    size_t lean_smem = 0;          // fp32 Euler/Verlet compact-format tile kernel (tile_f32.cuh), 0 = off
    size_t f64_smem = 0;           // fp64 Euler/Verlet compact-format tile kernel (tile_f64.cuh), 0 = off
    int f64_variant = 0;           // its (UNROLL, MINB) instantiation: 0 (2,4), 1 (1,4), 2 (2,3), 3 (3,3), 4 (1,5), 5 (2,5)
    int f64_rk4_variant = 0;       // the RK4 stages' instantiation: 0 (2,4) or 3 (3,3)
    int lean_lanes = 1;            // threads per mass of that kernel (2: scenes with few tiles)
    int persist_max_grid = 0;      // co-resident CTAs of the persistent kernel (0: never persistent)
    bool pdl = true;               // programmatic dependent launch between substeps (SS_PDL=0: off)
    int64_t device_bytes = 0;
    int64_t launches = 0;
    int64_t pending = 0;
    int64_t pending_n0 = 0;
    int pending_cur0 = 0;
    // async batches in flight (oldest first): the event recorded after each
    // and its step count (ss_pending_wait); spare events
    std::vector<std::pair<cudaEvent_t, int64_t>> inflight;
    std::vector<cudaEvent_t> spare_events;
    // a divergence found while settling async steps behind another call: it
    // is reported by the next ss_step / ss_sync, never dropped
    bool div_held = false;
    ss_step_result held{};

    // halo exchange (x-slab sharding); side 0 = lower neighbour, 1 = upper
    bool halo_on = false;
    int halo_n_send[2] = {0, 0}, halo_n_recv[2] = {0, 0};
    int *halo_send_idx[2] = {nullptr, nullptr}, *halo_recv_idx[2] = {nullptr, nullptr};
    void *halo_send[2] = {nullptr, nullptr}, *halo_recv[2] = {nullptr, nullptr};
    ncclComm_t nccl = nullptr;
    int nccl_peer[2] = {-1, -1};
    int64_t halo_exchanges = 0;
    int rk4_stage_only = 0;        // ss_step_group: launch only this RK4 stage (1-4) of a one-step batch
    long long *group_div_step = nullptr;   // ss_step_group: the group's shared divergence step word
    // fused peer-memory exchange (kernels.cuh xchg_*): own flag mailbox, the
    // neighbours' mailboxes and position buffers (IPC-mapped or, for shards of
    // one process, plain), their slots for this shard's planes
    void *mailbox = nullptr;
    void *peer_mailbox[2] = {nullptr, nullptr};
    void *peer_X[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};   // [side][buffer]
    void *peer_XA[2] = {nullptr, nullptr}, *peer_XB[2] = {nullptr, nullptr};   // RK4: the stage buffers
    bool peer_ipc[2] = {false, false};
    std::vector<int32_t> peer_recv[2];          // the neighbour's device slots for this shard's planes
    std::vector<int32_t> halo_send_host[2], halo_recv_host[2];   // this shard's plane slots
    unsigned char *d_tile_role = nullptr;
    int2 *d_peer_slot = nullptr;
    int *d_tile_order = nullptr;
    int xchg_arrivals = 0;         // CTAs that read ghosts or push (kernels.cuh xchg_finish)
    bool p2p_on = false;
    // CTA-resident small-scene kernel (resident.cuh): record image and launch shape
    void *res_image = nullptr;
    unsigned *res_segd = nullptr;                 // per-CTA segment offsets in the image (device)
    unsigned res_dict_bytes = 0, res_off[3] = {0, 0, 0};   // smem offsets: dict, groups, segment
    size_t res_smem = 0;
    int res_ctas = 0, res_pslots = 0, res_g = 0, res_threads = 0;
    // CUDA-graph replays of whole batches (launch_steps): a batch of `count`
    // substeps from buffer parity `cur` with identical launch parameters is
    // captured once (on its second occurrence) and replayed; the step
    // numbers come from the device word d_step_base (Params::step_base)
    struct GraphEntry {
        std::vector<unsigned char> key;
        cudaGraphExec_t exec = nullptr;
        uint64_t last_use = 0;
    };
    std::vector<GraphEntry> graphs;
    std::vector<std::vector<unsigned char>> graph_seen;   // keys met once
    uint64_t graph_clock = 0;
    long long *d_step_base = nullptr;
    int64_t graph_base_n = -1;                            // the device step base after the queued work (-1: unknown)
    bool use_graphs = true;                               // SS_GRAPH=0: off
    int pdl_graph = -1;                                   // PDL inside captured graphs (-1: as pdl; autotune_pdl)
    bool graph_capturing = false;

    ~ss_engine() {
        if (device >= 0) cudaSetDevice(device);
        if (stream) cudaStreamSynchronize(stream);
        for (auto &g : graphs)
            if (g.exec) cudaGraphExecDestroy(g.exec);
        for (int s = 0; s < 2; ++s) {
            if (!peer_ipc[s]) continue;
            if (peer_mailbox[s]) cudaIpcCloseMemHandle(peer_mailbox[s]);
            for (void *b : peer_X[s])
                if (b) cudaIpcCloseMemHandle(b);
        }
        if (nccl) {
            if (const NcclApi *api = nccl_api()) api->commDestroy(nccl);
        }
        for (auto &b : bufs) cudaFree(b.p);
        if (stream) cudaStreamSynchronize(stream);
        for (auto &f : inflight) cudaEventDestroy(f.first);
        for (cudaEvent_t e : spare_events) cudaEventDestroy(e);
        for (void *b : pinned)
            if (b) cudaFreeHost(b);
        for (void *b : chunk_buf)
            if (b) cudaFreeHost(b);
        for (cudaEvent_t e : chunk_done)
            if (e) cudaEventDestroy(e);
        if (staged) cudaEventDestroy(staged);
        for (cudaEvent_t e : chunk_ev)
            if (e) cudaEventDestroy(e);
        if (stream) cudaStreamDestroy(stream);
    }

    template <typename P_>
    int alloc(P_ **out, size_t bytes) {
        void *p = nullptr;
        if (bytes == 0) bytes = 16;
        cudaError_t e = cudaMalloc(&p, bytes);
        if (e != cudaSuccess)
            return ss::fail(SS_ECUDA, "cudaMalloc(%zu) failed: %s", bytes, cudaGetErrorString(e));
        bufs.push_back({p, bytes});
        device_bytes += (int64_t)bytes;
        *out = reinterpret_cast<P_ *>(p);
        return SS_OK;
    }

    int64_t src_of(int64_t i) const { return orig_of.empty() ? i : orig_of[i]; }
    int grid() const { return (int)((ND + kBlockThreads - 1) / kBlockThreads); }
};

namespace {

// ------------------------------------------------------------ conversions
// Host arrays are (N,3) f64 in caller order; device arrays are T4 in device
// order (orig_of permutation).  fp64: (x, y, z, +-m); fp32: r = float(x - P).

template <typename T, typename T4>
void pack_positions(const ss_engine *h, const double *x, T4 *out) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < h->ND; ++i) {
        const int64_t s = h->src_of(i);
        T4 o{};
        if (s < 0) {                 // padding slot
            out[i] = o;
            continue;
        }
        const double w = h->fixed[s] ? -h->m[s] : h->m[s];
        if constexpr (std::is_same<T, float>::value) {
            if (h->rx0) {
                const double *b = h->x0.data() + 3 * i;
                o.x = (float)(x[3 * s + 0] - b[0]);
                o.y = (float)(x[3 * s + 1] - b[1]);
                o.z = (float)(x[3 * s + 2] - b[2]);
            } else {
                const float *b = h->base.data() + 4 * i;
                o.x = (float)(x[3 * s + 0] - (double)b[0]);
                o.y = (float)(x[3 * s + 1] - (double)b[1]);
                o.z = (float)(x[3 * s + 2] - (double)b[2]);
            }
            o.w = (float)w;
        } else {
            o.x = x[3 * s + 0];
            o.y = x[3 * s + 1];
            o.z = x[3 * s + 2];
            o.w = w;
        }
        out[i] = o;
    }
}

template <typename T, typename T4>
void pack_vec(const ss_engine *h, const double *v, T4 *out) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < h->ND; ++i) {
        const int64_t s = h->src_of(i);
        T4 o{};
        if (s < 0) {
            out[i] = o;
            continue;
        }
        o.x = (T)v[3 * s + 0];
        o.y = (T)v[3 * s + 1];
        o.z = (T)v[3 * s + 2];
        o.w = (T)0;
        out[i] = o;
    }
}

template <typename T, typename T4>
void unpack_positions(const ss_engine *h, const T4 *in, double *x, int64_t i0, int64_t i1) {
#pragma omp parallel for schedule(static)
    for (int64_t i = i0; i < i1; ++i) {
        const int64_t s = h->src_of(i);
        if (s < 0) continue;
        if constexpr (std::is_same<T, float>::value) {
            if (h->rx0) {
                const double *b = h->x0.data() + 3 * i;
                x[3 * s + 0] = b[0] + (double)in[i].x;
                x[3 * s + 1] = b[1] + (double)in[i].y;
                x[3 * s + 2] = b[2] + (double)in[i].z;
            } else {
                const float *b = h->base.data() + 4 * i;
                x[3 * s + 0] = (double)b[0] + (double)in[i].x;
                x[3 * s + 1] = (double)b[1] + (double)in[i].y;
                x[3 * s + 2] = (double)b[2] + (double)in[i].z;
            }
        } else {
            x[3 * s + 0] = in[i].x;
            x[3 * s + 1] = in[i].y;
            x[3 * s + 2] = in[i].z;
        }
    }
}

template <typename T, typename T4>
void unpack_vec(const ss_engine *h, const T4 *in, double *v, int64_t i0, int64_t i1) {
#pragma omp parallel for schedule(static)
    for (int64_t i = i0; i < i1; ++i) {
        const int64_t s = h->src_of(i);
        if (s < 0) continue;
        v[3 * s + 0] = (double)in[i].x;
        v[3 * s + 1] = (double)in[i].y;
        v[3 * s + 2] = (double)in[i].z;
    }
}

int upload(ss_engine *h, void *dst, const void *src, size_t bytes) {
    CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    return SS_OK;
}
int download(ss_engine *h, void *dst, const void *src, size_t bytes) {
    CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    return SS_OK;
}

// Device state vector src (ND slots) -> pinned dst in chunks, each chunk
// handed to `consume(i0, i1)` (the unpacking loop) as soon as it has
// landed, while the next chunks are still crossing the bus.
template <typename T4, typename Fn>
int download_overlapped(ss_engine *h, T4 *dst, const void *src, Fn &&consume) {
    constexpr int kChunks = 4;
    const int64_t ND = h->ND;
    if (!h->chunk_ev[0])
        for (auto &e : h->chunk_ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    int64_t lo[kChunks + 1];
    for (int c = 0; c <= kChunks; ++c) lo[c] = ND * c / kChunks;
    for (int c = 0; c < kChunks; ++c) {
        const size_t n = (size_t)(lo[c + 1] - lo[c]);
        if (n) CK(cudaMemcpyAsync(dst + lo[c], reinterpret_cast<const T4 *>(src) + lo[c], n * sizeof(T4),
                                  cudaMemcpyDeviceToHost, h->stream));
        CK(cudaEventRecord(h->chunk_ev[c], h->stream));
    }
    for (int c = 0; c < kChunks; ++c) {
        CK(cudaEventSynchronize(h->chunk_ev[c]));
        consume(lo[c], lo[c + 1]);
    }
    return SS_OK;
}

// ----------------------------------------------------------- actuation

// Actuation scale of every group at time ts, the exact Python expression of
// engine.py:250-259 (math.sin is libm sin; host code built -ffp-contract=off).
void scales_at(const ss_engine *h, double ts, double *out) {
    for (size_t g = 0; g < h->groups.size(); ++g) {
        const Group &gr = h->groups[g];
        out[g] = gr.mode == SS_CONSTANT_EXPANSION
                     ? 1.0 + gr.amplitude
                     : 1.0 + gr.amplitude * std::sin(2.0 * M_PI * gr.frequency * ts + gr.phase);
    }
}

// Table for `count` steps starting at (t0, n0).  Euler/Verlet evaluate at
// self.t (t0 for the first step, n*dt afterwards); RK4 at t, t+dt/2 (x2), t+dt.
void build_scales(const ss_engine *h, int64_t count, int stages, double t0, int64_t n0,
                  std::vector<double> &out) {
    const size_t G = h->groups.size();
    out.resize((size_t)count * stages * G);
    for (int64_t s = 0; s < count; ++s) {
        const double ts = (s == 0) ? t0 : (double)(n0 + s) * h->dt;
        double st[4] = {ts, ts, ts, ts};
        if (stages == 4) {
            st[1] = ts + 0.5 * h->dt;
            st[2] = ts + 0.5 * h->dt;
            st[3] = ts + h->dt;
        }
        for (int q = 0; q < stages; ++q) scales_at(h, st[q], &out[((size_t)s * stages + q) * G]);
    }
}

template <typename T>
int upload_scales(ss_engine *h, const std::vector<double> &tab) {
    if (tab.empty()) return SS_OK;
    const size_t bytes = tab.size() * sizeof(T);
    if (bytes > h->scale_cap) {
        void *p;
        const size_t cap = std::max<size_t>(bytes, 4096);
        int rc = h->alloc(&p, cap);
        if (rc) return rc;
        h->scale = p;          // the old buffer stays owned by h->bufs until destruction
        h->scale_cap = cap;
    }
    if constexpr (std::is_same<T, double>::value) {
        return upload(h, h->scale, tab.data(), bytes);
    } else {
        std::vector<float> f(tab.begin(), tab.end());
        return upload(h, h->scale, f.data(), bytes);
    }
}

// ------------------------------------------------------------ params

template <typename T>
Params<T> base_params(const ss_engine *h) {
    using T4 = typename Params<T>::T4;
    Params<T> p{};
    p.n = (int)h->ND;
    p.P = reinterpret_cast<const T4 *>(h->P);
    p.F = h->has_fext ? reinterpret_cast<const T4 *>(h->F) : nullptr;
    p.orig_of = h->d_orig_of;
    Topology<T> &tp = p.topo;
    tp.row = h->row;
    tp.inc = h->inc;
    tp.k = reinterpret_cast<const T *>(h->k);
    tp.l0 = reinterpret_cast<const T *>(h->l0);
    tp.grp = h->grp;
    tp.e_other = h->e_other;
    tp.e_k = reinterpret_cast<const T *>(h->e_k);
    tp.e_l0 = reinterpret_cast<const T *>(h->e_l0);
    tp.e_grp = h->e_grp;
    tp.r_pos = h->r_pos;
    tp.cnt = h->cnt;
    tp.W = h->lay.W;
    tp.Wr = h->lay.Wr;
    tp.blob = h->d_blob;
    tp.toff = h->d_toff;
    tp.tsplit = h->d_tsplit;
    tp.blob_smem = h->blob_smem;
    tp.max_halo = h->max_halo;
    tp.n_tiles = (int)h->tl.n_tiles;
    tp.kl_inline = h->d_kl_inline;
    tp.g_inline = h->d_g_inline;
    tp.kl_off = h->d_kl_off;
    tp.kd_inline = h->d_kd_inline;
    tp.x0 = h->d_x0dev;
    for (int c = 0; c < 3; ++c) p.g[c] = (T)h->gravity[c];
    p.dt = (T)h->dt;
    p.half_dt = (T)(0.5 * h->dt);
    p.dt2_over = (T)(h->dt * h->dt);
    p.two_dt = (T)(2.0 * h->dt);
    p.one_minus_d = (T)(1.0 - h->damping);
    p.dt6 = (T)(h->dt / 6.0);
    p.damped = h->damping != 0.0;
    p.n_planes = (int)(h->planes.size() / 6);
    for (int q = 0; q < p.n_planes; ++q) {
        for (int c = 0; c < 3; ++c) p.pn[q][c] = (T)h->planes[6 * q + c];
        p.poff[q] = (T)h->planes[6 * q + 3];
        p.ppen[q] = (T)h->planes[6 * q + 4];
        p.pfric[q] = (T)h->planes[6 * q + 5];
    }
    p.degenerate = h->d_degenerate;
    p.div_step = h->group_div_step ? h->group_div_step : h->d_div_step;
    p.div_mass = h->d_div_mass;
    if (const char *dbg = getenv("SS_DEBUG")) p.debug = atoi(dbg);   // timing experiments only
    return p;
}

// Call fn(std::integral_constant<int, LAYOUT>{}) for the engine's layout.
template <typename Fn>
int with_layout(const ss_engine *h, Fn &&fn) {
    switch (h->layout) {
        case SS_LAYOUT_CSR: return fn(std::integral_constant<int, 1>{});
        case SS_LAYOUT_ELL: return fn(std::integral_constant<int, 2>{});
        default:
            if (h->tl.canonical && h->groups.empty()) return fn(std::integral_constant<int, 4>{});
            return fn(std::integral_constant<int, 3>{});
    }
}

// After a substep: pack the boundary planes of the new positions, exchange
// them with the neighbouring ranks (NCCL send/recv on the engine stream) and
// write the received planes into the halo slots.
// Exchange fields of one step's Params (fused peer-memory transport): the
// neighbours' buffers for this step's output parity, the flag words.
// RK4 (stage 1-4): the neighbours' buffer for this stage's trial positions
// (XA, XB, XA, then the state), sequence number 4 (step - 1) + stage.
template <typename T>
void xchg_params(const ss_engine *h, Params<T> &p, int stage = 0) {
    using T4 = typename Params<T>::T4;
    MailboxHead *mine = reinterpret_cast<MailboxHead *>(h->mailbox);
    p.xchg = 1;
    p.xseq = stage ? 4 * (p.step - 1) + stage : p.step;
    p.tile_role = h->d_tile_role;
    p.peer_slot = h->d_peer_slot;
    for (int s = 0; s < 2; ++s) {
        void *out = stage == 0 ? h->peer_X[s][h->cur ^ 1]
                  : stage == 4 ? h->peer_X[s][h->cur]
                  : stage == 2 ? h->peer_XB[s] : h->peer_XA[s];
        p.peer_out[s] = h->peer_mailbox[s] ? reinterpret_cast<T4 *>(out) : nullptr;
        p.peer_flag[s] = h->peer_mailbox[s] ? &reinterpret_cast<MailboxHead *>(h->peer_mailbox[s])->flag[1 - s]
                                            : nullptr;
        p.my_flag[s] = &mine->flag[s];
    }
    p.done_ctas = &mine->counter[0];
    p.xchg_arrivals = h->xchg_arrivals;
    p.tile_order = h->d_tile_order;
    p.xchg_error = &mine->error;
}

// X: the position buffer whose boundary planes travel (default: the current
// state; RK4 exchanges each stage's trial positions).
template <typename T4>
int halo_exchange_nccl(ss_engine *h, T4 *X = nullptr) {
    const NcclApi *api = nccl_api();
    if (!api) return SS_ECUDA;
    if (!X) X = reinterpret_cast<T4 *>(h->X[h->cur]);
    for (int s = 0; s < 2; ++s)
        if (h->halo_n_send[s] && h->nccl_peer[s] >= 0)
            halo_pack_kernel<T4><<<(h->halo_n_send[s] + 255) / 256, 256, 0, h->stream>>>(
                X, h->halo_send_idx[s], h->halo_n_send[s], reinterpret_cast<T4 *>(h->halo_send[s]));
    const size_t words = sizeof(T4) / sizeof(float);
    ncclResult_t r = api->groupStart();
    for (int s = 0; s < 2 && r == ncclSuccess; ++s) {
        if (h->nccl_peer[s] < 0) continue;
        if (h->halo_n_send[s])
            r = api->send(h->halo_send[s], (size_t)h->halo_n_send[s] * words, ncclFloat32, h->nccl_peer[s],
                          h->nccl, h->stream);
        if (r == ncclSuccess && h->halo_n_recv[s])
            r = api->recv(h->halo_recv[s], (size_t)h->halo_n_recv[s] * words, ncclFloat32, h->nccl_peer[s],
                          h->nccl, h->stream);
    }
    const ncclResult_t r2 = api->groupEnd();
    if (r != ncclSuccess || r2 != ncclSuccess)
        return ss::fail(SS_ECUDA, "NCCL halo exchange failed: %s",
                        api->getErrorString(r != ncclSuccess ? r : r2));
    for (int s = 0; s < 2; ++s)
        if (h->halo_n_recv[s] && h->nccl_peer[s] >= 0)
            halo_unpack_kernel<T4><<<(h->halo_n_recv[s] + 255) / 256, 256, 0, h->stream>>>(
                X, h->halo_recv_idx[s], h->halo_n_recv[s], reinterpret_cast<const T4 *>(h->halo_recv[s]));
    h->launches += 2;
    h->halo_exchanges += 1;
    CK(cudaGetLastError());
    return SS_OK;
}

// fp32 Euler/Verlet step on tiles: tile_lean_kernel in the compact or the
// explicit record format (tile_f32.cuh).
// Programmatic dependent launch: the kernel's CTAs may start (and prefetch
// their tile records) while the previous kernel on the stream drains; the
// kernel orders its state reads with griddepcontrol.wait.
template <typename P>
void launch_pdl(void (*k)(P), int grid, int block, size_t smem, cudaStream_t stream, const P &p) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k, p);
}

// RK4 stage `stage` (1-4) of a fp32 compact-tile engine on the lean kernel
// (tile_f32.cuh rk4_store), chained by programmatic dependent launch.
template <bool GROUPS>
void launch_rk4_lean(ss_engine *h, const Params<float> &p, int grid, int stage) {
    const bool two = h->lean_lanes == 2;
    void (*k)(Params<float>) = nullptr;
    if (h->tl.inline_kl || h->tl.dict_x0) {               // records with the staged X0 (REC 1 / 2)
        const bool i1 = h->tl.inline_kl;
        switch (stage) {
            case 1: k = i1 ? tile_lean_kernel<2, GROUPS, kInlineMinB, 1, false, 1>
                           : tile_lean_kernel<2, GROUPS, kInlineMinB, 1, false, 2>; break;
            case 2: k = i1 ? tile_lean_kernel<3, GROUPS, kInlineMinB, 1, false, 1>
                           : tile_lean_kernel<3, GROUPS, kInlineMinB, 1, false, 2>; break;
            case 3: k = i1 ? tile_lean_kernel<4, GROUPS, kInlineMinB, 1, false, 1>
                           : tile_lean_kernel<4, GROUPS, kInlineMinB, 1, false, 2>; break;
            default: k = i1 ? tile_lean_kernel<5, GROUPS, kInlineMinB, 1, false, 1>
                            : tile_lean_kernel<5, GROUPS, kInlineMinB, 1, false, 2>; break;
        }
        if (h->pdl) launch_pdl(k, grid, kTile, h->lean_smem, h->stream, p);
        else k<<<grid, kTile, h->lean_smem, h->stream>>>(p);
        return;
    }
    switch (stage) {
        case 1: k = two ? tile_lean_kernel<2, GROUPS, 6, 2> : tile_lean_kernel<2, GROUPS>; break;
        case 2: k = two ? tile_lean_kernel<3, GROUPS, 6, 2> : tile_lean_kernel<3, GROUPS>; break;
        case 3: k = two ? tile_lean_kernel<4, GROUPS, 6, 2> : tile_lean_kernel<4, GROUPS>; break;
        default: k = two ? tile_lean_kernel<5, GROUPS, 6, 2> : tile_lean_kernel<5, GROUPS>; break;
    }
    const int block = kTile * h->lean_lanes;
    if (h->pdl) launch_pdl(k, grid, block, h->lean_smem, h->stream, p);
    else k<<<grid, block, h->lean_smem, h->stream>>>(p);
}

template <bool GROUPS>
void launch_tile_f32(ss_engine *h, const Params<float> &p, int grid) {
    const bool euler = h->integrator == SS_EULER;
    if (h->tl.inline_kl) {                                 // general graphs: records streamed per incidence
        auto *ki = h->p2p_on ? (euler ? tile_lean_kernel<0, GROUPS, kInlineMinB, 1, true, 1>
                                      : tile_lean_kernel<1, GROUPS, kInlineMinB, 1, true, 1>)
                             : (euler ? tile_lean_kernel<0, GROUPS, kInlineMinB, 1, false, 1>
                                      : tile_lean_kernel<1, GROUPS, kInlineMinB, 1, false, 1>);
        if (h->pdl) launch_pdl(ki, grid, kTile, h->lean_smem, h->stream, p);
        else ki<<<grid, kTile, h->lean_smem, h->stream>>>(p);
        return;
    }
    if (h->tl.dict_x0) {                                   // (k, k*l0, group) dictionary, D from the staged X0
        auto *ki = h->p2p_on ? (euler ? tile_lean_kernel<0, GROUPS, kInlineMinB, 1, true, 2>
                                      : tile_lean_kernel<1, GROUPS, kInlineMinB, 1, true, 2>)
                             : (euler ? tile_lean_kernel<0, GROUPS, kInlineMinB, 1, false, 2>
                                      : tile_lean_kernel<1, GROUPS, kInlineMinB, 1, false, 2>);
        if (h->pdl) launch_pdl(ki, grid, kTile, h->lean_smem, h->stream, p);
        else ki<<<grid, kTile, h->lean_smem, h->stream>>>(p);
        return;
    }
    auto *k = h->integrator == SS_EULER ? tile_lean_kernel<0, GROUPS> : tile_lean_kernel<1, GROUPS>;
    if (h->lean_lanes == 2)
        k = h->integrator == SS_EULER ? tile_lean_kernel<0, GROUPS, 6, 2> : tile_lean_kernel<1, GROUPS, 6, 2>;
    else if (h->p2p_on)                                    // sharded: boundary tiles first
        k = h->integrator == SS_EULER ? tile_lean_kernel<0, GROUPS, 6, 1, true> : tile_lean_kernel<1, GROUPS, 6, 1, true>;
    const int block = kTile * h->lean_lanes;
    if (h->pdl) launch_pdl(k, grid, block, h->lean_smem, h->stream, p);      // tile_f32.cuh
    else k<<<grid, block, h->lean_smem, h->stream>>>(p);
}

// fp64 Euler/Verlet step on compact tiles: tile_f64_kernel (tile_f64.cuh).
template <bool GROUPS>
void launch_tile_f64(ss_engine *h, const Params<double> &p, int grid) {
    const bool euler = h->integrator == SS_EULER;
    void (*k)(Params<double>) = nullptr;
    if (h->tl.inline_kl) {                                 // general graphs: (k, l0) streamed per incidence
        // (UNROLL, MINB) = (2, 4), records software pipelined (tile_f64.cuh
        // fast_sum): 95.6 us on the 10M cube; (4, 3) 95.9, (2, 3) 110.8, (1, 4) 118.8
        k = euler ? tile_f64_kernel<0, GROUPS, 2, 4, true> : tile_f64_kernel<1, GROUPS, 2, 4, true>;
        if (h->pdl) launch_pdl(k, grid, kTile, h->f64_smem, h->stream, p);
        else k<<<grid, kTile, h->f64_smem, h->stream>>>(p);
        return;
    }
    switch (h->f64_variant) {
        case 1: k = euler ? tile_f64_kernel<0, GROUPS, 1, 4> : tile_f64_kernel<1, GROUPS, 1, 4>; break;
        case 2: k = euler ? tile_f64_kernel<0, GROUPS, 2, 3> : tile_f64_kernel<1, GROUPS, 2, 3>; break;
        case 3: k = euler ? tile_f64_kernel<0, GROUPS, 3, 3> : tile_f64_kernel<1, GROUPS, 3, 3>; break;
        case 4: k = euler ? tile_f64_kernel<0, GROUPS, 1, 5> : tile_f64_kernel<1, GROUPS, 1, 5>; break;
        case 5: k = euler ? tile_f64_kernel<0, GROUPS, 2, 5> : tile_f64_kernel<1, GROUPS, 2, 5>; break;
        default: k = euler ? tile_f64_kernel<0, GROUPS, 2, 4> : tile_f64_kernel<1, GROUPS, 2, 4>; break;
    }
    if (h->pdl) launch_pdl(k, grid, kTile, h->f64_smem, h->stream, p);
    else k<<<grid, kTile, h->f64_smem, h->stream>>>(p);
}

// RK4 stage `stage` (1-4) of a fp64 compact-tile engine on tile_f64_kernel
// (tile_f64.cuh f64_rk4_epilogue), chained by programmatic dependent launch.
template <bool GROUPS>
void launch_rk4_f64(ss_engine *h, const Params<double> &p, int grid, int stage) {
    void (*k)(Params<double>) = nullptr;
    const bool inl = h->tl.inline_kl;
    const bool v3 = !inl && h->f64_rk4_variant == 3;      // (3, 3): grids of a few waves
    switch (stage) {
        case 1: k = inl ? tile_f64_kernel<2, GROUPS, 2, 4, true> : v3 ? tile_f64_kernel<2, GROUPS, 3, 3>
                                                                      : tile_f64_kernel<2, GROUPS, 2, 4>; break;
        case 2: k = inl ? tile_f64_kernel<3, GROUPS, 2, 4, true> : v3 ? tile_f64_kernel<3, GROUPS, 3, 3>
                                                                      : tile_f64_kernel<3, GROUPS, 2, 4>; break;
        case 3: k = inl ? tile_f64_kernel<4, GROUPS, 2, 4, true> : v3 ? tile_f64_kernel<4, GROUPS, 3, 3>
                                                                      : tile_f64_kernel<4, GROUPS, 2, 4>; break;
        default: k = inl ? tile_f64_kernel<5, GROUPS, 2, 4, true> : v3 ? tile_f64_kernel<5, GROUPS, 3, 3>
                                                                       : tile_f64_kernel<5, GROUPS, 2, 4>; break;
    }
    if (h->pdl) launch_pdl(k, grid, kTile, h->f64_smem, h->stream, p);
    else k<<<grid, kTile, h->f64_smem, h->stream>>>(p);
}

__global__ void step_base_set(long long *base, long long n) { *base = n; }
__global__ void step_base_add(long long *base, long long count) { *base += count; }

// The identity of a batch for the graph cache: its launch parameters (the
// Params every substep starts from, which holds every pointer and scalar the
// kernels read), count, parity and the engine's kernel choices.
template <typename T>
std::vector<unsigned char> graph_key(const ss_engine *h, const Params<T> &p, int64_t count) {
    std::vector<unsigned char> k(sizeof(Params<T>) + 64, 0);
    std::memcpy(k.data(), &p, sizeof(Params<T>));
    int64_t extra[8] = {count, h->cur, h->integrator, (h->pdl ? 1 : 0) | (h->pdl_graph + 1) << 1, h->lean_lanes,
                        h->f64_variant, (int64_t)(intptr_t)h->scale, h->has_prev ? 1 : 0};
    std::memcpy(k.data() + sizeof(Params<T>), extra, sizeof extra);
    return k;
}

template <bool F32, int LAYOUT>
int launch_steps(ss_engine *h, int64_t count);

// Replay (or capture, on a key's second occurrence) the launch loop of a
// batch as a CUDA graph: the launch gap between substeps goes (mid-size
// scenes 1.5-2 us of ~8 us per substep, 0.7 us of 64 us on the 10M cube).
// Returns 1 if the batch was enqueued as a graph, 0 to launch it normally.
template <bool F32, int LAYOUT>
int try_graph(ss_engine *h, int64_t count, Params<typename Prec<F32>::T> p, int *rc_out) {
    using T = typename Prec<F32>::T;
    *rc_out = SS_OK;
    if (!h->use_graphs || count < 2 || h->nccl || h->p2p_on || (h->integrator == SS_VERLET && !h->has_prev))
        return 0;
    const auto key = graph_key<T>(h, p, count);
    auto *entry = [&]() -> ss_engine::GraphEntry * {
        for (auto &g : h->graphs)
            if (g.key == key) return &g;
        return nullptr;
    }();
    if (!entry) {
        bool seen = false;
        for (auto &k : h->graph_seen) seen = seen || k == key;
        if (!seen) {                                         // first occurrence: remember, launch normally
            if (h->graph_seen.size() >= 16) h->graph_seen.erase(h->graph_seen.begin());
            h->graph_seen.push_back(key);
            return 0;
        }
        if (!h->d_step_base) {
            int rc = h->alloc(&h->d_step_base, sizeof(long long));
            if (rc) { *rc_out = rc; return 1; }
        }
        // capture the loop with step numbers relative to the device base
        const int cur0 = h->cur;
        const bool prev0 = h->has_prev;
        const int64_t launches0 = h->launches, n0 = h->n;
        cudaGraph_t graph = nullptr;
        CK(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
        h->n = 0;                                            // (the loop numbers steps h->n + s + 1)
        h->graph_capturing = true;
        const bool pdl0 = h->pdl;
        if (h->pdl_graph >= 0) h->pdl = h->pdl_graph != 0;    // (replays may prefer the other choice)
        int rc = launch_steps<F32, LAYOUT>(h, count);
        h->pdl = pdl0;
        h->graph_capturing = false;
        h->n = n0;
        if (rc == SS_OK) step_base_add<<<1, 1, 0, h->stream>>>(h->d_step_base, (long long)count);
        const cudaError_t ec = cudaStreamEndCapture(h->stream, &graph);
        h->cur = cur0;                                       // (replayed below)
        h->has_prev = prev0;
        h->launches = launches0;
        if (rc) { *rc_out = rc; return 1; }
        if (ec != cudaSuccess || !graph) {
            cudaGetLastError();
            h->use_graphs = false;                           // capture unsupported here: launch normally from now on
            return 0;
        }
        cudaGraphExec_t exec = nullptr;
        const cudaError_t ei = cudaGraphInstantiate(&exec, graph, 0);
        cudaGraphDestroy(graph);
        if (ei != cudaSuccess) {
            cudaGetLastError();
            h->use_graphs = false;
            return 0;
        }
        if (h->graphs.size() >= 4) {                         // evict the least recently used
            auto victim = std::min_element(h->graphs.begin(), h->graphs.end(),
                                           [](const auto &a, const auto &b) { return a.last_use < b.last_use; });
            cudaGraphExecDestroy(victim->exec);
            h->graphs.erase(victim);
        }
        h->graphs.push_back({key, exec, 0});
        entry = &h->graphs.back();
    }
    entry->last_use = ++h->graph_clock;
    if (h->graph_base_n != h->n) step_base_set<<<1, 1, 0, h->stream>>>(h->d_step_base, (long long)h->n);
    CK(cudaGraphLaunch(entry->exec, h->stream));
    h->graph_base_n = h->n + count;
    const int stages = h->integrator == SS_RK4 ? 4 : 1;
    h->launches += count * stages;
    if (h->integrator != SS_RK4) h->cur ^= (int)(count & 1);
    if (h->integrator == SS_VERLET) h->has_prev = true;
    return 1;
}

template <bool F32, int LAYOUT>
int launch_steps(ss_engine *h, int64_t count) {
    using T = typename Prec<F32>::T;
    using T4 = typename Prec<F32>::T4;
    const int stages = h->integrator == SS_RK4 ? 4 : 1;
    const size_t G = h->groups.size();
    if (G && !h->graph_capturing) {                          // (a capture re-enters here: the table is uploaded)
        std::vector<double> tab;
        build_scales(h, count, stages, h->t, h->n, tab);
        int rc = upload_scales<T>(h, tab);
        if (rc) return rc;
    }
    const int grid = h->grid();
    const size_t smem = LAYOUT >= 3 ? h->smem_bytes : 0;
    Params<T> p = base_params<T>(h);
    const T *scale = reinterpret_cast<const T *>(h->scale);
    if (h->res_image && h->integrator != SS_RK4 && !h->nccl && !h->p2p_on && count >= 1) {
        // (every batch size, one step included: fp32 results must not depend on
        // how the steps are batched, and the resident kernel sums in its own order)
        // small scene: one CTA keeps the state on chip for the whole batch (resident.cuh)
        ResidentArgs a{};
        a.image = reinterpret_cast<const unsigned char *>(h->res_image);
        a.seg = h->res_segd;
        a.dict_bytes = h->res_dict_bytes;
        a.nd = (int)h->ND;
        a.pslots = h->res_pslots;
        a.cur0 = h->cur;
        a.count = count;
        a.step0 = h->n;
        a.bootstrap0 = (h->integrator == SS_VERLET && !h->has_prev) ? 1 : 0;
        a.G = (int)G;
        a.off_dict = h->res_off[0];
        a.off_grp = h->res_off[1];
        a.off_seg = h->res_off[2];
        p.X = reinterpret_cast<const T4 *>(h->X[0]);
        p.Xout = reinterpret_cast<T4 *>(h->X[1]);
        p.V = reinterpret_cast<T4 *>(h->V);
        p.Vout = reinterpret_cast<T4 *>(h->V);
        p.Xprev = reinterpret_cast<const T4 *>(h->X[h->cur ^ 1]);
        if (F32 && h->U) {
            p.Xprev = reinterpret_cast<const T4 *>(h->U);
            p.U = reinterpret_cast<T4 *>(h->U);
        }
        p.scale = G ? scale : nullptr;
        const bool euler = h->integrator == SS_EULER;
        auto *k = h->res_g == 8 ? (euler ? resident_kernel<F32, 0, 8> : resident_kernel<F32, 1, 8>)
                : h->res_g == 4 ? (euler ? resident_kernel<F32, 0, 4> : resident_kernel<F32, 1, 4>)
                : h->res_g == 2 ? (euler ? resident_kernel<F32, 0, 2> : resident_kernel<F32, 1, 2>)
                                : (euler ? resident_kernel<F32, 0, 1> : resident_kernel<F32, 1, 1>);
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3((unsigned)h->res_ctas);
        cfg.blockDim = dim3((unsigned)h->res_threads);
        cfg.dynamicSmemBytes = h->res_smem;
        cfg.stream = h->stream;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = (unsigned)h->res_ctas;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        CK(cudaLaunchKernelEx(&cfg, k, p, a));
        h->launches += 1;
        h->cur ^= (int)(count & 1);
        if (h->integrator == SS_VERLET) h->has_prev = true;
        return SS_OK;
    }
    if (h->integrator != SS_RK4 && !h->nccl && !h->p2p_on && count >= 1 && h->persist_max_grid >= grid) {
        // small scene: one cooperative launch steps the whole batch
        // (kernels.cuh persist_step_kernel / tile_f32.cuh persist_lean_kernel)
        PersistArgs<T> a{};
        a.Xb[0] = reinterpret_cast<T4 *>(h->X[0]);
        a.Xb[1] = reinterpret_cast<T4 *>(h->X[1]);
        a.cur0 = h->cur;
        a.count = count;
        a.step0 = h->n;
        a.bootstrap0 = (h->integrator == SS_VERLET && !h->has_prev) ? 1 : 0;
        a.G = (int)G;
        a.scale = G ? scale : nullptr;
        a.xprev_is_other = (h->integrator == SS_VERLET && !(F32 && h->U)) ? 1 : 0;
        p.V = reinterpret_cast<T4 *>(h->V);
        p.V0 = reinterpret_cast<T4 *>(h->V);
        p.Vout = reinterpret_cast<T4 *>(h->V);
        if (F32 && h->U) {
            p.Xprev = reinterpret_cast<const T4 *>(h->U);
            p.U = reinterpret_cast<T4 *>(h->U);
        }
        void *args[] = {&p, &a};
        const bool euler = h->integrator == SS_EULER;
        const void *fn = euler ? (const void *)persist_step_kernel<F32, 0, LAYOUT>
                               : (const void *)persist_step_kernel<F32, 1, LAYOUT>;
        size_t sm = smem;
        if constexpr (F32 && LAYOUT >= 3) {
            if (h->lean_smem) {
                constexpr bool GROUPS = LAYOUT == 3;
                fn = euler ? (const void *)persist_lean_kernel<0, GROUPS> : (const void *)persist_lean_kernel<1, GROUPS>;
                sm = h->lean_smem;
            }
        }
        CK(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(kBlock), args, sm, h->stream));
        h->launches += 1;
        h->cur ^= (int)(count & 1);
        if (h->integrator == SS_VERLET) h->has_prev = true;
        CK(cudaGetLastError());
        return SS_OK;
    }
    if (!h->graph_capturing) {
        int grc = SS_OK;
        if (try_graph<F32, LAYOUT>(h, count, p, &grc)) return grc;
    } else {
        p.step_base = h->d_step_base;                        // capturing: step numbers relative to the base
    }
    for (int64_t s = 0; s < count; ++s) {
        p.step = h->n + s + 1;
        if (h->p2p_on && h->integrator != SS_RK4) xchg_params(h, p);   // fused peer-memory exchange (kernels.cuh)
        T4 *Xc = reinterpret_cast<T4 *>(h->X[h->cur]);
        T4 *Xo = reinterpret_cast<T4 *>(h->X[h->cur ^ 1]);
        T4 *V = reinterpret_cast<T4 *>(h->V);
        if (h->integrator != SS_RK4) {
            p.scale = G ? scale + (size_t)s * G : nullptr;
            p.X = Xc;
            p.X0 = Xc;
            p.V = V;
            p.V0 = V;
            p.Xout = Xo;
            p.Vout = V;
            p.Xprev = Xo;
            if (F32 && h->U) {                       // increment-form Verlet: u read and written in place
                p.Xprev = reinterpret_cast<const T4 *>(h->U);
                p.U = reinterpret_cast<T4 *>(h->U);
            }
            p.bootstrap = (h->integrator == SS_VERLET && !h->has_prev) ? 1 : 0;
            if constexpr (F32 && LAYOUT >= 3) {
                if (h->lean_smem) {
                    constexpr bool GROUPS = LAYOUT == 3;
                    launch_tile_f32<GROUPS>(h, p, grid);
                    goto launched;
                }
            }
            if constexpr (!F32 && LAYOUT >= 3) {
                if (h->f64_smem) {
                    if (G) launch_tile_f64<true>(h, p, grid);
                    else launch_tile_f64<false>(h, p, grid);
                    goto launched;
                }
            }
            {
                auto *k = h->integrator == SS_EULER ? step_kernel<F32, 0, LAYOUT> : step_kernel<F32, 1, LAYOUT>;
                if (LAYOUT >= 3 && h->pdl) launch_pdl(k, grid, kBlock, smem, h->stream, p);
                else k<<<grid, kBlock, smem, h->stream>>>(p);
            }
        launched:
            h->launches += 1;
            h->cur ^= 1;
            if (h->integrator == SS_VERLET) h->has_prev = true;
            if (h->nccl) {                                   // boundary planes -> neighbours' halos
                int rc = halo_exchange_nccl<T4>(h);
                if (rc) return rc;
            }
        } else {
            T4 *XA = reinterpret_cast<T4 *>(h->XA), *XB = reinterpret_cast<T4 *>(h->XB);
            T4 *VS = reinterpret_cast<T4 *>(h->VS);
            p.X0 = Xc;
            p.V0 = V;
            p.SV = reinterpret_cast<T4 *>(h->SV);
            p.SA = reinterpret_cast<T4 *>(h->SA);
            // tiles: stages chained by programmatic dependent launch (the
            // kernel waits in stage_tile before its first state read)
            int stage = 0;
            auto rk4_launch = [&](void (*k)(Params<T>)) {
                ++stage;
                if constexpr (F32 && LAYOUT >= 3) {
                    if (h->lean_smem) {                      // fp32 compact tiles: the lean kernel
                        launch_rk4_lean<LAYOUT == 3>(h, p, grid, stage);
                        return;
                    }
                }
                if constexpr (!F32 && LAYOUT >= 3) {
                    if (h->f64_smem) {                       // fp64 compact tiles: tile_f64_kernel
                        if (G) launch_rk4_f64<true>(h, p, grid, stage);
                        else launch_rk4_f64<false>(h, p, grid, stage);
                        return;
                    }
                }
                if (LAYOUT >= 3 && h->pdl) launch_pdl(k, grid, kBlock, smem, h->stream, p);
                else k<<<grid, kBlock, smem, h->stream>>>(p);
            };
            // sharded (NCCL): every stage's trial positions cross to the
            // neighbours' halos before the next stage reads them (SURVEY
            // 8e: four exchanges per step); ss_step_group launches one
            // stage at a time (rk4_stage_only) and copies the planes itself
            const int only = h->rk4_stage_only;
            auto stage_at = [&](int st, void (*k)(Params<T>), T4 *x, T4 *v, T4 *xo, T4 *vo) -> int {
                if (only && only != st) {
                    ++stage;
                    return SS_OK;
                }
                p.scale = G ? scale + ((size_t)s * 4 + (st - 1)) * G : nullptr;
                p.X = x; p.V = v; p.Xout = xo; p.Vout = vo;
                if (h->p2p_on) xchg_params(h, p, st);      // fused: pushes into the neighbours' stage buffer
                rk4_launch(k);
                h->launches += 1;
                return h->nccl ? halo_exchange_nccl<T4>(h, xo) : SS_OK;
            };
            int rc = stage_at(1, rk4_kernel<F32, 1, LAYOUT>, Xc, V, XA, VS);
            if (!rc) rc = stage_at(2, rk4_kernel<F32, 2, LAYOUT>, XA, VS, XB, VS);
            if (!rc) rc = stage_at(3, rk4_kernel<F32, 3, LAYOUT>, XB, VS, XA, VS);
            if (!rc) rc = stage_at(4, rk4_kernel<F32, 4, LAYOUT>, XA, VS, Xc, V);
            if (rc) return rc;
        }
    }
    CK(cudaGetLastError());
    return SS_OK;
}

int dispatch_steps(ss_engine *h, int64_t count) {
    return with_layout(h, [&](auto L) -> int {
        return h->precision == SS_F32 ? launch_steps<true, decltype(L)::value>(h, count)
                                      : launch_steps<false, decltype(L)::value>(h, count);
    });
}

template <bool F32, int LY>
int set_tile_smem_ly(size_t bytes) {
    const int b = (int)bytes;
    CK(cudaFuncSetAttribute(step_kernel<F32, 0, LY>, cudaFuncAttributeMaxDynamicSharedMemorySize, b));
    CK(cudaFuncSetAttribute(step_kernel<F32, 1, LY>, cudaFuncAttributeMaxDynamicSharedMemorySize, b));
    CK(cudaFuncSetAttribute(rk4_kernel<F32, 1, LY>, cudaFuncAttributeMaxDynamicSharedMemorySize, b));
    CK(cudaFuncSetAttribute(rk4_kernel<F32, 2, LY>, cudaFuncAttributeMaxDynamicSharedMemorySize, b));
    CK(cudaFuncSetAttribute(rk4_kernel<F32, 3, LY>, cudaFuncAttributeMaxDynamicSharedMemorySize, b));
    CK(cudaFuncSetAttribute(rk4_kernel<F32, 4, LY>, cudaFuncAttributeMaxDynamicSharedMemorySize, b));
    CK(cudaFuncSetAttribute(forces_kernel<F32, LY>, cudaFuncAttributeMaxDynamicSharedMemorySize, b));
    return SS_OK;
}

template <bool F32>
int set_tile_smem(size_t bytes) {
    int rc = set_tile_smem_ly<F32, 3>(bytes);
    return rc ? rc : set_tile_smem_ly<F32, 4>(bytes);
}

int reset_divergence(ss_engine *h) {
    const long long none = LLONG_MAX;
    const int nonei = INT_MAX;
    CK(cudaMemcpyAsync(h->d_div_step, &none, sizeof none, cudaMemcpyHostToDevice, h->stream));
    CK(cudaMemcpyAsync(h->d_div_mass, &nonei, sizeof nonei, cudaMemcpyHostToDevice, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    return SS_OK;
}

// Programmatic dependent launch on or off, timed on this scene.  For grids
// of one to eight CTAs per SM the next substep's early CTAs can pile onto a
// few SMs and cost more than the overlap gains, and where that happens
// depends on the scene (178-686 tiles, 6-17%).  PDL changes no
// bit, so the engine times a few substeps of each choice on its own buffers
// and keeps the faster (by at least 3%); the state, counters and step
// number are restored afterwards.  SS_PDL fixes the choice, SS_AUTOTUNE=0
// keeps the static one.
int autotune_pdl(ss_engine *h) {
    if (getenv("SS_PDL")) return SS_OK;
    if (const char *e = getenv("SS_AUTOTUNE"))
        if (atoi(e) == 0) return SS_OK;
    if (h->layout != SS_LAYOUT_TILE || h->res_image || !(h->lean_smem || h->f64_smem)) return SS_OK;
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->device));
    const int64_t tiles = h->tl.n_tiles;
    if (tiles < sms || tiles > 8 * (int64_t)sms) return SS_OK;
    const size_t vb = (size_t)h->ND * (h->precision == SS_F32 ? sizeof(float4) : sizeof(double4));
    void *live[4] = {h->X[0], h->X[1], h->V, h->U};
    void *keep[4] = {nullptr, nullptr, nullptr, nullptr};
    int rc = SS_OK;
    for (int i = 0; i < 4 && rc == SS_OK; ++i) {
        if (!live[i]) continue;
        if (cudaMalloc(&keep[i], vb) != cudaSuccess) {
            cudaGetLastError();
            keep[i] = nullptr;
            rc = -1;                                        // no room to snapshot: keep the static choice
            break;
        }
        if (cudaMemcpyAsync(keep[i], live[i], vb, cudaMemcpyDeviceToDevice, h->stream) != cudaSuccess) rc = -1;
    }
    unsigned long long deg0 = 0;
    if (rc == SS_OK && cudaMemcpy(&deg0, h->d_degenerate, sizeof deg0, cudaMemcpyDeviceToHost) != cudaSuccess) rc = -1;
    const int64_t n0 = h->n, launches0 = h->launches;
    const double t0 = h->t;
    const int cur0 = h->cur;
    const bool prev0 = h->has_prev, graphs0 = h->use_graphs, pdl0 = h->pdl;
    if (rc == SS_OK) {
        cudaEvent_t ev[2];
        CK(cudaEventCreate(&ev[0]));
        CK(cudaEventCreate(&ev[1]));
        // ms[mode][choice]: mode 0 launches one by one, mode 1 graph replays
        // (a batch shape's second occurrence is captured, later ones replay)
        float ms[2][2] = {{0.f, 0.f}, {0.f, 0.f}};
        for (int mode = 0; mode < 2 && rc == SS_OK; ++mode) {
            h->use_graphs = mode == 1;
            for (int c = 0; c < 2 && rc == SS_OK; ++c) {
                const bool pdl = c == 0 ? pdl0 : !pdl0;
                h->pdl = pdl;
                h->pdl_graph = pdl ? 1 : 0;
                for (int w = 0; w < 3 && rc == SS_OK; ++w) rc = dispatch_steps(h, 32);   // even counts: the parity returns
                if (rc == SS_OK) CK(cudaEventRecord(ev[0], h->stream));
                for (int w = 0; w < 2 && rc == SS_OK; ++w) rc = dispatch_steps(h, 32);
                if (rc == SS_OK) CK(cudaEventRecord(ev[1], h->stream));
                if (rc == SS_OK) {
                    CK(cudaEventSynchronize(ev[1]));
                    CK(cudaEventElapsedTime(&ms[mode][c], ev[0], ev[1]));
                }
            }
        }
        cudaEventDestroy(ev[0]);
        cudaEventDestroy(ev[1]);
        h->pdl = (rc == SS_OK && ms[0][1] < 0.97f * ms[0][0]) ? !pdl0 : pdl0;
        h->pdl_graph = ((rc == SS_OK && ms[1][1] < 0.97f * ms[1][0]) ? !pdl0 : pdl0) ? 1 : 0;
        // the tuning batches' graphs go: they captured this state's buffers
        for (auto &g : h->graphs)
            if (g.exec) cudaGraphExecDestroy(g.exec);
        h->graphs.clear();
        h->graph_seen.clear();
        h->graph_base_n = -1;
    }
    // restore the state the engine was created with
    for (int i = 0; i < 4; ++i)
        if (keep[i]) cudaMemcpyAsync(live[i], keep[i], vb, cudaMemcpyDeviceToDevice, h->stream);
    cudaMemcpyAsync(h->d_degenerate, &deg0, sizeof deg0, cudaMemcpyHostToDevice, h->stream);
    CK(cudaStreamSynchronize(h->stream));
    for (void *k : keep)
        if (k) cudaFree(k);
    h->n = n0;
    h->t = t0;
    h->cur = cur0;
    h->has_prev = prev0;
    h->launches = launches0;
    h->use_graphs = graphs0;
    if (rc != SS_OK && rc != -1) return rc;
    return reset_divergence(h);
}

// After an enqueued batch: read the divergence record, fix up n/t/cur.
int finish_batch(ss_engine *h, int64_t count, int64_t n0, int cur0, ss_step_result *res) {
    CK(cudaStreamSynchronize(h->stream));
    if (h->p2p_on) {
        int err = 0;
        CK(cudaMemcpy(&err, &reinterpret_cast<MailboxHead *>(h->mailbox)->error, sizeof err, cudaMemcpyDeviceToHost));
        if (err) return ss::fail(SS_ECUDA, "halo exchange: a neighbour did not publish its boundary planes within 20 s");
    }
    long long dstep = LLONG_MAX;
    int dmass = INT_MAX;
    CK(cudaMemcpy(&dstep, h->d_div_step, sizeof dstep, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&dmass, h->d_div_mass, sizeof dmass, cudaMemcpyDeviceToHost));
    int64_t done = count;
    if (dstep != LLONG_MAX) done = (int64_t)dstep - n0;
    h->n = n0 + done;
    h->t = (double)h->n * h->dt;
    if (h->integrator != SS_RK4) h->cur = cur0 ^ (int)(done & 1);
    if (res) {
        res->steps_done = done;
        res->n = h->n;
        res->t = h->t;
        res->diverged_mass = dstep != LLONG_MAX ? dmass : -1;
        res->diverged_step = dstep != LLONG_MAX ? (int64_t)dstep : -1;
    }
    if (dstep != LLONG_MAX) {
        int rc = reset_divergence(h);
        if (rc) return rc;
        return ss::fail(SS_EDIVERGED,
                        "simulation diverged at step %lld: mass %d has a non-finite position or "
                        "velocity (try a smaller dt)",
                        dstep, dmass);
    }
    return SS_OK;
}

template <typename T>
int up_vec(ss_engine *h, void **dst, const std::vector<T> &src) {
    int r = h->alloc(dst, src.size() * sizeof(T));
    if (r) return r;
    return upload(h, *dst, src.data(), src.size() * sizeof(T));
}

// Record image of the cluster-resident kernel (resident.cuh) for scenes of at
// most kResidentMaxCtas tiles whose per-CTA image fits shared memory; every
// mass's incidences in ascending spring id (the reference's summation order),
// springs deduplicated into a dictionary, partners renumbered into the CTA's
// own slots and its halo.  SS_RESIDENT=0 disables it.
template <bool F32>
int setup_resident(ss_engine *h, const ss_scene_desc *d) {
    using T4 = typename Prec<F32>::T4;
    const int64_t ND = h->ND, S = h->S;
    const int64_t n_ctas = (ND + kResidentSlots - 1) / kResidentSlots;
    if (h->integrator == SS_RK4 || n_ctas > kResidentMaxCtas || (F32 && !h->rx0) ||
        h->groups.size() > (size_t)kResidentMaxGroups)
        return SS_OK;
    // clusters of up to kResidentMaxCtas CTAs, one tile each (measured
    // faster than a launch per step: fp32 beam 4.80 -> 3.67 us, fp64 with one
    // lane per mass 6.73 -> 6.39 us, 64 fp64 walkers 5.85 -> 4.89 us)
    int max_ctas = kResidentMaxCtas;
    if (const char *e = getenv("SS_RESIDENT")) max_ctas = std::min(max_ctas, atoi(e));  // 0: off
    if (n_ctas > max_ctas) return SS_OK;
    std::vector<int64_t> dev(h->N);
    for (int64_t i = 0; i < h->N; ++i)
        dev[i] = h->tl.new_of.empty() || h->orig_of.empty() ? i : (int64_t)h->tl.new_of[i];
    std::vector<uint32_t> row((size_t)ND + 1, 0);
    for (int64_t s = 0; s < S; ++s) {
        row[dev[d->si[s]] + 1]++;
        row[dev[d->sj[s]] + 1]++;
    }
    for (int64_t i = 0; i < ND; ++i) row[i + 1] += row[i];
    const int64_t nnz = row[ND];
    std::vector<uint32_t> inc((size_t)nnz), fill(row.begin(), row.end() - 1);
    std::vector<int32_t> partner((size_t)nnz);
    const bool has_g = d->group && !h->groups.empty();
    // dictionary: fp64 (k, l0, group) bit patterns; fp32 (k, k*l0, D, group) as tiles_f32.cpp
    std::map<std::array<uint64_t, 4>, uint32_t> dict;
    std::vector<std::array<uint64_t, 4>> keys;
    auto key_of = [&](int64_t s, int64_t me, int64_t other) {
        std::array<uint64_t, 4> k{};
        const int64_t g = has_g ? d->group[s] : -1;
        if constexpr (F32) {
            const float kf = (float)d->k[s], kl = (float)(d->k[s] * d->l0[s]);
            float D[3];
            for (int c = 0; c < 3; ++c) D[c] = (float)(d->x[3 * other + c] - d->x[3 * me + c]);
            uint32_t b[5];
            std::memcpy(&b[0], &kf, 4);
            std::memcpy(&b[1], &kl, 4);
            std::memcpy(&b[2], D, 12);
            k[0] = ((uint64_t)b[0] << 32) | b[1];
            k[1] = ((uint64_t)b[2] << 32) | b[3];
            k[2] = b[4];
        } else {
            std::memcpy(&k[0], &d->k[s], 8);
            std::memcpy(&k[1], &d->l0[s], 8);
        }
        k[3] = (uint64_t)(g + 1);
        return k;
    };
    for (int64_t s = 0; s < S; ++s) {
        const int64_t a = d->si[s], b = d->sj[s];
        for (int end = 0; end < 2; ++end) {
            const int64_t me = end ? b : a, other = end ? a : b;
            const auto key = key_of(s, me, other);
            auto it = dict.find(key);
            uint32_t di;
            if (it == dict.end()) {
                di = (uint32_t)keys.size();
                if (di >= (1u << 19)) return SS_OK;                 // too many distinct springs: not resident
                dict.emplace(key, di);
                keys.push_back(key);
            } else {
                di = it->second;
            }
            const uint32_t owner = me < other ? 0x1000u : 0u;      // degenerate springs counted at the lower id
            const int64_t q = fill[dev[me]]++;
            inc[q] = owner | (di << 13);
            partner[q] = (int32_t)dev[other];
        }
    }
    // per CTA: halo list (partners owned by other CTAs) and local partner slots
    std::vector<std::vector<uint32_t>> halo((size_t)n_ctas);
    size_t max_halo = 0;
    for (int64_t r = 0; r < n_ctas; ++r) {
        const int64_t lo = r * kResidentSlots, hi = std::min<int64_t>(ND, lo + kResidentSlots);
        std::vector<uint32_t> &hl = halo[r];
        for (uint32_t q = row[lo]; q < row[hi]; ++q)
            if (partner[q] < lo || partner[q] >= hi) hl.push_back((uint32_t)partner[q]);
        std::sort(hl.begin(), hl.end());
        hl.erase(std::unique(hl.begin(), hl.end()), hl.end());
        for (uint32_t q = row[lo]; q < row[hi]; ++q) {
            const int64_t o = partner[q];
            const uint32_t local = (o >= lo && o < hi)
                                       ? (uint32_t)(o - lo)
                                       : (uint32_t)(kResidentSlots +
                                                    (std::lower_bound(hl.begin(), hl.end(), (uint32_t)o) - hl.begin()));
            inc[q] |= local;
        }
        max_halo = std::max(max_halo, hl.size());
    }
    const int64_t nd = (int64_t)keys.size();
    auto al16 = [](size_t v) { return (v + 15) & ~(size_t)15; };
    const size_t pslots = (size_t)((kResidentSlots + max_halo + 31) / 32 * 32);
    if (pslots > 4096) return SS_OK;                               // 12-bit partner slots
    const size_t dict_bytes = al16((size_t)nd * (F32 ? 32 : 16));
    const size_t grp_bytes = F32 ? 0 : al16((size_t)nd * 4);
    std::vector<size_t> seg((size_t)n_ctas + 1);
    seg[0] = dict_bytes + grp_bytes;
    size_t max_seg = 0;
    for (int64_t r = 0; r < n_ctas; ++r) {
        const int64_t lo = r * kResidentSlots, hi = std::min<int64_t>(ND, lo + kResidentSlots);
        const size_t bytes = 16 + 260 * 4 + ((halo[r].size() + 3) & ~(size_t)3) * 4 + al16((size_t)(row[hi] - row[lo]) * 4);
        seg[r + 1] = seg[r] + al16(bytes);
        max_seg = std::max(max_seg, al16(bytes));
    }
    const size_t off_dict = 2 * pslots * sizeof(T4);
    const size_t off_seg = off_dict + dict_bytes + grp_bytes;
    const size_t smem = off_seg + max_seg;
    int dev_max = 0;
    CK(cudaDeviceGetAttribute(&dev_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, h->device));
    if (smem + 2048 > (size_t)dev_max) return SS_OK;                // does not fit one SM (+ static smem)
    std::vector<unsigned char> img(seg[n_ctas], 0);
    for (int64_t q = 0; q < nd; ++q) {
        const auto &k = keys[q];
        unsigned char *e = img.data() + (size_t)q * (F32 ? 32 : 16);
        const int32_t g = (int32_t)((int64_t)k[3] - 1);
        if constexpr (F32) {
            const uint32_t b[6] = {(uint32_t)(k[0] >> 32), (uint32_t)k[0], (uint32_t)(k[1] >> 32), (uint32_t)k[1],
                                   (uint32_t)k[2], (uint32_t)g};
            std::memcpy(e, b, 24);                                  // k, k*l0, Dx, Dy | Dz, group, 0, 0
        } else {
            std::memcpy(e, &k[0], 8);
            std::memcpy(e + 8, &k[1], 8);
            std::memcpy(img.data() + dict_bytes + (size_t)q * 4, &g, 4);
        }
    }
    for (int64_t r = 0; r < n_ctas; ++r) {                         // header, rows, halo, incidences
        const int64_t lo = r * kResidentSlots, hi = std::min<int64_t>(ND, lo + kResidentSlots);
        uint32_t *w = reinterpret_cast<uint32_t *>(img.data() + seg[r]);
        w[0] = (uint32_t)halo[r].size();
        uint32_t *rw = w + 4;
        for (int64_t i = 0; i <= kResidentSlots; ++i) rw[i] = row[std::min(lo + i, hi)] - row[lo];
        uint32_t *hl = rw + 260;
        std::copy(halo[r].begin(), halo[r].end(), hl);
        uint32_t *iw = hl + ((halo[r].size() + 3) & ~(size_t)3);
        std::memcpy(iw, inc.data() + row[lo], (size_t)(row[hi] - row[lo]) * 4);
    }
    int rc = h->alloc(&h->res_image, img.size());
    if (rc || (rc = upload(h, h->res_image, img.data(), img.size()))) return rc;
    {
        std::vector<unsigned> sg(seg.begin(), seg.end());
        if ((rc = up_vec(h, reinterpret_cast<void **>(&h->res_segd), sg))) return rc;
    }
    h->res_dict_bytes = (unsigned)(dict_bytes + grp_bytes);
    h->res_off[0] = (unsigned)off_dict;
    h->res_off[1] = (unsigned)(off_dict + dict_bytes);
    h->res_off[2] = (unsigned)off_seg;
    h->res_pslots = (int)pslots;
    h->res_smem = smem;
    h->res_ctas = (int)n_ctas;
    // lanes per mass slot; a lone CTA gets threads only up to its last real mass
    int64_t used = kResidentSlots;
    if (n_ctas == 1) {
        used = 0;
        for (int64_t i = 0; i < ND; ++i)
            if (h->src_of(i) >= 0) used = i + 1;
    }
    // lanes per mass.  fp64 adds in list order, where lanes cost more in
    // shuffles than they save: one lane per mass, four incidences in flight
    // through the branch-free IEEE sequences (crawler 2.50 -> 2.14 us, 12
    // crawlers 5.72 -> 2.68, the 40x4x4 beam as a cluster 5.08 against 6.71
    // with launches).  fp32: 8 lanes with a fixed-order tree for scenes of
    // <= 128 masses (crawler 1.03 us against 1.53 with one lane), else two
    // lanes (64 crawlers 2.66 us against 2.90 with one lane and four partial
    // sums, the beam 3.36 against 3.43, the 9^3 cube 3.52 against 3.48;
    // 4 lanes: 3.68, 3.67, 4.47).  fp64 stays at one lane: a group's ordered
    // shuffle-and-add rounds cost more than they save (beam 5.07 us with one
    // lane, 13.5 with two, 10.8 with four; tools/resident_g_probe.py)
    h->res_g = F32 ? (used * 8 <= 1024 ? 8 : 2) : 1;
    if (const char *e = getenv("SS_RESIDENT_G")) {                 // A/B: 1, 2, 4 or 8
        const int g = atoi(e);
        if ((g == 1 || g == 2 || g == 4 || g == 8) && used * g <= 1024) h->res_g = g;
    }
    h->res_threads = (int)std::max<int64_t>(32, (used * h->res_g + 31) / 32 * 32);
    for (const void *fn : {(const void *)resident_kernel<F32, 0, 4>, (const void *)resident_kernel<F32, 1, 4>,
                           (const void *)resident_kernel<F32, 0, 8>, (const void *)resident_kernel<F32, 1, 8>,
                           (const void *)resident_kernel<F32, 0, 2>, (const void *)resident_kernel<F32, 1, 2>,
                           (const void *)resident_kernel<F32, 0, 1>, (const void *)resident_kernel<F32, 1, 1>}) {
        // per-function attributes are shared by every engine in the process:
        // grant the device maximum, never this engine's size
        cudaFuncAttributes fa{};
        CK(cudaFuncGetAttributes(&fa, fn));
        CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, dev_max - (int)fa.sharedSizeBytes));
        CK(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    }
    if (n_ctas > 1) {                                               // can the cluster be scheduled at all?
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3((unsigned)n_ctas);
        cfg.blockDim = dim3((unsigned)h->res_threads);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = (unsigned)n_ctas;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int clusters = 0;
        const bool e0 = h->integrator == SS_EULER;
        const void *fn = h->res_g == 1 ? (e0 ? (const void *)resident_kernel<F32, 0, 1> : (const void *)resident_kernel<F32, 1, 1>)
                       : h->res_g == 2 ? (e0 ? (const void *)resident_kernel<F32, 0, 2> : (const void *)resident_kernel<F32, 1, 2>)
                                       : (e0 ? (const void *)resident_kernel<F32, 0, 4> : (const void *)resident_kernel<F32, 1, 4>);
        if (cudaOccupancyMaxActiveClusters(&clusters, fn, &cfg) != cudaSuccess || clusters < 1) {
            cudaGetLastError();
            h->res_image = nullptr;                                  // (freed with the engine)
        }
    }
    return SS_OK;
}

// The tiled layout of a scene: masses in spatial bricks first; where that
// gives tiles whose halo does not fit shared memory (dev_smem bytes), or
// whose halo is several times the tile (instances of a batch stacked at the
// same place: a brick holds the same mass of many robots, whose partners are
// all elsewhere), the caller's order, which keeps each instance's masses
// together -- the order with the smaller halo wins.
int choose_tiles(const ss_scene_desc *d, bool f32, int64_t dev_smem, TileLayout &out) {
    const size_t vec = f32 ? sizeof(float4) : sizeof(double4);
    TileLayout best;
    bool have = false;
    int rc = SS_OK;
    for (int order = 1; order >= 0; --order) {
        TileInput ti{d->n_masses, d->n_springs, d->si, d->sj, d->x, d->k, d->l0,
                     (d->group && d->n_groups) ? d->group : nullptr, f32, order};
        TileLayout cand;
        rc = build_tiles(ti, cand);
        if (rc != SS_OK) continue;
        const size_t need = 128 + ((cand.max_tile_smem + 127u) & ~127u) + (size_t)(kTile + cand.max_halo) * vec;
        if ((int64_t)need > dev_smem) {
            rc = ss::fail(SS_EINVAL, "tile needs %zu B of shared memory (> %lld)", need, (long long)dev_smem);
            continue;
        }
        if (!have || cand.halo_ratio < best.halo_ratio) {
            best = std::move(cand);
            have = true;
        }
        if (best.halo_ratio <= 3.0) break;                     // bricks did their job (lattices: 1.2-2.6)
    }
    if (!have) return rc;
    out = std::move(best);
    return SS_OK;
}

template <bool F32>
int create_impl(ss_engine *h, const ss_scene_desc *d, int want_layout) {
    using T = typename Prec<F32>::T;
    using T4 = typename Prec<F32>::T4;
    const int64_t N = h->N, S = h->S;
    int rc;
    // ---- topology first: it may renumber the masses
    int layout = want_layout;
    if (layout == SS_LAYOUT_AUTO || layout == SS_LAYOUT_TILE) {
        int dev_smem = 0;
        CK(cudaDeviceGetAttribute(&dev_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, h->device));
        rc = choose_tiles(d, F32, dev_smem, h->tl);
        if (rc == SS_OK) {
            layout = SS_LAYOUT_TILE;
        } else if (want_layout == SS_LAYOUT_TILE) {
            return rc;
        } else {
            layout = SS_LAYOUT_CSR;
            h->tl = TileLayout{};
        }
    }
    h->layout = layout;
    h->ND = N;
    if (layout == SS_LAYOUT_TILE) {
        h->orig_of = h->tl.orig_of;        // padded slot order
        h->ND = (int64_t)h->orig_of.size();
    }
    const int64_t ND = h->ND;
    if (!h->orig_of.empty()) {
        void *p;
        if ((rc = up_vec(h, &p, h->orig_of))) return rc;
        h->d_orig_of = reinterpret_cast<int *>(p);
    }
    // ---- fp32 base positions (device order)
    if (F32) {
        // P = X0 snapped to a power-of-two grid q with |P| <= 2^22 q: every
        // difference P_o - P_m (and P - tile anchor) is exact in fp32, and
        // r = x - P keeps the residual plus the motion.
        double amax = 1.0;
        for (int64_t i = 0; i < 3 * N; ++i) amax = std::max(amax, std::fabs(d->x[i]));
        const double q = std::ldexp(1.0, (int)std::ceil(std::log2(amax)) - 22);
        h->base.assign((size_t)ND * 4, 0.f);
        for (int64_t i = 0; i < ND; ++i) {
            const int64_t s = h->src_of(i);
            if (s < 0) continue;
            for (int c = 0; c < 3; ++c) h->base[4 * i + c] = (float)(std::nearbyint(d->x[3 * s + c] / q) * q);
        }
        if ((rc = h->alloc(&h->P, (size_t)ND * sizeof(T4)))) return rc;
        if ((rc = upload(h, h->P, h->base.data(), (size_t)ND * sizeof(T4)))) return rc;
        if (layout == SS_LAYOUT_TILE) {             // r = x - X0 with the records' rest vectors
            h->rx0 = true;
            h->x0.assign((size_t)ND * 3, 0.0);
            for (int64_t i = 0; i < ND; ++i) {
                const int64_t s = h->src_of(i);
                if (s < 0) continue;
                for (int c = 0; c < 3; ++c) h->x0[3 * i + c] = d->x[3 * s + c];
            }
        }
    }
    for (int b = 0; b < 2; ++b)
        if ((rc = h->alloc(&h->X[b], (size_t)ND * sizeof(T4)))) return rc;
    if ((rc = h->alloc(&h->V, (size_t)ND * sizeof(T4)))) return rc;
    if ((rc = h->alloc(&h->F, (size_t)ND * sizeof(T4)))) return rc;
    if (F32 && h->integrator == SS_VERLET) {
        if ((rc = h->alloc(&h->U, (size_t)ND * sizeof(T4)))) return rc;
        CK(cudaMemsetAsync(h->U, 0, (size_t)ND * sizeof(T4), h->stream));
    }
    if (h->integrator == SS_RK4) {
        // XA and XB in one allocation: a sharded RK4 engine exports both
        // stage buffers to its neighbours under one IPC handle
        if ((rc = h->alloc(&h->XA, 2 * (size_t)ND * sizeof(T4)))) return rc;
        h->XB = static_cast<char *>(h->XA) + (size_t)ND * sizeof(T4);
        for (void **b : {&h->VS, &h->SV, &h->SA})
            if ((rc = h->alloc(b, (size_t)ND * sizeof(T4)))) return rc;
    }
    {
        std::vector<T4> tmp((size_t)ND);
        pack_positions<T, T4>(h, d->x, tmp.data());
        if ((rc = upload(h, h->X[0], tmp.data(), (size_t)ND * sizeof(T4)))) return rc;
        if ((rc = upload(h, h->X[1], tmp.data(), (size_t)ND * sizeof(T4)))) return rc;
        pack_vec<T, T4>(h, d->v, tmp.data());
        if ((rc = upload(h, h->V, tmp.data(), (size_t)ND * sizeof(T4)))) return rc;
        if (d->f_ext) {
            pack_vec<T, T4>(h, d->f_ext, tmp.data());
            for (int64_t i = 0; i < 3 * N && !h->has_fext; ++i) h->has_fext = d->f_ext[i] != 0.0;
        } else {
            std::memset(tmp.data(), 0, (size_t)ND * sizeof(T4));
        }
        if ((rc = upload(h, h->F, tmp.data(), (size_t)ND * sizeof(T4)))) return rc;
    }
    const bool has_g = d->group && !h->groups.empty();
    if (layout == SS_LAYOUT_TILE) {
        const TileLayout &L = h->tl;
        void *p;
        if ((rc = up_vec(h, &p, L.blob))) return rc;
        h->d_blob = reinterpret_cast<unsigned char *>(p);
        std::vector<unsigned long long> off(L.off.begin(), L.off.end());
        if ((rc = up_vec(h, &p, off))) return rc;
        h->d_toff = reinterpret_cast<unsigned long long *>(p);
        if ((rc = up_vec(h, &p, L.split))) return rc;
        h->d_tsplit = reinterpret_cast<unsigned int *>(p);
        if (F32 && L.dict_x0) {                   // rest vectors formed from X0 on the device
            if ((rc = h->alloc(&h->d_x0dev, h->x0.size() * sizeof(double)))) return rc;
            if ((rc = upload(h, h->d_x0dev, h->x0.data(), h->x0.size() * sizeof(double)))) return rc;
        }
        if (L.inline_kl) {                        // general-graph format: records streamed, not staged
            if (F32) {
                if ((rc = up_vec(h, &p, L.kd_inline))) return rc;
                h->d_kd_inline = reinterpret_cast<float2 *>(p);
                if ((rc = h->alloc(&h->d_x0dev, h->x0.size() * sizeof(double)))) return rc;
                if ((rc = upload(h, h->d_x0dev, h->x0.data(), h->x0.size() * sizeof(double)))) return rc;
            } else {
                if ((rc = up_vec(h, &p, L.kl_inline))) return rc;
                h->d_kl_inline = reinterpret_cast<double2 *>(p);
            }
            if (!L.g_inline.empty()) {
                if ((rc = up_vec(h, &p, L.g_inline))) return rc;
                h->d_g_inline = reinterpret_cast<int8_t *>(p);
            }
            std::vector<unsigned long long> ko(L.kl_off.begin(), L.kl_off.end());
            if ((rc = up_vec(h, &p, ko))) return rc;
            h->d_kl_off = reinterpret_cast<unsigned long long *>(p);
        }
        h->blob_smem = (L.max_tile_smem + 127u) & ~127u;
        h->max_halo = L.max_halo;
        h->smem_bytes = 128 + h->blob_smem + (size_t)(kTile + L.max_halo) * sizeof(T4);   // one staged vector per mass
        int dev_max = 0;
        CK(cudaDeviceGetAttribute(&dev_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, h->device));
        if ((int64_t)h->smem_bytes > dev_max)
            return ss::fail(SS_EINVAL, "tile needs %zu B of shared memory (> %d)", h->smem_bytes, dev_max);
        // the attribute is a per-function permission shared by every engine in
        // the process: grant the device maximum, never a per-engine size
        if ((rc = set_tile_smem<F32>((size_t)dev_max))) return rc;
        if (const char *e = getenv("SS_PDL")) h->pdl = atoi(e) != 0;
        if (const char *e = getenv("SS_GRAPH")) h->use_graphs = atoi(e) != 0;
        if constexpr (F32) {
            // fp32 Euler/Verlet on compact tiles: tile_lean_kernel (tile_f32.cuh)
            // unless SS_KERNEL=step1 asks for kernels.cuh's step_kernel; the
            // explicit format and RK4 use the kernels.cuh kernels.
            const char *kenv = getenv("SS_KERNEL");
            const std::string kname = kenv ? kenv : "lean";
            if (kname != "step1" && !L.has_self && L.compact &&
                (int64_t)h->smem_bytes <= dev_max) {
                h->lean_smem = h->smem_bytes;
                if (L.inline_kl || L.dict_x0) h->lean_smem += (size_t)(kTile + L.max_halo) * 3 * sizeof(double);   // staged X0
                // scenes with few tiles (at most 3 per SM) use two lanes per mass:
                // 512-thread CTAs, twice the warps for the same tiles
                int sms = 0;
                CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->device));
                h->lean_lanes = L.n_tiles <= 3 * (int64_t)sms && !L.inline_kl && !L.dict_x0 ? 2 : 1;
                if (const char *e = getenv("SS_LEAN_LANES")) h->lean_lanes = atoi(e) == 2 ? 2 : 1;
                if (h->lean_lanes == 2) {
                    h->lean_smem += (size_t)kTile * sizeof(float4);        // lane 1's partial sums
                    if ((int64_t)h->lean_smem > dev_max) {
                        h->lean_lanes = 1;
                        h->lean_smem = h->smem_bytes;
                    }
                }
                const int b = dev_max;
                for (auto *kk : {tile_lean_kernel<0, false>, tile_lean_kernel<1, false>, tile_lean_kernel<0, true>,
                                 tile_lean_kernel<1, true>, tile_lean_kernel<0, false, 6, 2>,
                                 tile_lean_kernel<1, false, 6, 2>, tile_lean_kernel<0, true, 6, 2>,
                                 tile_lean_kernel<1, true, 6, 2>, tile_lean_kernel<0, false, 6, 1, true>,
                                 tile_lean_kernel<1, false, 6, 1, true>, tile_lean_kernel<0, true, 6, 1, true>,
                                 tile_lean_kernel<1, true, 6, 1, true>, tile_lean_kernel<2, false>,
                                 tile_lean_kernel<3, false>, tile_lean_kernel<4, false>, tile_lean_kernel<5, false>,
                                 tile_lean_kernel<2, true>, tile_lean_kernel<3, true>, tile_lean_kernel<4, true>,
                                 tile_lean_kernel<5, true>, tile_lean_kernel<2, false, 6, 2>,
                                 tile_lean_kernel<3, false, 6, 2>, tile_lean_kernel<4, false, 6, 2>,
                                 tile_lean_kernel<5, false, 6, 2>, tile_lean_kernel<2, true, 6, 2>,
                                 tile_lean_kernel<3, true, 6, 2>, tile_lean_kernel<4, true, 6, 2>,
                                 tile_lean_kernel<5, true, 6, 2>, tile_lean_kernel<0, false, kInlineMinB, 1, false, true>,
                                 tile_lean_kernel<1, false, kInlineMinB, 1, false, true>, tile_lean_kernel<0, true, kInlineMinB, 1, false, true>,
                                 tile_lean_kernel<1, true, kInlineMinB, 1, false, true>, tile_lean_kernel<0, false, kInlineMinB, 1, true, true>,
                                 tile_lean_kernel<1, false, kInlineMinB, 1, true, true>, tile_lean_kernel<0, true, kInlineMinB, 1, true, true>,
                                 tile_lean_kernel<1, true, kInlineMinB, 1, true, true>, tile_lean_kernel<2, false, kInlineMinB, 1, false, true>,
                                 tile_lean_kernel<3, false, kInlineMinB, 1, false, true>, tile_lean_kernel<4, false, kInlineMinB, 1, false, true>,
                                 tile_lean_kernel<5, false, kInlineMinB, 1, false, true>, tile_lean_kernel<2, true, kInlineMinB, 1, false, true>,
                                 tile_lean_kernel<3, true, kInlineMinB, 1, false, true>, tile_lean_kernel<4, true, kInlineMinB, 1, false, true>,
                                 tile_lean_kernel<5, true, kInlineMinB, 1, false, true>,
                                 tile_lean_kernel<0, false, kInlineMinB, 1, false, 2>, tile_lean_kernel<1, false, kInlineMinB, 1, false, 2>,
                                 tile_lean_kernel<0, true, kInlineMinB, 1, false, 2>, tile_lean_kernel<1, true, kInlineMinB, 1, false, 2>,
                                 tile_lean_kernel<0, false, kInlineMinB, 1, true, 2>, tile_lean_kernel<1, false, kInlineMinB, 1, true, 2>,
                                 tile_lean_kernel<0, true, kInlineMinB, 1, true, 2>, tile_lean_kernel<1, true, kInlineMinB, 1, true, 2>,
                                 tile_lean_kernel<2, false, kInlineMinB, 1, false, 2>, tile_lean_kernel<3, false, kInlineMinB, 1, false, 2>,
                                 tile_lean_kernel<4, false, kInlineMinB, 1, false, 2>, tile_lean_kernel<5, false, kInlineMinB, 1, false, 2>,
                                 tile_lean_kernel<2, true, kInlineMinB, 1, false, 2>, tile_lean_kernel<3, true, kInlineMinB, 1, false, 2>,
                                 tile_lean_kernel<4, true, kInlineMinB, 1, false, 2>, tile_lean_kernel<5, true, kInlineMinB, 1, false, 2>})
                    CK(cudaFuncSetAttribute(kk, cudaFuncAttributeMaxDynamicSharedMemorySize, b));
            }
        }
        if constexpr (!F32) {
            // fp64 Euler/Verlet on compact tiles: tile_f64_kernel (split
            // staging planes, 24 B per slot) unless SS_F64_KERNEL=step asks
            // for kernels.cuh's step_kernel
            const char *kenv = getenv("SS_F64_KERNEL");
            const std::string kname = kenv ? kenv : "tile";
            const size_t f64s = 128 + h->blob_smem + (size_t)(kTile + L.max_halo) * 24;
            if (kname != "step" && L.compact && !L.has_self &&
                (int64_t)f64s <= dev_max) {
                h->f64_smem = f64s;
                // programmatic dependent launch lets the next substep's CTAs
                // take SM slots early; for grids of ~1/3 to 3 CTAs per SM the
                // waiting CTAs pile onto the SMs left idle and the fp64 step
                // then runs two tiles on one SM: 360K springs 14.4 us with PDL
                // against 8.3 without (tools/wave_probe.py); smaller and
                // larger grids keep it (47 tiles 6.8 vs 8.3, 10M 63.4 vs 67.4)
                int sms = 0;
                CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->device));
                if (!getenv("SS_PDL") && L.n_tiles >= 48 && L.n_tiles <= 3 * (int64_t)sms) h->pdl = false;
                // (UNROLL, MINB) = (3, 3) up to ~13 tiles per SM: three incidences
                // in flight per lane beat the fourth CTA per SM while the grid is a
                // few waves (42-cell cube 12.3 -> 12.0 us, 60: 22.7 -> 21.9, 75:
                // 37.4 -> 37.0); (2, 4) beyond (80 cells 44.6 vs 45.2, the 10M
                // cube 63.3 vs 64.4; tools/f64_variant_probe.py)
                if (L.n_tiles <= 13 * (int64_t)sms) h->f64_variant = 3;
                // RK4 stages: up to 7 tiles per SM (42 cells 52.1 -> 50.5 us per
                // step, 60 cells 94.4 -> 91.9; 75 cells 163.8 against 169.0)
                if (L.n_tiles <= 7 * (int64_t)sms) h->f64_rk4_variant = 3;
                if (const char *e = getenv("SS_F64_VARIANT")) {
                    h->f64_variant = atoi(e);
                    h->f64_rk4_variant = h->f64_variant == 3 ? 3 : 0;
                }
                for (auto *kk : {tile_f64_kernel<0, false, 2, 4>, tile_f64_kernel<1, false, 2, 4>,
                                 tile_f64_kernel<0, true, 2, 4>, tile_f64_kernel<1, true, 2, 4>,
                                 tile_f64_kernel<0, false, 1, 4>, tile_f64_kernel<1, false, 1, 4>,
                                 tile_f64_kernel<0, true, 1, 4>, tile_f64_kernel<1, true, 1, 4>,
                                 tile_f64_kernel<0, false, 2, 3>, tile_f64_kernel<1, false, 2, 3>,
                                 tile_f64_kernel<0, true, 2, 3>, tile_f64_kernel<1, true, 2, 3>,
                                 tile_f64_kernel<0, false, 3, 3>, tile_f64_kernel<1, false, 3, 3>,
                                 tile_f64_kernel<0, true, 3, 3>, tile_f64_kernel<1, true, 3, 3>,
                                 tile_f64_kernel<0, false, 1, 5>, tile_f64_kernel<1, false, 1, 5>,
                                 tile_f64_kernel<0, true, 1, 5>, tile_f64_kernel<1, true, 1, 5>,
                                 tile_f64_kernel<0, false, 2, 5>, tile_f64_kernel<1, false, 2, 5>,
                                 tile_f64_kernel<0, true, 2, 5>, tile_f64_kernel<1, true, 2, 5>,
                                 tile_f64_kernel<2, false, 2, 4>, tile_f64_kernel<3, false, 2, 4>,
                                 tile_f64_kernel<4, false, 2, 4>, tile_f64_kernel<5, false, 2, 4>,
                                 tile_f64_kernel<2, true, 2, 4>, tile_f64_kernel<3, true, 2, 4>,
                                 tile_f64_kernel<4, true, 2, 4>, tile_f64_kernel<5, true, 2, 4>,
                                 tile_f64_kernel<0, false, 2, 4, true>, tile_f64_kernel<1, false, 2, 4, true>,
                                 tile_f64_kernel<0, true, 2, 4, true>, tile_f64_kernel<1, true, 2, 4, true>,
                                 tile_f64_kernel<2, false, 2, 4, true>, tile_f64_kernel<3, false, 2, 4, true>,
                                 tile_f64_kernel<4, false, 2, 4, true>, tile_f64_kernel<5, false, 2, 4, true>,
                                 tile_f64_kernel<2, true, 2, 4, true>, tile_f64_kernel<3, true, 2, 4, true>,
                                 tile_f64_kernel<4, true, 2, 4, true>, tile_f64_kernel<5, true, 2, 4, true>,
                                 tile_f64_kernel<2, false, 3, 3>, tile_f64_kernel<3, false, 3, 3>,
                                 tile_f64_kernel<4, false, 3, 3>, tile_f64_kernel<5, false, 3, 3>,
                                 tile_f64_kernel<2, true, 3, 3>, tile_f64_kernel<3, true, 3, 3>,
                                 tile_f64_kernel<4, true, 3, 3>, tile_f64_kernel<5, true, 3, 3>})
                    CK(cudaFuncSetAttribute(kk, cudaFuncAttributeMaxDynamicSharedMemorySize, dev_max));
            }
        }
        h->lay.canonical = L.canonical;
        return setup_resident<F32>(h, d);
    }
    LayoutInput li{N, S, d->si, d->sj};
    if ((rc = build_layout(li, layout, h->lay))) return rc;
    h->layout = h->lay.kind;
    auto up_typed = [&](void **dst, const std::vector<double> &src) -> int {
        std::vector<T> tv(src.begin(), src.end());
        return up_vec(h, dst, tv);
    };
    auto up_int = [&](int **dst, const std::vector<int> &src) -> int {
        void *p;
        int r = up_vec(h, &p, src);
        *dst = reinterpret_cast<int *>(p);
        return r;
    };
    if (h->layout == SS_LAYOUT_CSR) {
        if ((rc = up_int(&h->row, h->lay.row))) return rc;
        void *p;
        if ((rc = up_vec(h, &p, h->lay.inc))) return rc;
        h->inc = reinterpret_cast<int2 *>(p);
        std::vector<double> kv(d->k, d->k + S), lv(d->l0, d->l0 + S);
        if ((rc = up_typed(&h->k, kv))) return rc;
        if ((rc = up_typed(&h->l0, lv))) return rc;
        if (has_g) {
            std::vector<int> g(d->group, d->group + S);
            if ((rc = up_int(&h->grp, g))) return rc;
        }
    } else {
        const auto &L = h->lay;
        std::vector<double> ek(L.e_spring.size(), 0.0), el(L.e_spring.size(), 0.0);
        std::vector<int> eg;
        if (has_g) eg.assign(L.e_spring.size(), -1);
        for (size_t q = 0; q < L.e_spring.size(); ++q) {
            const int64_t s = L.e_spring[q];
            if (s < 0) continue;
            ek[q] = d->k[s];
            el[q] = d->l0[s];
            if (has_g) eg[q] = d->group[s];
        }
        if ((rc = up_int(&h->e_other, L.e_other))) return rc;
        if ((rc = up_typed(&h->e_k, ek))) return rc;
        if ((rc = up_typed(&h->e_l0, el))) return rc;
        if (has_g && (rc = up_int(&h->e_grp, eg))) return rc;
        if ((rc = up_int(&h->r_pos, L.r_pos))) return rc;
        if ((rc = up_int(&h->cnt, L.cnt))) return rc;
    }
    return setup_resident<F32>(h, d);
}

int64_t algorithmic_bytes(const ss_engine *h) {
    // fp32 16 B/spring + 64 B/mass; fp64 24 B/spring + 128 B/mass.
    const int64_t per_spring = h->precision == SS_F32 ? 16 : 24;
    const int64_t per_mass = h->precision == SS_F32 ? 64 : 128;
    return per_spring * h->S + per_mass * h->N;
}

// Settle asynchronously enqueued steps before another operation.  A
// divergence among them is held on the handle (the state is the diverged
// state, as in the reference) and raised by the next ss_step / ss_sync.
int sync_pending(ss_engine *h) {
    if (!h->pending) return SS_OK;
    ss_step_result r{};
    int rc = ss_sync(h, &r);
    if (rc == SS_EDIVERGED) {
        h->div_held = true;
        h->held = r;
        return SS_OK;
    }
    return rc;
}

// The held divergence, if any: reported once.
int take_held(ss_engine *h, ss_step_result *res) {
    if (!h->div_held) return SS_OK;
    h->div_held = false;
    if (res) *res = h->held;
    return ss::fail(SS_EDIVERGED,
                    "simulation diverged at step %lld: mass %lld has a non-finite position or "
                    "velocity (try a smaller dt)",
                    (long long)h->held.diverged_step, (long long)h->held.diverged_mass);
}

void release_inflight(ss_engine *h) {
    for (auto &f : h->inflight) h->spare_events.push_back(f.first);
    h->inflight.clear();
}

template <bool F32>
int forces_impl(ss_engine *h, const double *x, const double *v, double t) {
    using T = typename Prec<F32>::T;
    using T4 = typename Prec<F32>::T4;
    int rc;
    std::vector<double> tab(h->groups.size());
    if (!tab.empty()) {
        scales_at(h, t, tab.data());
        if ((rc = upload_scales<T>(h, tab))) return rc;
    }
    std::vector<T4> tx((size_t)h->ND), tv((size_t)h->ND);
    pack_positions<T, T4>(h, x, tx.data());
    pack_vec<T, T4>(h, v, tv.data());
    if ((rc = upload(h, h->d_tmp[0], tx.data(), tx.size() * sizeof(T4)))) return rc;
    if ((rc = upload(h, h->d_tmp[1], tv.data(), tv.size() * sizeof(T4)))) return rc;
    Params<T> p = base_params<T>(h);
    p.X = (const T4 *)h->d_tmp[0];
    p.V = (const T4 *)h->d_tmp[1];
    p.scale = tab.empty() ? nullptr : (const T *)h->scale;
    p.acc_out = (V3<double> *)h->d_acc;
    const int grid = h->grid();
    return with_layout(h, [&](auto L) -> int {
        constexpr int LY = decltype(L)::value;
        forces_kernel<F32, LY><<<grid, kBlock, LY >= 3 ? h->smem_bytes : 0, h->stream>>>(p);
        CK(cudaGetLastError());
        return SS_OK;
    });
}

// Page-locked staging buffer `which` (0-2) for one (ND) state vector, kept
// for the engine's lifetime: transfers run at full PCIe/C2C speed and the
// packing loop never page-faults a fresh allocation.  Uploads from these
// buffers are asynchronous (set_state_impl); a buffer is handed out for
// host writes only after they have completed.
template <typename T4>
int staging(ss_engine *h, T4 **out, int which = 0) {
    const size_t bytes = (size_t)h->ND * sizeof(T4);
    if (h->staged_pending) {
        CK(cudaEventSynchronize(h->staged));
        h->staged_pending = false;
    }
    void *&buf = h->pinned[which];
    size_t &have = h->pinned_bytes[which];
    if (have < bytes) {
        if (buf) cudaFreeHost(buf);
        buf = nullptr;
        have = 0;
        CK(cudaHostAlloc(&buf, bytes, cudaHostAllocDefault));
        have = bytes;
    }
    *out = reinterpret_cast<T4 *>(buf);
    return SS_OK;
}

// ---------------------------------------------- fp64 caller-layout transfers
// The caller's (N,3) f64 arrays cross the bus as they are (24 B per mass,
// not the 32 B device vectors) and are permuted into / out of the device
// order by these kernels, so the host does a plain parallel memcpy into
// pinned memory instead of a permuting gather.

__global__ void raw_to_device_kernel(const double *__restrict__ raw, const int *__restrict__ orig_of, int64_t nd,
                                     const double *__restrict__ w, double4 *__restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nd) return;
    const int64_t s = orig_of ? orig_of[i] : i;
    double4 o = make_double4(0.0, 0.0, 0.0, 0.0);
    if (s >= 0) {
        o.x = raw[3 * s];
        o.y = raw[3 * s + 1];
        o.z = raw[3 * s + 2];
        o.w = w ? w[i] : 0.0;                             // +-m for positions, 0 for velocities
    }
    out[i] = o;
}

__global__ void device_to_raw_kernel(const double4 *__restrict__ in, const int *__restrict__ orig_of, int64_t nd,
                                     double *__restrict__ raw) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nd) return;
    const int64_t s = orig_of ? orig_of[i] : i;
    if (s < 0) return;
    const double4 o = in[i];
    raw[3 * s] = o.x;
    raw[3 * s + 1] = o.y;
    raw[3 * s + 2] = o.z;
}

// fp32 tile engines (displacement state r = x - X0, X0 fp64 per device
// slot): the caller-layout f64 arrays converted on the device with the host
// packers' exact arithmetic (pack_positions / pack_vec / the u = x - x_prev
// rounding of set_state_impl, and their inverses), so fp32 state also
// crosses the bus as the caller's (N,3) f64 arrays.
__global__ void raw_to_f32_kernel(const double *__restrict__ raw, const double *__restrict__ raw_prev,
                                  const int *__restrict__ orig_of, int64_t nd, const double *__restrict__ x0,
                                  const double *__restrict__ w, float4 *__restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nd) return;
    const int64_t s = orig_of ? orig_of[i] : i;
    float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
    if (s >= 0) {
        if (x0) {                                          // position: r = x - X0, w = +-m
            o.x = (float)(raw[3 * s] - x0[3 * i]);
            o.y = (float)(raw[3 * s + 1] - x0[3 * i + 1]);
            o.z = (float)(raw[3 * s + 2] - x0[3 * i + 2]);
            o.w = (float)w[i];
        } else if (raw_prev) {                             // increment: u = x - x_prev
            o.x = (float)(raw[3 * s] - raw_prev[3 * s]);
            o.y = (float)(raw[3 * s + 1] - raw_prev[3 * s + 1]);
            o.z = (float)(raw[3 * s + 2] - raw_prev[3 * s + 2]);
        } else {                                           // velocity
            o.x = (float)raw[3 * s];
            o.y = (float)raw[3 * s + 1];
            o.z = (float)raw[3 * s + 2];
        }
    }
    out[i] = o;
}

// x = X0 + r (u == null), x_prev = X0 + (r - u), or v (x0 == null).
__global__ void f32_to_raw_kernel(const float4 *__restrict__ in, const float4 *__restrict__ u,
                                  const int *__restrict__ orig_of, int64_t nd, const double *__restrict__ x0,
                                  double *__restrict__ raw) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nd) return;
    const int64_t s = orig_of ? orig_of[i] : i;
    if (s < 0) return;
    const float4 r = in[i];
    if (!x0) {
        raw[3 * s] = (double)r.x;
        raw[3 * s + 1] = (double)r.y;
        raw[3 * s + 2] = (double)r.z;
    } else if (!u) {
        raw[3 * s] = x0[3 * i] + (double)r.x;
        raw[3 * s + 1] = x0[3 * i + 1] + (double)r.y;
        raw[3 * s + 2] = x0[3 * i + 2] + (double)r.z;
    } else {
        const float4 q = u[i];
        raw[3 * s] = x0[3 * i] + ((double)r.x - (double)q.x);
        raw[3 * s + 1] = x0[3 * i + 1] + ((double)r.y - (double)q.y);
        raw[3 * s + 2] = x0[3 * i + 2] + ((double)r.z - (double)q.z);
    }
}

size_t chunk_bytes() {
    static const size_t bytes = [] {
        const char *e = getenv("SS_CHUNK_MB");                // transfer chunk (MB), 4 by default
        const long mb = e ? atol(e) : 4;
        return (size_t)std::max(1l, std::min(mb, 256l)) << 20;
    }();
    return bytes;
}
#define kChunkBytes chunk_bytes()

int chunk_setup(ss_engine *h) {
    if (h->chunk_buf[0]) return SS_OK;
    for (int b = 0; b < 2; ++b) {
        CK(cudaHostAlloc(&h->chunk_buf[b], kChunkBytes, cudaHostAllocDefault));
        CK(cudaEventCreateWithFlags(&h->chunk_done[b], cudaEventDisableTiming));
    }
    if (!h->d_raw) {
        int rc = h->alloc(&h->d_raw, (size_t)h->N * 3 * sizeof(double));
        if (rc) return rc;
    }
    if (!h->d_w) {
        std::vector<double> w((size_t)h->ND, 0.0);
        for (int64_t i = 0; i < h->ND; ++i) {
            const int64_t s = h->src_of(i);
            if (s >= 0) w[i] = h->fixed[s] ? -h->m[s] : h->m[s];
        }
        int rc = up_vec(h, reinterpret_cast<void **>(&h->d_w), w);
        if (rc) return rc;
    }
    return SS_OK;
}

void par_copy(void *dst, const void *src, size_t bytes) {
    constexpr size_t kPiece = 256u << 10;
    const int64_t n = (int64_t)((bytes + kPiece - 1) / kPiece);
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < n; ++k) {
        const size_t o = (size_t)k * kPiece;
        std::memcpy(static_cast<char *>(dst) + o, static_cast<const char *>(src) + o, std::min(kPiece, bytes - o));
    }
}

// True if [p, p + bytes) lies in page-locked host memory (cudaHostAlloc'd
// or registered: torch pin_memory, ss_pinned_alloc), which the DMA engines
// read and write directly.
bool pinned_range(const void *p, size_t bytes) {
    if (!p || !bytes) return false;
    for (const void *q : {p, static_cast<const void *>(static_cast<const char *>(p) + bytes - 1)}) {
        cudaPointerAttributes a{};
        if (cudaPointerGetAttributes(&a, q) != cudaSuccess) {
            cudaGetLastError();
            return false;
        }
        if (a.type != cudaMemoryTypeHost) return false;
    }
    return true;
}

// host -> device.  Pinned source: one DMA straight from the caller's array
// (waited for before returning: the caller may reuse it).  Pageable source:
// chunk k is copied into pinned buffer k%2 while the DMA of chunk k-1 runs
// (pageable transfers are bound near 30 GB/s by host memory traffic on the
// B200 hosts, against 53 GB/s for a pinned DMA; tools/xfer_probe.py).
int h2d_chunked(ss_engine *h, void *dst, const void *src, size_t bytes) {
    if (pinned_range(src, bytes)) {
        CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, h->stream));
        CK(cudaEventRecord(h->chunk_done[0], h->stream));
        CK(cudaEventSynchronize(h->chunk_done[0]));
        return SS_OK;
    }
    for (size_t o = 0, k = 0; o < bytes; o += kChunkBytes, ++k) {
        const int b = (int)(k & 1);
        const size_t n = std::min(kChunkBytes, bytes - o);
        CK(cudaEventSynchronize(h->chunk_done[b]));               // its previous DMA (any call) has finished
        par_copy(h->chunk_buf[b], static_cast<const char *>(src) + o, n);
        CK(cudaMemcpyAsync(static_cast<char *>(dst) + o, h->chunk_buf[b], n, cudaMemcpyHostToDevice, h->stream));
        CK(cudaEventRecord(h->chunk_done[b], h->stream));
    }
    return SS_OK;
}

// device -> host.  Pinned destination: one DMA.  Pageable: the DMA of chunk
// k+1 runs while chunk k is copied out of its pinned buffer.
int d2h_chunked(ss_engine *h, void *dst, const void *src, size_t bytes) {
    if (pinned_range(dst, bytes)) {
        CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, h->stream));
        CK(cudaStreamSynchronize(h->stream));
        return SS_OK;
    }
    const size_t nk = (bytes + kChunkBytes - 1) / kChunkBytes;
    auto issue = [&](size_t k) -> int {
        const size_t o = k * kChunkBytes, n = std::min(kChunkBytes, bytes - o);
        CK(cudaMemcpyAsync(h->chunk_buf[k & 1], static_cast<const char *>(src) + o, n, cudaMemcpyDeviceToHost,
                           h->stream));
        CK(cudaEventRecord(h->chunk_done[k & 1], h->stream));
        return SS_OK;
    };
    int rc;
    if (nk && (rc = issue(0))) return rc;
    for (size_t k = 0; k < nk; ++k) {
        if (k + 1 < nk && (rc = issue(k + 1))) return rc;
        CK(cudaEventSynchronize(h->chunk_done[k & 1]));
        const size_t o = k * kChunkBytes;
        par_copy(static_cast<char *>(dst) + o, h->chunk_buf[k & 1], std::min(kChunkBytes, bytes - o));
    }
    return SS_OK;
}

int raw_upload(ss_engine *h, const double *src, void *dst_vec, bool position) {
    const size_t bytes = (size_t)h->N * 3 * sizeof(double);
    int rc = h2d_chunked(h, h->d_raw, src, bytes);
    if (rc) return rc;
    const unsigned grid = (unsigned)((h->ND + 255) / 256);
    raw_to_device_kernel<<<grid, 256, 0, h->stream>>>(h->d_raw, h->d_orig_of, h->ND, position ? h->d_w : nullptr,
                                                      reinterpret_cast<double4 *>(dst_vec));
    CK(cudaGetLastError());
    return SS_OK;
}

int raw_download(ss_engine *h, const void *src_vec, double *dst) {
    const unsigned grid = (unsigned)((h->ND + 255) / 256);
    device_to_raw_kernel<<<grid, 256, 0, h->stream>>>(reinterpret_cast<const double4 *>(src_vec), h->d_orig_of,
                                                      h->ND, h->d_raw);
    CK(cudaGetLastError());
    return d2h_chunked(h, dst, h->d_raw, (size_t)h->N * 3 * sizeof(double));
}

// Device X0 and the second raw buffer of the fp32 caller-layout transfers.
int f32_xfer_setup(ss_engine *h) {
    int rc = chunk_setup(h);
    if (rc) return rc;
    if (!h->d_raw2 && (rc = h->alloc(&h->d_raw2, (size_t)h->N * 3 * sizeof(double)))) return rc;
    if (!h->d_x0dev) {
        if ((rc = h->alloc(&h->d_x0dev, h->x0.size() * sizeof(double)))) return rc;
        if ((rc = upload(h, h->d_x0dev, h->x0.data(), h->x0.size() * sizeof(double)))) return rc;
    }
    return SS_OK;
}

// raw (caller layout, already on the device) -> one fp32 state vector
void f32_from_raw(ss_engine *h, const double *raw, const double *raw_prev, bool position, void *dst) {
    const unsigned grid = (unsigned)((h->ND + 255) / 256);
    raw_to_f32_kernel<<<grid, 256, 0, h->stream>>>(raw, raw_prev, h->d_orig_of, h->ND,
                                                   position ? h->d_x0dev : nullptr, h->d_w,
                                                   reinterpret_cast<float4 *>(dst));
}

int f32_download(ss_engine *h, const void *vec, const void *u, bool position, double *dst) {
    const unsigned grid = (unsigned)((h->ND + 255) / 256);
    f32_to_raw_kernel<<<grid, 256, 0, h->stream>>>(reinterpret_cast<const float4 *>(vec),
                                                   reinterpret_cast<const float4 *>(u), h->d_orig_of, h->ND,
                                                   position ? h->d_x0dev : nullptr, h->d_raw);
    CK(cudaGetLastError());
    return d2h_chunked(h, dst, h->d_raw, (size_t)h->N * 3 * sizeof(double));
}

template <bool F32>
int get_state_impl(ss_engine *h, double *x, double *v, double *x_prev) {
    using T = typename Prec<F32>::T;
    using T4 = typename Prec<F32>::T4;
    int rc;
    if constexpr (!F32) {                         // caller layout over the bus, permuted on the device
        if ((rc = chunk_setup(h))) return rc;
        if (h->staged_pending) {
            CK(cudaEventSynchronize(h->staged));
            h->staged_pending = false;
        }
        if (x && (rc = raw_download(h, h->X[h->cur], x))) return rc;
        if (v && (rc = raw_download(h, h->V, v))) return rc;
        if (x_prev && h->has_prev && (rc = raw_download(h, h->X[h->cur ^ 1], x_prev))) return rc;
        return SS_OK;
    } else if (h->rx0) {                          // fp32 tiles: converted on the device, caller layout over the bus
        if ((rc = f32_xfer_setup(h))) return rc;
        if (h->staged_pending) {
            CK(cudaEventSynchronize(h->staged));
            h->staged_pending = false;
        }
        if (x && (rc = f32_download(h, h->X[h->cur], nullptr, true, x))) return rc;
        if (v && (rc = f32_download(h, h->V, nullptr, false, v))) return rc;
        if (x_prev && h->has_prev) {
            rc = h->U ? f32_download(h, h->X[h->cur], h->U, true, x_prev)
                      : f32_download(h, h->X[h->cur ^ 1], nullptr, true, x_prev);
            if (rc) return rc;
        }
        return SS_OK;
    }
    T4 *tmp;
    rc = staging<T4>(h, &tmp);
    if (rc) return rc;
    const size_t bytes = (size_t)h->ND * sizeof(T4);
    if (x) {
        if ((rc = download_overlapped(h, tmp, h->X[h->cur], [&](int64_t i0, int64_t i1) {
                 unpack_positions<T, T4>(h, tmp, x, i0, i1);
             })))
            return rc;
    }
    if (v) {
        if ((rc = download_overlapped(h, tmp, h->V, [&](int64_t i0, int64_t i1) {
                 unpack_vec<T, T4>(h, tmp, v, i0, i1);
             })))
            return rc;
    }
    if (x_prev && h->has_prev) {
        if (F32 && h->U) {                        // x_prev = x - u, in fp64
            T4 *xr;
            if ((rc = staging<T4>(h, &xr, 1))) return rc;
            if ((rc = download(h, xr, h->X[h->cur], bytes))) return rc;
            if ((rc = download(h, tmp, h->U, bytes))) return rc;
#pragma omp parallel for schedule(static)
            for (int64_t i = 0; i < h->ND; ++i) {
                const int64_t s = h->src_of(i);
                if (s < 0) continue;
                const double r[3] = {(double)xr[i].x, (double)xr[i].y, (double)xr[i].z};
                const double u[3] = {(double)tmp[i].x, (double)tmp[i].y, (double)tmp[i].z};
                for (int c = 0; c < 3; ++c) {
                    const double b = h->rx0 ? h->x0[3 * i + c] : (double)h->base[4 * i + c];
                    x_prev[3 * s + c] = b + (r[c] - u[c]);
                }
            }
        } else {
            if ((rc = download_overlapped(h, tmp, h->X[h->cur ^ 1], [&](int64_t i0, int64_t i1) {
                     unpack_positions<T, T4>(h, tmp, x_prev, i0, i1);
                 })))
                return rc;
        }
    }
    return SS_OK;
}

template <bool F32>
int set_state_impl(ss_engine *h, const double *x, const double *v, const double *x_prev) {
    using T = typename Prec<F32>::T;
    using T4 = typename Prec<F32>::T4;
    // increment-form Verlet: a new x with the old x_prev means a new u
    std::vector<double> keep_prev;
    if (F32 && h->U && x && !x_prev && h->has_prev) {
        keep_prev.resize((size_t)h->N * 3);
        int r0 = get_state_impl<F32>(h, nullptr, nullptr, keep_prev.data());
        if (r0) return r0;
        x_prev = keep_prev.data();
    }
    int rc;
    if constexpr (F32) {
        // fp32 tiles: caller layout over the bus, converted on the device
        // (an x_prev without x, under increment-form Verlet, keeps the host path)
        if (h->rx0 && !(h->U && x_prev && !x)) {
            if ((rc = f32_xfer_setup(h))) return rc;
            const size_t bytes = (size_t)h->N * 3 * sizeof(double);
            if (x) {
                if ((rc = h2d_chunked(h, h->d_raw, x, bytes))) return rc;
                f32_from_raw(h, h->d_raw, nullptr, true, h->X[h->cur]);
            }
            if (v) {
                if ((rc = h2d_chunked(h, h->d_raw2, v, bytes))) return rc;
                f32_from_raw(h, h->d_raw2, nullptr, false, h->V);
            }
            if (x_prev) {
                if ((rc = h2d_chunked(h, h->d_raw2, x_prev, bytes))) return rc;
                if (h->U) f32_from_raw(h, h->d_raw, h->d_raw2, false, h->U);     // u = x - x_prev
                else f32_from_raw(h, h->d_raw2, nullptr, true, h->X[h->cur ^ 1]);
                h->has_prev = true;
            }
            CK(cudaGetLastError());
            return SS_OK;
        }
    }
    if constexpr (!F32) {                         // caller layout over the bus, permuted on the device
        if ((rc = chunk_setup(h))) return rc;
        if (x && (rc = raw_upload(h, x, h->X[h->cur], true))) return rc;
        if (v && (rc = raw_upload(h, v, h->V, false))) return rc;
        if (x_prev) {
            if ((rc = raw_upload(h, x_prev, h->X[h->cur ^ 1], true))) return rc;
            h->has_prev = true;
        }
        return SS_OK;
    }
    // each vector is packed into its own staging buffer and its upload is
    // queued at once, so packing the next vector overlaps the DMA of the
    // previous one; the stream orders the uploads before the next step
    T4 *bx, *bv, *tmp;
    if ((rc = staging<T4>(h, &bx, 0)) || (rc = staging<T4>(h, &bv, 1)) || (rc = staging<T4>(h, &tmp, 2)))
        return rc;
    const size_t bytes = (size_t)h->ND * sizeof(T4);
    auto upload_async = [&](void *dst, const void *src) -> int {
        CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, h->stream));
        CK(cudaEventRecord(h->staged, h->stream));
        h->staged_pending = true;
        return SS_OK;
    };
    if (x) {
        pack_positions<T, T4>(h, x, bx);
        if ((rc = upload_async(h->X[h->cur], bx))) return rc;
    }
    if (v) {
        pack_vec<T, T4>(h, v, bv);
        if ((rc = upload_async(h->V, bv))) return rc;
    }
    if (x_prev) {
        if (F32 && h->U) {                        // u = x - x_prev, in fp64 then rounded once
            std::vector<double> xc;
            const double *xs = x;
            if (!xs) {
                xc.resize((size_t)h->N * 3);
                if ((rc = get_state_impl<F32>(h, xc.data(), nullptr, nullptr))) return rc;
                xs = xc.data();
                if ((rc = staging<T4>(h, &tmp, 2))) return rc;
            }
#pragma omp parallel for schedule(static)
            for (int64_t i = 0; i < h->ND; ++i) {
                const int64_t s = h->src_of(i);
                T4 o{};
                if (s >= 0) {
                    o.x = (float)(xs[3 * s + 0] - x_prev[3 * s + 0]);
                    o.y = (float)(xs[3 * s + 1] - x_prev[3 * s + 1]);
                    o.z = (float)(xs[3 * s + 2] - x_prev[3 * s + 2]);
                }
                tmp[i] = o;
            }
            if ((rc = upload_async(h->U, tmp))) return rc;
        } else {
            pack_positions<T, T4>(h, x_prev, tmp);
            if ((rc = upload_async(h->X[h->cur ^ 1], tmp))) return rc;
        }
        h->has_prev = true;
    }
    return SS_OK;
}

}  // namespace

// ================================================================ C ABI

extern "C" {

int ss_abi_version(void) { return SS_ABI_VERSION; }

const char *ss_last_error(void) { return ss::last_error_slot().c_str(); }

int ss_device_count(int *count) {
    int c = 0;
    cudaError_t e = cudaGetDeviceCount(&c);
    if (e != cudaSuccess) {
        if (count) *count = 0;
        return ss::fail(SS_ECUDA, "cudaGetDeviceCount: %s", cudaGetErrorString(e));
    }
    if (count) *count = c;
    return SS_OK;
}

int ss_pinned_alloc(size_t bytes, void **out) {
    if (!out) return ss::fail(SS_EINVAL, "ss_pinned_alloc: null out");
    *out = nullptr;
    cudaError_t e = cudaHostAlloc(out, std::max<size_t>(bytes, 1), cudaHostAllocPortable);
    if (e != cudaSuccess) return ss::fail(SS_ECUDA, "cudaHostAlloc(%zu): %s", bytes, cudaGetErrorString(e));
    return SS_OK;
}

int ss_pinned_free(void *p) {
    if (!p) return SS_OK;
    cudaError_t e = cudaFreeHost(p);
    if (e != cudaSuccess) return ss::fail(SS_ECUDA, "cudaFreeHost: %s", cudaGetErrorString(e));
    return SS_OK;
}

}  // extern "C"
namespace {
int setup_persistent(ss_engine *h);
}  // namespace
extern "C" {

int ss_create(const ss_scene_desc *d, ss_engine **out) {
    if (!d || !out) return ss::fail(SS_EINVAL, "ss_create: null argument");
    *out = nullptr;
    if (d->n_masses <= 0) return ss::fail(SS_EINVAL, "scene has no masses");
    if (d->n_springs < 0) return ss::fail(SS_EINVAL, "negative spring count");
    if (!d->x || !d->v || !d->m) return ss::fail(SS_EINVAL, "x, v and m are required");
    if (d->n_springs && (!d->si || !d->sj || !d->k || !d->l0))
        return ss::fail(SS_EINVAL, "si, sj, k and l0 are required when n_springs > 0");
    if (d->integrator < SS_EULER || d->integrator > SS_RK4)
        return ss::fail(SS_EINVAL, "unknown integrator %d", d->integrator);
    if (d->precision != SS_F64 && d->precision != SS_F32)
        return ss::fail(SS_EINVAL, "unknown precision %d", d->precision);
    if (d->layout < SS_LAYOUT_AUTO || d->layout > SS_LAYOUT_TILE)
        return ss::fail(SS_EINVAL, "unknown layout %d", d->layout);
    if (d->n_planes < 0 || d->n_planes > kMaxPlanes)
        return ss::fail(SS_EINVAL, "at most %d contact planes are supported", kMaxPlanes);
    if (d->n_masses >= INT32_MAX || 2 * d->n_springs >= INT32_MAX)
        return ss::fail(SS_EINVAL, "scene too large for one device shard (use slab sharding)");
    for (int64_t s = 0; s < d->n_springs; ++s) {
        if (d->si[s] < 0 || d->si[s] >= d->n_masses || d->sj[s] < 0 || d->sj[s] >= d->n_masses)
            return ss::fail(SS_EINVAL, "spring %lld has an endpoint out of range", (long long)s);
        if (d->si[s] == d->sj[s])
            return ss::fail(SS_EINVAL, "spring %lld connects a mass to itself", (long long)s);
    }
    std::unique_ptr<ss_engine> h(new ss_engine);
    h->device = d->device;
    h->precision = d->precision;
    h->integrator = d->integrator;
    h->N = d->n_masses;
    h->S = d->n_springs;
    h->dt = d->dt;
    h->damping = d->damping;
    for (int c = 0; c < 3; ++c) h->gravity[c] = d->gravity[c];
    h->m.assign(d->m, d->m + h->N);
    h->fixed.assign((size_t)h->N, 0);
    if (d->fixed)
        for (int64_t i = 0; i < h->N; ++i) h->fixed[i] = d->fixed[i] ? 1 : 0;
    for (int g = 0; g < d->n_groups; ++g)
        h->groups.push_back({d->group_mode[g], d->group_amplitude[g], d->group_frequency[g],
                             d->group_phase[g]});
    h->planes.assign(d->planes, d->planes + 6 * d->n_planes);

    CK(cudaSetDevice(h->device));
    CK(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&h->staged, cudaEventDisableTiming));
    int rc;
    if ((rc = h->alloc(&h->d_degenerate, sizeof(unsigned long long)))) return rc;
    if ((rc = h->alloc(&h->d_div_step, sizeof(long long)))) return rc;
    if ((rc = h->alloc(&h->d_div_mass, sizeof(int)))) return rc;
    CK(cudaMemsetAsync(h->d_degenerate, 0, sizeof(unsigned long long), h->stream));
    if ((rc = reset_divergence(h.get()))) return rc;
    rc = h->precision == SS_F32 ? create_impl<true>(h.get(), d, d->layout)
                                : create_impl<false>(h.get(), d, d->layout);
    if (rc) return rc;
    if ((rc = setup_persistent(h.get()))) return rc;
    if ((rc = autotune_pdl(h.get()))) return rc;
    CK(cudaStreamSynchronize(h->stream));
    *out = h.release();
    return SS_OK;
}

int ss_destroy(ss_engine *h) {
    delete h;
    return SS_OK;
}

}  // extern "C"

namespace {

// Persistent cooperative stepping for small scenes (opt-in: SS_PERSIST=1),
// allowed when the whole grid fits co-resident and is at most 4 waves of
// SMs.  Measured slower than back-to-back launches on B200 (crawler fp32
// 6.5 vs 3.9 us/step, 40x4x4 beam 7.1 vs 4.4): a grid-wide barrier costs
// more than a pipelined launch boundary, and the per-step latency chain
// (TMA, halo gather) is the same.  DESIGN.md §4.
template <bool F32, int LAYOUT>
int setup_persistent_ly(ss_engine *h) {
    if (h->integrator == SS_RK4 || h->tl.inline_kl) return SS_OK;   // (persist_lean_kernel: dictionary tiles)
    const char *e = getenv("SS_PERSIST");
    if (!e || atoi(e) == 0) return SS_OK;
    int sms = 0, dev_max = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->device));
    CK(cudaDeviceGetAttribute(&dev_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, h->device));
    const bool euler = h->integrator == SS_EULER;
    const void *fn = euler ? (const void *)persist_step_kernel<F32, 0, LAYOUT>
                           : (const void *)persist_step_kernel<F32, 1, LAYOUT>;
    size_t sm = LAYOUT >= 3 ? h->smem_bytes : 0;
    if constexpr (F32 && LAYOUT >= 3) {
        if (h->lean_smem) {
            constexpr bool GROUPS = LAYOUT == 3;
            fn = euler ? (const void *)persist_lean_kernel<0, GROUPS> : (const void *)persist_lean_kernel<1, GROUPS>;
            sm = h->lean_smem;
        }
    }
    cudaFuncAttributes fa{};
    CK(cudaFuncGetAttributes(&fa, fn));
    CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, dev_max - (int)fa.sharedSizeBytes));
    if ((int64_t)(sm + fa.sharedSizeBytes) > dev_max) return SS_OK;
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kBlock, sm));
    const int grid = h->grid();
    if (per_sm > 0 && grid <= per_sm * sms && grid <= 4 * sms) h->persist_max_grid = per_sm * sms;
    return SS_OK;
}

int setup_persistent(ss_engine *h) {
    return with_layout(h, [&](auto L) -> int {
        return h->precision == SS_F32 ? setup_persistent_ly<true, decltype(L)::value>(h)
                                      : setup_persistent_ly<false, decltype(L)::value>(h);
    });
}

}  // namespace

extern "C" {

int ss_step(ss_engine *h, int64_t count, ss_step_result *res) {
    if (!h) return ss::fail(SS_EINVAL, "null engine");
    CK(cudaSetDevice(h->device));
    int rc = sync_pending(h);
    if (rc || (rc = take_held(h, res))) return rc;
    if (count <= 0) {
        if (res) *res = {0, h->n, h->t, -1, -1};
        return SS_OK;
    }
    const int64_t n0 = h->n;
    const int cur0 = h->cur;
    if ((rc = dispatch_steps(h, count))) return rc;
    return finish_batch(h, count, n0, cur0, res);
}

int ss_step_async(ss_engine *h, int64_t count) {
    if (!h) return ss::fail(SS_EINVAL, "null engine");
    if (count <= 0) return SS_OK;
    CK(cudaSetDevice(h->device));
    if (h->div_held) return take_held(h, nullptr);
    if (!h->pending) {
        h->pending_n0 = h->n;
        h->pending_cur0 = h->cur;
    }
    int rc = dispatch_steps(h, count);
    if (rc) return rc;
    h->pending += count;
    h->n += count;                   // provisional; ss_sync settles it
    h->t = (double)h->n * h->dt;
    cudaEvent_t ev = nullptr;
    if (!h->spare_events.empty()) {
        ev = h->spare_events.back();
        h->spare_events.pop_back();
    } else {
        CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    }
    CK(cudaEventRecord(ev, h->stream));
    h->inflight.push_back({ev, count});
    return SS_OK;
}

int ss_pending_wait(ss_engine *h, int64_t max_ahead) {
    if (!h) return ss::fail(SS_EINVAL, "null engine");
    CK(cudaSetDevice(h->device));
    int64_t ahead = 0;
    for (auto &f : h->inflight) ahead += f.second;
    size_t done = 0;
    while (done < h->inflight.size() && ahead > max_ahead) {
        CK(cudaEventSynchronize(h->inflight[done].first));
        ahead -= h->inflight[done].second;
        h->spare_events.push_back(h->inflight[done].first);
        ++done;
    }
    h->inflight.erase(h->inflight.begin(), h->inflight.begin() + (std::ptrdiff_t)done);
    return SS_OK;
}

}  // extern "C"

namespace {

int64_t dev_of(const ss_engine *h, int64_t caller) {
    return h->tl.new_of.empty() || h->orig_of.empty() ? caller : (int64_t)h->tl.new_of[caller];
}

int ensure(ss_engine *h, DevBuf &b, size_t bytes) {
    if (b.bytes >= bytes) return SS_OK;
    void *p;
    const int rc = h->alloc(&p, std::max<size_t>(bytes, 256));   // old buffer freed with the engine
    if (rc) return rc;
    b.p = p;
    b.bytes = std::max<size_t>(bytes, 256);
    return SS_OK;
}

// numpy's pairwise-summation recursion over n elements (sampling.cuh):
// leaves in order, internal nodes grouped by height, uploaded once.
int build_pw_plan(ss_engine *h, long long n, PwPlanDev &pl, double **vals, int nvals) {
    pl = PwPlanDev{};
    if (n <= 0) return SS_OK;
    std::vector<long long> off;
    std::vector<int> len;
    struct Inner { int l, r, height; };
    std::vector<Inner> inner;                    // child ids: >= 0 leaf, < 0 inner -(k + 1)
    struct Rec {
        std::vector<long long> &off; std::vector<int> &len; std::vector<Inner> &inner;
        int go(long long lo, long long m, int &height) {
            if (m <= 128) {
                off.push_back(lo);
                len.push_back((int)m);
                height = 0;
                return (int)off.size() - 1;
            }
            long long m2 = m / 2;
            m2 -= m2 % 8;
            int hl, hr;
            const int l = go(lo, m2, hl);
            const int r = go(lo + m2, m - m2, hr);
            height = std::max(hl, hr) + 1;
            inner.push_back({l, r, height});
            return -(int)inner.size();
        }
    } rec{off, len, inner};
    int top_h = 0;
    const int top = rec.go(0, n, top_h);
    const int L = (int)off.size();
    auto id = [&](int t) { return t >= 0 ? t : L + (-t - 1); };
    std::vector<int> order(inner.size());
    for (size_t k = 0; k < order.size(); ++k) order[k] = (int)k;
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return inner[a].height < inner[b].height; });
    std::vector<int4> nodes;
    std::vector<int> level_start;
    int cur_h = 0;
    for (int k : order) {
        while (cur_h < inner[k].height) {
            level_start.push_back((int)nodes.size());
            ++cur_h;
        }
        nodes.push_back(make_int4(id(inner[k].l), id(inner[k].r), L + k, 0));
    }
    level_start.push_back((int)nodes.size());
    int rc;
    void *p;
    if ((rc = up_vec(h, &p, off))) return rc;
    pl.leaf_off = reinterpret_cast<const long long *>(p);
    if ((rc = up_vec(h, &p, len))) return rc;
    pl.leaf_len = reinterpret_cast<const int *>(p);
    if (!nodes.empty()) {
        if ((rc = up_vec(h, &p, nodes))) return rc;
        pl.nodes = reinterpret_cast<const int4 *>(p);
        if ((rc = up_vec(h, &p, level_start))) return rc;
        pl.level_start = reinterpret_cast<const int *>(p);
    }
    pl.n_leaves = L;
    pl.n_levels = nodes.empty() ? 0 : (int)level_start.size() - 1;
    pl.root = id(top);
    for (int v = 0; v < nvals; ++v)
        if ((rc = h->alloc(&vals[v], (size_t)(L + inner.size()) * sizeof(double)))) return rc;
    return SS_OK;
}

// Launch the sample kernels for one row at the current device state
// (Verlet: x_prev buffer, others: x), scales row `scale_row`: traced
// positions, then EPE over the springs and GPE/KE over the masses, each a
// numpy pairwise sum in caller order (sampling.cuh).
int launch_sample(ss_engine *h, int64_t row, int n_ids, int use_prev) {
    SampleArgs a{};
    a.X = h->X[use_prev && !h->U ? (h->cur ^ 1) : h->cur];
    a.Usub = use_prev && h->U ? h->U : nullptr;          // fp32 Verlet: x_prev = x - u
    a.V = h->V;
    a.P = h->precision == SS_F32 ? reinterpret_cast<const float4 *>(h->P) : nullptr;
    a.mass = h->d_smass;
    a.x0 = h->rx0 ? h->d_sx0 : nullptr;
    a.nd = (int)h->ND;
    a.ssi = h->d_ssi;
    a.ssj = h->d_ssj;
    a.sk = h->d_sk;
    a.sl0 = h->d_sl0;
    a.sgrp = h->groups.empty() ? nullptr : h->d_sgrp;
    a.scale = reinterpret_cast<const double *>(h->d_sscale.p) + (size_t)row * std::max<size_t>(h->groups.size(), 1);
    a.n_springs = h->energy_springs;
    a.n_masses = h->N;
    a.dev_of = h->d_sdev_of;
    // |g| = np.linalg.norm(gravity): BLAS ddot, fma(g2, g2, fma(g1, g1, g0 g0)) (as lattice.cpp's l0)
    const double *g = h->gravity;
    a.g_mag = std::sqrt(std::fma(g[2], g[2], std::fma(g[1], g[1], g[0] * g[0])));
    for (int c = 0; c < 3; ++c) a.up[c] = a.g_mag > 0.0 ? -g[c] / a.g_mag : 0.0;
    a.datum = h->gpe_datum;
    a.ids = reinterpret_cast<const int *>(h->d_sids.p);
    a.n_ids = n_ids;
    a.pos_row = reinterpret_cast<double *>(h->d_srows.p) + (size_t)row * n_ids * 3;
    a.energy_row = reinterpret_cast<double *>(h->d_serows.p) + (size_t)row * 4;
    const bool f32 = h->precision == SS_F32;
    int launched = 0;
    if (n_ids) {
        const int gi = (n_ids + kSampleThreads - 1) / kSampleThreads;
        if (f32) sample_ids_kernel<true><<<gi, kSampleThreads, 0, h->stream>>>(a);
        else sample_ids_kernel<false><<<gi, kSampleThreads, 0, h->stream>>>(a);
        ++launched;
    }
    auto leaves = [&](const PwPlanDev &pl, auto kernel, double *v0, double *v1) {
        const unsigned gl = (unsigned)((8LL * pl.n_leaves + kSampleThreads - 1) / kSampleThreads);
        kernel<<<gl, kSampleThreads, 0, h->stream>>>(a, pl, v0, v1);
        ++launched;
        if (pl.n_levels) {
            pw_combine_kernel<<<1, 1024, 0, h->stream>>>(pl, v0, v1);
            ++launched;
        }
    };
    const bool springs = h->energy_springs > 0;
    if (springs) {
        if (f32) leaves(h->pw_springs, pw_leaf_kernel<true, true>, h->d_pwv[0], nullptr);
        else leaves(h->pw_springs, pw_leaf_kernel<false, true>, h->d_pwv[0], nullptr);
    }
    if (f32) leaves(h->pw_masses, pw_leaf_kernel<true, false>, h->d_pwv[1], h->d_pwv[2]);
    else leaves(h->pw_masses, pw_leaf_kernel<false, false>, h->d_pwv[1], h->d_pwv[2]);
    pw_final_kernel<<<1, 1, 0, h->stream>>>(h->d_pwv[0], h->pw_springs.root, h->d_pwv[1], h->d_pwv[2],
                                            h->pw_masses.root, springs, a.g_mag, a.energy_row);
    ++launched;
    CK(cudaGetLastError());
    h->launches += launched;
    return SS_OK;
}

}  // namespace

extern "C" {

int ss_energy_setup(ss_engine *h, int64_t n_springs, const int64_t *si, const int64_t *sj, const double *k,
                    const double *l0, const int32_t *group, double gpe_datum) {
    if (!h || n_springs < 0 || (n_springs && (!si || !sj || !k || !l0)))
        return ss::fail(SS_EINVAL, "ss_energy_setup: bad arguments");
    CK(cudaSetDevice(h->device));
    int rc = sync_pending(h);
    if (rc) return rc;
    h->gpe_datum = gpe_datum;
    if (h->energy_springs < 0) {
        const size_t S = (size_t)std::max<int64_t>(n_springs, 1);
        if ((rc = h->alloc(&h->d_ssi, S * sizeof(int))) || (rc = h->alloc(&h->d_ssj, S * sizeof(int))) ||
            (rc = h->alloc(&h->d_sgrp, S * sizeof(int))) || (rc = h->alloc(&h->d_sk, S * sizeof(double))) ||
            (rc = h->alloc(&h->d_sl0, S * sizeof(double))) ||
            (rc = h->alloc(&h->d_smass, (size_t)h->ND * sizeof(double))))
            return rc;
        std::vector<double> md((size_t)h->ND, 0.0);
        for (int64_t i = 0; i < h->ND; ++i) {
            const int64_t src = h->src_of(i);
            if (src >= 0) md[i] = h->m[src];
        }
        if ((rc = upload(h, h->d_smass, md.data(), md.size() * sizeof(double)))) return rc;
        if (h->rx0) {
            if ((rc = h->alloc(&h->d_sx0, h->x0.size() * sizeof(double)))) return rc;
            if ((rc = upload(h, h->d_sx0, h->x0.data(), h->x0.size() * sizeof(double)))) return rc;
        }
        std::vector<int> dv((size_t)h->N);
        for (int64_t c = 0; c < h->N; ++c) dv[c] = (int)dev_of(h, c);
        void *p;
        if ((rc = up_vec(h, &p, dv))) return rc;
        h->d_sdev_of = reinterpret_cast<int *>(p);
        if ((rc = build_pw_plan(h, n_springs, h->pw_springs, h->d_pwv, 1)) ||
            (rc = build_pw_plan(h, h->N, h->pw_masses, h->d_pwv + 1, 2)))
            return rc;
    } else if (n_springs != h->energy_springs) {
        return ss::fail(SS_EINVAL, "ss_energy_setup: spring count changed");
    }
    std::vector<int> a((size_t)n_springs), b((size_t)n_springs), g((size_t)n_springs, -1);
    for (int64_t s = 0; s < n_springs; ++s) {
        a[s] = (int)dev_of(h, si[s]);
        b[s] = (int)dev_of(h, sj[s]);
        if (group) g[s] = group[s];
    }
    if (n_springs) {
        if ((rc = upload(h, h->d_ssi, a.data(), a.size() * sizeof(int))) ||
            (rc = upload(h, h->d_ssj, b.data(), b.size() * sizeof(int))) ||
            (rc = upload(h, h->d_sgrp, g.data(), g.size() * sizeof(int))) ||
            (rc = upload(h, h->d_sk, k, (size_t)n_springs * sizeof(double))) ||
            (rc = upload(h, h->d_sl0, l0, (size_t)n_springs * sizeof(double))))
            return rc;
    }
    h->energy_springs = n_springs;
    return SS_OK;
}

int ss_step_sampled(ss_engine *h, int64_t count, int64_t sample_every, const int64_t *ids, int64_t n_ids,
                    int64_t max_rows, double *times_out, double *pos_out, double *energy_out,
                    int64_t *rows_out, ss_step_result *res) {
    if (!h || count < 0 || sample_every < 1 || n_ids < 0 || (n_ids && !ids) || max_rows < 0 || !rows_out)
        return ss::fail(SS_EINVAL, "ss_step_sampled: bad arguments");
    if (h->energy_springs < 0) return ss::fail(SS_EINVAL, "ss_step_sampled: call ss_energy_setup first");
    CK(cudaSetDevice(h->device));
    int rc = sync_pending(h);
    if (rc) return rc;
    const bool verlet = h->integrator == SS_VERLET;
    // plan the chunks exactly like simulate() (engine.py:546-559 with the
    // reference's sampling points): samples after steps whose index d
    // (Verlet: n-1, paired with x_prev) is a multiple of sample_every
    std::vector<int64_t> chunks, sample_d;
    {
        int64_t n = h->n, done = 0;
        while (done < count) {
            const int64_t target = verlet ? n - 1 : n;
            int64_t chunk = sample_every - (((target % sample_every) + sample_every) % sample_every);
            if (chunk <= 0) chunk = sample_every;
            chunk = std::min(chunk, count - done);
            n += chunk;
            done += chunk;
            chunks.push_back(chunk);
            const int64_t d = verlet ? n - 1 : n;
            sample_d.push_back(d % sample_every == 0 ? d : -1);
        }
    }
    int64_t rows = 0;
    for (int64_t d : sample_d) rows += d >= 0 ? 1 : 0;
    if (rows > max_rows) return ss::fail(SS_EINVAL, "ss_step_sampled: %lld rows > max_rows %lld",
                                         (long long)rows, (long long)max_rows);
    const size_t G = std::max<size_t>(h->groups.size(), 1);
    std::vector<double> sc((size_t)std::max<int64_t>(rows, 1) * G, 1.0);
    std::vector<int> dids((size_t)std::max<int64_t>(n_ids, 1), 0);
    for (int64_t i = 0; i < n_ids; ++i) dids[i] = (int)dev_of(h, ids[i]);
    {
        int64_t r = 0;
        for (int64_t d : sample_d)
            if (d >= 0) {
                if (!h->groups.empty()) scales_at(h, (double)d * h->dt, &sc[(size_t)r * G]);
                ++r;
            }
    }
    if ((rc = ensure(h, h->d_sids, dids.size() * sizeof(int))) ||
        (rc = ensure(h, h->d_srows, (size_t)std::max<int64_t>(rows, 1) * std::max<int64_t>(n_ids, 1) * 3 * sizeof(double))) ||
        (rc = ensure(h, h->d_serows, (size_t)std::max<int64_t>(rows, 1) * 4 * sizeof(double))) ||
        (rc = ensure(h, h->d_sscale, sc.size() * sizeof(double))))
        return rc;
    if ((rc = upload(h, h->d_sids.p, dids.data(), dids.size() * sizeof(int))) ||
        (rc = upload(h, h->d_sscale.p, sc.data(), sc.size() * sizeof(double))))
        return rc;
    // enqueue: chunk of steps, then the sample kernels (stream order), one
    // host synchronisation at the end
    const int64_t n0 = h->n;
    const int cur0 = h->cur;
    int64_t r = 0, total = 0;
    for (size_t c = 0; c < chunks.size(); ++c) {
        if ((rc = dispatch_steps(h, chunks[c]))) return rc;
        h->n += chunks[c];                    // provisional (dispatch reads h->n for scales)
        h->t = (double)h->n * h->dt;
        total += chunks[c];
        if (sample_d[c] >= 0) {
            if (times_out) times_out[r] = (double)sample_d[c] * h->dt;
            if ((rc = launch_sample(h, r, (int)n_ids, verlet ? 1 : 0))) return rc;
            ++r;
        }
    }
    h->n = n0;
    rc = finish_batch(h, total, n0, cur0, res);
    const int64_t valid = rc == SS_OK ? rows : 0;       // simulate() raises on divergence
    if (valid > 0) {
        if (pos_out && n_ids)
            CK(cudaMemcpy(pos_out, h->d_srows.p, (size_t)valid * n_ids * 3 * sizeof(double), cudaMemcpyDeviceToHost));
        if (energy_out) CK(cudaMemcpy(energy_out, h->d_serows.p, (size_t)valid * 4 * sizeof(double), cudaMemcpyDeviceToHost));
    }
    *rows_out = valid;
    return rc;
}

// Steering snapshot (service.py:378-389 _snapshot_bytes): the positions of
// `ids` and (epe, gpe, ke, total) at the current state (x, v; l0 scaled at
// t), gathered and reduced on the device -- no full-state download, no
// host-side O(S) energy pass.
int ss_snapshot(ss_engine *h, const int64_t *ids, int64_t n_ids, double gpe_datum, double *pos_out,
                double *energy_out) {
    if (!h || n_ids < 0 || (n_ids && (!ids || !pos_out))) return ss::fail(SS_EINVAL, "ss_snapshot: bad arguments");
    if (h->energy_springs < 0) return ss::fail(SS_EINVAL, "ss_snapshot: call ss_energy_setup first");
    CK(cudaSetDevice(h->device));
    int rc = sync_pending(h);
    if (rc) return rc;
    for (int64_t i = 0; i < n_ids; ++i)
        if (ids[i] < 0 || ids[i] >= h->N) return ss::fail(SS_EINVAL, "ss_snapshot: mass id %lld out of range", (long long)ids[i]);
    const size_t G = std::max<size_t>(h->groups.size(), 1);
    std::vector<double> sc(G, 1.0);
    if (!h->groups.empty()) scales_at(h, h->t, sc.data());
    std::vector<int> dids((size_t)std::max<int64_t>(n_ids, 1), 0);
    for (int64_t i = 0; i < n_ids; ++i) dids[i] = (int)dev_of(h, ids[i]);
    if ((rc = ensure(h, h->d_sids, dids.size() * sizeof(int))) ||
        (rc = ensure(h, h->d_srows, (size_t)std::max<int64_t>(n_ids, 1) * 3 * sizeof(double))) ||
        (rc = ensure(h, h->d_serows, 4 * sizeof(double))) || (rc = ensure(h, h->d_sscale, G * sizeof(double))))
        return rc;
    if ((rc = upload(h, h->d_sids.p, dids.data(), dids.size() * sizeof(int))) ||
        (rc = upload(h, h->d_sscale.p, sc.data(), G * sizeof(double))))
        return rc;
    const double datum = h->gpe_datum;
    h->gpe_datum = gpe_datum;
    rc = launch_sample(h, 0, (int)n_ids, 0);
    h->gpe_datum = datum;
    if (rc) return rc;
    CK(cudaStreamSynchronize(h->stream));
    if (n_ids) CK(cudaMemcpy(pos_out, h->d_srows.p, (size_t)n_ids * 3 * sizeof(double), cudaMemcpyDeviceToHost));
    if (energy_out) CK(cudaMemcpy(energy_out, h->d_serows.p, 4 * sizeof(double), cudaMemcpyDeviceToHost));
    return SS_OK;
}

int ss_sync(ss_engine *h, ss_step_result *res) {
    if (!h) return ss::fail(SS_EINVAL, "null engine");
    CK(cudaSetDevice(h->device));
    const int64_t count = h->pending;
    h->pending = 0;
    release_inflight(h);
    if (count == 0) {
        CK(cudaStreamSynchronize(h->stream));
        if (res) *res = {0, h->n, h->t, -1, -1};
        return take_held(h, res);
    }
    const int rc = finish_batch(h, count, h->pending_n0, h->pending_cur0, res);
    return h->div_held ? take_held(h, res) : rc;
}

int ss_set_gpe_datum(ss_engine *h, double datum) {
    if (!h) return ss::fail(SS_EINVAL, "null engine");
    h->gpe_datum = datum;
    return SS_OK;
}

void *ss_stream(ss_engine *h) { return h ? (void *)h->stream : nullptr; }

int ss_forces(ss_engine *h, const double *x, const double *v, double t, double *acc_out,
              int64_t *degenerate_out) {
    if (!h || !x || !v || !acc_out) return ss::fail(SS_EINVAL, "ss_forces: null argument");
    CK(cudaSetDevice(h->device));
    int rc = sync_pending(h);
    if (rc) return rc;
    const size_t vec = h->precision == SS_F32 ? sizeof(float4) : sizeof(double4);
    for (int b = 0; b < 2; ++b)
        if (!h->d_tmp[b] && (rc = h->alloc(&h->d_tmp[b], (size_t)h->ND * vec))) return rc;
    if (!h->d_acc && (rc = h->alloc(&h->d_acc, (size_t)h->N * 3 * sizeof(double)))) return rc;
    unsigned long long before = 0;
    CK(cudaMemcpy(&before, h->d_degenerate, sizeof before, cudaMemcpyDeviceToHost));
    rc = h->precision == SS_F32 ? forces_impl<true>(h, x, v, t) : forces_impl<false>(h, x, v, t);
    if (rc) return rc;
    h->launches += 1;
    if ((rc = download(h, acc_out, h->d_acc, (size_t)h->N * 3 * sizeof(double)))) return rc;
    unsigned long long after = 0;
    CK(cudaMemcpy(&after, h->d_degenerate, sizeof after, cudaMemcpyDeviceToHost));
    if (degenerate_out) *degenerate_out = (int64_t)(after - before);
    return SS_OK;
}

int ss_get_state(ss_engine *h, double *x, double *v, double *x_prev, int *has_prev) {
    if (!h) return ss::fail(SS_EINVAL, "null engine");
    CK(cudaSetDevice(h->device));
    int rc = sync_pending(h);
    if (rc) return rc;
    if (has_prev) *has_prev = h->has_prev ? 1 : 0;
    return h->precision == SS_F32 ? get_state_impl<true>(h, x, v, x_prev)
                                  : get_state_impl<false>(h, x, v, x_prev);
}

int ss_get_positions(ss_engine *h, double *x) { return ss_get_state(h, x, nullptr, nullptr, nullptr); }

int ss_set_state(ss_engine *h, const double *x, const double *v, const double *x_prev) {
    if (!h) return ss::fail(SS_EINVAL, "null engine");
    CK(cudaSetDevice(h->device));
    int rc = sync_pending(h);
    if (rc) return rc;
    return h->precision == SS_F32 ? set_state_impl<true>(h, x, v, x_prev)
                                  : set_state_impl<false>(h, x, v, x_prev);
}

int ss_clear_prev(ss_engine *h) {
    if (!h) return ss::fail(SS_EINVAL, "null engine");
    int rc = sync_pending(h);
    if (rc) return rc;
    h->has_prev = false;
    return SS_OK;
}

int ss_get_time(ss_engine *h, double *t, int64_t *n) {
    if (!h) return ss::fail(SS_EINVAL, "null engine");
    int rc = sync_pending(h);
    if (rc) return rc;
    if (t) *t = h->t;
    if (n) *n = h->n;
    return SS_OK;
}

int ss_set_time(ss_engine *h, double t, int64_t n) {
    if (!h) return ss::fail(SS_EINVAL, "null engine");
    int rc = sync_pending(h);
    if (rc) return rc;
    h->t = t;
    h->n = n;
    return SS_OK;
}

int ss_set_f_ext(ss_engine *h, const double *f) {
    if (!h || !f) return ss::fail(SS_EINVAL, "ss_set_f_ext: null argument");
    CK(cudaSetDevice(h->device));
    int rc = sync_pending(h);
    if (rc) return rc;
    bool any = false;
    for (int64_t i = 0; i < 3 * h->N && !any; ++i) any = f[i] != 0.0;
    h->has_fext = any;
    if (h->precision == SS_F32) {
        std::vector<float4> tmp((size_t)h->ND);
        pack_vec<float, float4>(h, f, tmp.data());
        return upload(h, h->F, tmp.data(), h->ND * sizeof(float4));
    }
    std::vector<double4> tmp((size_t)h->ND);
    pack_vec<double, double4>(h, f, tmp.data());
    return upload(h, h->F, tmp.data(), h->ND * sizeof(double4));
}

int ss_set_damping(ss_engine *h, double damping) {
    if (!h) return ss::fail(SS_EINVAL, "null engine");
    if (!std::isfinite(damping)) return ss::fail(SS_EINVAL, "damping must be finite");
    h->damping = damping;
    return SS_OK;
}

int ss_set_gravity(ss_engine *h, const double g[3]) {
    if (!h || !g) return ss::fail(SS_EINVAL, "ss_set_gravity: null argument");
    for (int c = 0; c < 3; ++c) h->gravity[c] = g[c];
    return SS_OK;
}

int ss_set_group(ss_engine *h, int32_t group, int32_t mode, double amplitude, double frequency,
                 double phase) {
    if (!h) return ss::fail(SS_EINVAL, "null engine");
    if (group < 0 || group >= (int32_t)h->groups.size())
        return ss::fail(SS_EINVAL, "unknown actuation group %d", group);
    h->groups[group] = {mode, amplitude, frequency, phase};
    return SS_OK;
}

int ss_degenerate_count(ss_engine *h, int64_t *count) {
    if (!h || !count) return ss::fail(SS_EINVAL, "ss_degenerate_count: null argument");
    CK(cudaSetDevice(h->device));
    unsigned long long c = 0;
    CK(cudaStreamSynchronize(h->stream));
    CK(cudaMemcpy(&c, h->d_degenerate, sizeof c, cudaMemcpyDeviceToHost));
    *count = (int64_t)c;
    return SS_OK;
}

int ss_get_info(ss_engine *h, ss_info *info) {
    if (!h || !info) return ss::fail(SS_EINVAL, "ss_get_info: null argument");
    std::memset(info, 0, sizeof *info);
    info->n_masses = h->N;
    info->n_springs = h->S;
    info->precision = h->precision;
    info->layout = h->layout;
    info->integrator = h->integrator;
    info->device = h->device;
    info->device_bytes = h->device_bytes;
    info->algorithmic_bytes_per_step = (double)algorithmic_bytes(h);
    if (h->layout == SS_LAYOUT_TILE) {
        info->ell_width_own = h->tl.max_W;
        info->ell_width_ref = h->tl.max_Wr;
        info->canonical_order = h->tl.canonical ? 1 : 0;
        info->tile_count = h->tl.n_tiles;
        info->tile_blob_bytes = (int64_t)(h->tl.blob.size() + 8 * h->tl.kl_inline.size() + h->tl.g_inline.size() +
                                          4 * h->tl.kd_inline.size());
        info->tile_halo_ratio = h->tl.halo_ratio;
        info->tile_foreign_frac = h->tl.foreign_frac;
        info->smem_per_block = (int32_t)h->smem_bytes;
        info->tile_kernel = h->lean_smem ? (h->tl.inline_kl ? 6 : h->tl.dict_x0 ? 7 : h->tl.compact ? 2 : 1)
                          : h->f64_smem ? (h->tl.inline_kl ? 5 : 4)
                                        : (h->precision == SS_F64 && h->tl.compact ? 3 : 0);
        info->kernel_smem = (int32_t)(h->lean_smem ? h->lean_smem : h->f64_smem ? h->f64_smem : h->smem_bytes);
    } else {
        info->ell_width_own = h->lay.W;
        info->ell_width_ref = h->lay.Wr;
        info->canonical_order = h->lay.canonical ? 1 : 0;
    }
    return SS_OK;
}

int64_t ss_launch_count(ss_engine *h) { return h ? h->launches : 0; }


}  // extern "C"

// Host-only planning: build the tiled layout of a scene without touching the
// device and report its statistics (used by tests and to size shards).
extern "C" int ss_plan(const ss_scene_desc *d, ss_info *info) {
    if (!d || !info) return ss::fail(SS_EINVAL, "ss_plan: null argument");
    if (d->n_masses <= 0 || !d->x || (d->n_springs && (!d->si || !d->sj || !d->k || !d->l0)))
        return ss::fail(SS_EINVAL, "ss_plan: incomplete scene");
    const bool f32 = d->precision == SS_F32;
    TileLayout tl;
    int rc = choose_tiles(d, f32, 232448, tl);             // (host-only: B200's opt-in shared memory per CTA)
    if (rc) return rc;
    std::memset(info, 0, sizeof *info);
    info->n_masses = d->n_masses;
    info->n_springs = d->n_springs;
    info->precision = d->precision;
    info->layout = SS_LAYOUT_TILE;
    info->integrator = d->integrator;
    info->ell_width_own = tl.max_W;
    info->ell_width_ref = tl.max_Wr;
    info->canonical_order = tl.canonical ? 1 : 0;
    info->tile_count = tl.n_tiles;
    info->tile_blob_bytes = (int64_t)(tl.blob.size() + 8 * tl.kl_inline.size() + tl.g_inline.size() +
                                      4 * tl.kd_inline.size());
    info->tile_halo_ratio = tl.halo_ratio;
    info->tile_foreign_frac = tl.foreign_frac;
    const size_t vec = f32 ? sizeof(float4) : sizeof(double4);
    info->smem_per_block =
        (int32_t)(128 + ((tl.max_tile_smem + 127u) & ~127u) + (size_t)(kTile + tl.max_halo) * vec);
    const int64_t per_spring = f32 ? 16 : 24, per_mass = f32 ? 64 : 128;
    info->algorithmic_bytes_per_step = (double)(per_spring * d->n_springs + per_mass * d->n_masses);
    info->kernel_smem = info->smem_per_block;
    info->tile_kernel = f32 ? (tl.inline_kl ? 6 : tl.dict_x0 ? 7 : tl.compact ? 2 : 1) : (tl.inline_kl ? 5 : tl.compact ? 3 : 0);
    return SS_OK;
}

// ============================================================ sharding
// x-slab sharding: halo lists, NCCL transport across
// processes, and same-process "virtual shards" stepped in lockstep.

namespace {

int64_t device_slot(const ss_engine *h, int64_t caller_id) {
    return h->tl.new_of.empty() || h->orig_of.empty() ? caller_id : (int64_t)h->tl.new_of[caller_id];
}

}  // namespace

extern "C" int ss_halo_setup(ss_engine *h, int64_t n_send_lo, const int64_t *send_lo, int64_t n_send_hi,
                             const int64_t *send_hi, int64_t n_recv_lo, const int64_t *recv_lo,
                             int64_t n_recv_hi, const int64_t *recv_hi) {
    if (!h) return ss::fail(SS_EINVAL, "null engine");
    CK(cudaSetDevice(h->device));
    const int64_t ns[2] = {n_send_lo, n_send_hi}, nr[2] = {n_recv_lo, n_recv_hi};
    const int64_t *sid[2] = {send_lo, send_hi}, *rid[2] = {recv_lo, recv_hi};
    const size_t vec = h->precision == SS_F32 ? sizeof(float4) : sizeof(double4);
    int rc;
    for (int s = 0; s < 2; ++s) {
        std::vector<int> si((size_t)ns[s]), ri((size_t)nr[s]);
        for (int64_t i = 0; i < ns[s]; ++i) {
            if (sid[s][i] < 0 || sid[s][i] >= h->N) return ss::fail(SS_EINVAL, "halo send id out of range");
            si[i] = (int)device_slot(h, sid[s][i]);
        }
        for (int64_t i = 0; i < nr[s]; ++i) {
            if (rid[s][i] < 0 || rid[s][i] >= h->N) return ss::fail(SS_EINVAL, "halo recv id out of range");
            if (!h->fixed[rid[s][i]]) return ss::fail(SS_EINVAL, "halo masses must be marked fixed");
            ri[i] = (int)device_slot(h, rid[s][i]);
        }
        h->halo_n_send[s] = (int)ns[s];
        h->halo_n_recv[s] = (int)nr[s];
        h->halo_send_host[s] = si;
        h->halo_recv_host[s] = ri;
        void *p;
        if ((rc = h->alloc(&p, si.size() * sizeof(int)))) return rc;
        h->halo_send_idx[s] = (int *)p;
        if (!si.empty() && (rc = upload(h, p, si.data(), si.size() * sizeof(int)))) return rc;
        if ((rc = h->alloc(&p, ri.size() * sizeof(int)))) return rc;
        h->halo_recv_idx[s] = (int *)p;
        if (!ri.empty() && (rc = upload(h, p, ri.data(), ri.size() * sizeof(int)))) return rc;
        if ((rc = h->alloc(&h->halo_send[s], (size_t)ns[s] * vec))) return rc;
        if ((rc = h->alloc(&h->halo_recv[s], (size_t)nr[s] * vec))) return rc;
    }
    h->halo_on = true;
    return SS_OK;
}

extern "C" int ss_nccl_unique_id(unsigned char id[128]) {
    const NcclApi *api = nccl_api();
    if (!api) return SS_ECUDA;
    ncclUniqueId u;
    const ncclResult_t r = api->getUniqueId(&u);
    if (r != ncclSuccess) return ss::fail(SS_ECUDA, "ncclGetUniqueId: %s", api->getErrorString(r));
    std::memcpy(id, &u, sizeof u);
    return SS_OK;
}

extern "C" int ss_halo_nccl(ss_engine *h, const unsigned char id[128], int nranks, int rank, int rank_lo,
                            int rank_hi) {
    if (!h || !id) return ss::fail(SS_EINVAL, "ss_halo_nccl: null argument");
    if (!h->halo_on) return ss::fail(SS_EINVAL, "call ss_halo_setup first");
    const NcclApi *api = nccl_api();
    if (!api) return SS_ECUDA;
    CK(cudaSetDevice(h->device));
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof u);
    const ncclResult_t r = api->commInitRank(&h->nccl, nranks, u, rank);
    if (r != ncclSuccess) return ss::fail(SS_ECUDA, "ncclCommInitRank: %s", api->getErrorString(r));
    h->nccl_peer[0] = rank_lo;
    h->nccl_peer[1] = rank_hi;
    return SS_OK;
}

// ------------------------------------------------ peer-memory halo transport

namespace {

constexpr char kMailboxMagic[8] = {'S', 'S', 'M', 'B', 'O', 'X', '0', '2'};

struct MailboxBlob {               // what ss_halo_p2p_export hands to the neighbours (256 B)
    char magic[8];
    cudaIpcMemHandle_t mailbox;    // 64 B each
    cudaIpcMemHandle_t x[2];       // the two position buffers (RK4: the state, then the XA|XB stage block)
    int64_t n_recv[2];
    int64_t vec;
    int64_t n;
    int32_t cur;
    int32_t device;
    int32_t integrator;
    int32_t pad;
    int64_t xb_off;                // RK4: XB's byte offset in the stage block
};
static_assert(sizeof(MailboxBlob) <= 256, "mailbox blob must fit 256 bytes");

int ensure_mailbox(ss_engine *h) {
    if (h->mailbox) return SS_OK;
    if (!h->halo_on) return ss::fail(SS_EINVAL, "call ss_halo_setup first");
    if (h->integrator == SS_RK4 && h->cur != 0) return ss::fail(SS_EINVAL, "RK4 halo: unexpected buffer parity");
    int rc = h->alloc(&h->mailbox, kMailboxHead);
    if (rc) return rc;
    MailboxHead head{};
    // the halos match the current state: its sequence number (RK4: four per step)
    head.flag[0] = head.flag[1] = (long long)h->n * (h->integrator == SS_RK4 ? 4 : 1);
    CK(cudaMemset(h->mailbox, 0, kMailboxHead));
    CK(cudaMemcpy(h->mailbox, &head, sizeof head, cudaMemcpyHostToDevice));
    return SS_OK;
}

// Per-slot push targets / ghost marks and per-CTA roles (kernels.cuh
// xchg_*): bit 0 wait for the neighbours' previous step (the CTA reads a
// ghost, as an own mass or through its halo, or pushes), bit 1 pushes, bit
// 2 owns ghosts.
int build_xchg(ss_engine *h) {
    const int64_t ND = h->ND;
    const int64_t nb = (ND + kBlockThreads - 1) / kBlockThreads;
    std::vector<int2> ps((size_t)ND, make_int2(-1, -1));
    for (int s = 0; s < 2; ++s)
        for (int32_t slot : h->halo_recv_host[s]) ps[slot].x = -2;
    for (int s = 0; s < 2; ++s) {
        if (!h->peer_mailbox[s]) continue;
        for (size_t k = 0; k < h->halo_send_host[s].size(); ++k) {
            int2 &q = ps[h->halo_send_host[s][k]];
            (s == 0 ? q.x : q.y) = h->peer_recv[s][k];
        }
    }
    std::vector<unsigned char> role((size_t)nb, 0);
    for (int64_t i = 0; i < ND; ++i) {
        unsigned char &r = role[i / kBlockThreads];
        if (ps[i].x >= 0 || ps[i].y >= 0) r |= 3;
        if (ps[i].x == -2) r |= 5;
    }
    if (h->layout == SS_LAYOUT_TILE && !h->tl.blob.empty()) {
        for (int64_t t = 0; t < h->tl.n_tiles && t < nb; ++t) {
            TileHdr th;
            std::memcpy(&th, h->tl.blob.data() + h->tl.off[t], sizeof th);
            const int32_t *halo = reinterpret_cast<const int32_t *>(h->tl.blob.data() + h->tl.off[t] + th.off_halo);
            for (uint32_t k = 0; k < th.n_halo && !(role[t] & 1); ++k)
                if (halo[k] >= 0 && ps[halo[k]].x == -2) role[t] |= 1;
        }
    } else {
        for (auto &r : role) r |= 1;                           // untiled layouts: every block may read a ghost
    }
    h->xchg_arrivals = 0;
    for (unsigned char r : role) h->xchg_arrivals += (r & 3) ? 1 : 0;
    // fp32 lean kernel launch order: the tiles the neighbours wait on first
    std::vector<int32_t> order;
    order.reserve((size_t)nb);
    for (int pass = 0; pass < 2; ++pass)
        for (int64_t b = 0; b < nb; ++b)
            if (((role[b] & 3) != 0) == (pass == 0)) order.push_back((int32_t)b);
    int rc;
    if (!h->d_tile_order && (rc = h->alloc(&h->d_tile_order, order.size() * sizeof(int32_t)))) return rc;
    if ((rc = upload(h, h->d_tile_order, order.data(), order.size() * sizeof(int32_t)))) return rc;
    if (!h->d_peer_slot && (rc = h->alloc(&h->d_peer_slot, ps.size() * sizeof(int2)))) return rc;
    if (!h->d_tile_role && (rc = h->alloc(&h->d_tile_role, role.size()))) return rc;
    if ((rc = upload(h, h->d_peer_slot, ps.data(), ps.size() * sizeof(int2)))) return rc;
    return upload(h, h->d_tile_role, role.data(), role.size());
}

// peer_xa / peer_xb: the neighbour's RK4 stage buffers (null unless RK4).
int link_side(ss_engine *h, int side, void *peer_mailbox, void *peer_x0, void *peer_x1, void *peer_xa,
              void *peer_xb, int integrator, bool ipc, const int64_t peer_n_recv[2], int64_t vec, int64_t n,
              int cur, const int32_t *peer_slots, int64_t n_slots) {
    const int64_t my_vec = h->precision == SS_F32 ? (int64_t)sizeof(float4) : (int64_t)sizeof(double4);
    if (vec != my_vec) return ss::fail(SS_EINVAL, "halo peer: precision differs");
    if (integrator != h->integrator) return ss::fail(SS_EINVAL, "halo peer: integrator differs");
    if (n != h->n || cur != h->cur) return ss::fail(SS_EINVAL, "halo peer: shards are not at the same step");
    if (peer_n_recv[1 - side] != h->halo_n_send[side] || n_slots != h->halo_n_send[side])
        return ss::fail(SS_EINVAL, "halo peer: plane sizes disagree (%lld received, %d sent)",
                        (long long)peer_n_recv[1 - side], h->halo_n_send[side]);
    h->peer_mailbox[side] = peer_mailbox;
    h->peer_X[side][0] = peer_x0;
    h->peer_X[side][1] = peer_x1;
    h->peer_XA[side] = peer_xa;
    h->peer_XB[side] = peer_xb;
    h->peer_ipc[side] = ipc;
    h->peer_recv[side].assign(peer_slots, peer_slots + n_slots);
    h->p2p_on = true;
    return build_xchg(h);
}

}  // namespace

extern "C" int ss_halo_p2p_export(ss_engine *h, unsigned char blob[256]) {
    if (!h || !blob) return ss::fail(SS_EINVAL, "ss_halo_p2p_export: null argument");
    CK(cudaSetDevice(h->device));
    int rc = sync_pending(h);
    if (rc || (rc = ensure_mailbox(h))) return rc;
    MailboxBlob b{};
    std::memcpy(b.magic, kMailboxMagic, 8);
    CK(cudaIpcGetMemHandle(&b.mailbox, h->mailbox));
    CK(cudaIpcGetMemHandle(&b.x[0], h->X[0]));
    CK(cudaIpcGetMemHandle(&b.x[1], h->integrator == SS_RK4 ? h->XA : h->X[1]));
    b.integrator = h->integrator;
    b.xb_off = h->integrator == SS_RK4 ? static_cast<char *>(h->XB) - static_cast<char *>(h->XA) : 0;
    b.n_recv[0] = h->halo_n_recv[0];
    b.n_recv[1] = h->halo_n_recv[1];
    b.vec = h->precision == SS_F32 ? (int64_t)sizeof(float4) : (int64_t)sizeof(double4);
    b.n = h->n;
    b.cur = h->cur;
    b.device = h->device;
    std::memset(blob, 0, 256);
    std::memcpy(blob, &b, sizeof b);
    return SS_OK;
}

extern "C" int ss_halo_recv_slots(ss_engine *h, int side, int32_t *out) {
    if (!h || side < 0 || side > 1 || (!out && h->halo_n_recv[side]))
        return ss::fail(SS_EINVAL, "ss_halo_recv_slots: bad argument");
    if (!h->halo_on) return ss::fail(SS_EINVAL, "call ss_halo_setup first");
    std::memcpy(out, h->halo_recv_host[side].data(), h->halo_recv_host[side].size() * sizeof(int32_t));
    return SS_OK;
}

extern "C" int ss_halo_p2p_attach(ss_engine *h, int side, const unsigned char blob[256], const int32_t *peer_slots,
                                  int64_t n_slots) {
    if (!h || !blob || side < 0 || side > 1 || (n_slots && !peer_slots))
        return ss::fail(SS_EINVAL, "ss_halo_p2p_attach: bad argument");
    MailboxBlob b;
    std::memcpy(&b, blob, sizeof b);
    if (std::memcmp(b.magic, kMailboxMagic, 8) != 0) return ss::fail(SS_EINVAL, "ss_halo_p2p_attach: not a mailbox blob");
    CK(cudaSetDevice(h->device));
    int rc = sync_pending(h);
    if (rc || (rc = ensure_mailbox(h))) return rc;
    void *pm[3] = {nullptr, nullptr, nullptr};
    const cudaIpcMemHandle_t hs[3] = {b.mailbox, b.x[0], b.x[1]};
    for (int i = 0; i < 3; ++i) {
        const cudaError_t e = cudaIpcOpenMemHandle(&pm[i], hs[i], cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) {
            for (int j = 0; j < i; ++j) cudaIpcCloseMemHandle(pm[j]);
            return ss::fail(SS_ECUDA, "cudaIpcOpenMemHandle (neighbour on device %d): %s", b.device,
                            cudaGetErrorString(e));
        }
    }
    // (an RK4 neighbour's second handle is its XA|XB stage block; RK4 never
    // pushes into the other parity of its state)
    const bool rk4 = b.integrator == SS_RK4;
    rc = link_side(h, side, pm[0], pm[1], pm[2], rk4 ? pm[2] : nullptr,
                   rk4 ? static_cast<char *>(pm[2]) + b.xb_off : nullptr, b.integrator, true, b.n_recv, b.vec,
                   b.n, b.cur, peer_slots, n_slots);
    if (rc)
        for (void *q : pm) cudaIpcCloseMemHandle(q);
    return rc;
}

extern "C" int ss_halo_p2p_link(ss_engine *h, int side, ss_engine *peer) {
    if (!h || !peer || side < 0 || side > 1) return ss::fail(SS_EINVAL, "ss_halo_p2p_link: bad argument");
    if (!peer->halo_on) return ss::fail(SS_EINVAL, "ss_halo_p2p_link: the peer has no halo");
    if (peer->device != h->device) {
        int ok = 0;
        CK(cudaDeviceCanAccessPeer(&ok, h->device, peer->device));
        if (!ok) return ss::fail(SS_EINVAL, "ss_halo_p2p_link: device %d cannot access device %d", h->device, peer->device);
        CK(cudaSetDevice(h->device));
        const cudaError_t e = cudaDeviceEnablePeerAccess(peer->device, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
            return ss::fail(SS_ECUDA, "cudaDeviceEnablePeerAccess: %s", cudaGetErrorString(e));
        cudaGetLastError();
    }
    CK(cudaSetDevice(peer->device));
    int rc = sync_pending(peer);
    if (rc || (rc = ensure_mailbox(peer))) return rc;
    CK(cudaSetDevice(h->device));
    if ((rc = sync_pending(h)) || (rc = ensure_mailbox(h))) return rc;
    const int64_t pnr[2] = {peer->halo_n_recv[0], peer->halo_n_recv[1]};
    const int64_t vec = peer->precision == SS_F32 ? (int64_t)sizeof(float4) : (int64_t)sizeof(double4);
    const std::vector<int32_t> &slots = peer->halo_recv_host[1 - side];
    return link_side(h, side, peer->mailbox, peer->X[0], peer->X[1], peer->XA, peer->XB, peer->integrator, false,
                     pnr, vec, peer->n, peer->cur, slots.data(), (int64_t)slots.size());
}

namespace {

// After a group batch: the shared divergence step decides how many steps
// every shard committed; the lowest shard whose own mass word was set names
// the mass (shards hold increasing global ids, and within a shard the word
// holds the lowest caller id).
int finish_group(ss_engine **hs, int n, int64_t count, const std::vector<int64_t> &n0, const std::vector<int> &cur0,
                 ss_step_result *res, int32_t *diverged_shard) {
    CK(cudaSetDevice(hs[0]->device));
    CK(cudaStreamSynchronize(hs[0]->stream));
    for (int k = 0; k < n; ++k) {
        if (!hs[k]->p2p_on) continue;
        int err = 0;
        CK(cudaMemcpy(&err, &reinterpret_cast<MailboxHead *>(hs[k]->mailbox)->error, sizeof err,
                      cudaMemcpyDeviceToHost));
        if (err) return ss::fail(SS_ECUDA, "halo exchange: a neighbour did not publish its boundary planes within 20 s");
    }
    long long dstep = LLONG_MAX;
    CK(cudaMemcpy(&dstep, hs[0]->d_div_step, sizeof dstep, cudaMemcpyDeviceToHost));
    int shard = -1, dmass = INT_MAX;
    for (int k = 0; k < n; ++k) {
        int mk = INT_MAX;
        CK(cudaMemcpy(&mk, hs[k]->d_div_mass, sizeof mk, cudaMemcpyDeviceToHost));
        if (mk != INT_MAX && shard < 0) {
            shard = k;
            dmass = mk;
        }
        ss_engine *h = hs[k];
        const int64_t done = dstep != LLONG_MAX ? (int64_t)dstep - n0[k] : count;
        h->n = n0[k] + done;
        h->t = (double)h->n * h->dt;
        if (h->integrator != SS_RK4) h->cur = cur0[k] ^ (int)(done & 1);
        if (dstep != LLONG_MAX) {
            int rc = reset_divergence(h);
            if (rc) return rc;
        }
    }
    if (res) {
        res->steps_done = dstep != LLONG_MAX ? (int64_t)dstep - n0[0] : count;
        res->n = hs[0]->n;
        res->t = hs[0]->t;
        res->diverged_mass = dstep != LLONG_MAX ? dmass : -1;
        res->diverged_step = dstep != LLONG_MAX ? (int64_t)dstep : -1;
    }
    if (diverged_shard) *diverged_shard = dstep != LLONG_MAX ? shard : -1;
    if (dstep != LLONG_MAX)
        return ss::fail(SS_EDIVERGED,
                        "simulation diverged at step %lld: mass %d of shard %d has a non-finite position or "
                        "velocity (try a smaller dt)",
                        dstep, dmass, shard);
    return SS_OK;
}

}  // namespace

// Step n same-device shards in lockstep; shard k's upper side is shard k+1's
// lower side.  All work is serialised on shard 0's stream.
extern "C" int ss_step_group(ss_engine **hs, int n, int64_t count, ss_step_result *res, int32_t *diverged_shard) {
    if (!hs || n <= 0) return ss::fail(SS_EINVAL, "ss_step_group: no engines");
    for (int k = 0; k < n; ++k) {
        if (!hs[k] || !hs[k]->halo_on) return ss::fail(SS_EINVAL, "ss_step_group: engine %d has no halo", k);
        if (hs[k]->device != hs[0]->device || hs[k]->precision != hs[0]->precision)
            return ss::fail(SS_EINVAL, "ss_step_group: engines must share device and precision");
        int rc = sync_pending(hs[k]);
        if (rc) return rc;
    }
    CK(cudaSetDevice(hs[0]->device));
    std::vector<cudaStream_t> saved(n);
    std::vector<int64_t> n0(n);
    std::vector<int> cur0(n);
    for (int k = 0; k < n; ++k) {
        saved[k] = hs[k]->stream;
        hs[k]->stream = hs[0]->stream;
        n0[k] = hs[k]->n;
        cur0[k] = hs[k]->cur;
    }
    int rc = SS_OK;
    const bool f32 = hs[0]->precision == SS_F32;
    const bool p2p = hs[0]->p2p_on;
    for (int k = 0; k < n; ++k) {
        if (hs[k]->p2p_on != p2p) {
            rc = ss::fail(SS_EINVAL, "ss_step_group: mix of peer-linked and unlinked shards");
            break;
        }
    }
    // the planes between neighbouring shards: buf(engine) is the position
    // buffer that just changed (the current state, or an RK4 stage's output)
    auto copy_planes = [&](auto buf) {
        for (int k = 0; k + 1 < n && rc == SS_OK; ++k) {
            ss_engine *a = hs[k], *b = hs[k + 1];
            const int na = a->halo_n_send[1], nb = b->halo_n_send[0];
            if (na != b->halo_n_recv[0] || nb != a->halo_n_recv[1]) {
                rc = ss::fail(SS_EINVAL, "ss_step_group: halo sizes of shards %d/%d disagree", k, k + 1);
                break;
            }
            void *xa = buf(a), *xb = buf(b);
            // (an empty plane -- no spring crosses this cut -- launches nothing)
            if (f32) {
                if (na) halo_copy_kernel<float4><<<(na + 255) / 256, 256, 0, a->stream>>>(
                    (const float4 *)xa, a->halo_send_idx[1], (float4 *)xb, b->halo_recv_idx[0], na);
                if (nb) halo_copy_kernel<float4><<<(nb + 255) / 256, 256, 0, a->stream>>>(
                    (const float4 *)xb, b->halo_send_idx[0], (float4 *)xa, a->halo_recv_idx[1], nb);
            } else {
                if (na) halo_copy_kernel<double4><<<(na + 255) / 256, 256, 0, a->stream>>>(
                    (const double4 *)xa, a->halo_send_idx[1], (double4 *)xb, b->halo_recv_idx[0], na);
                if (nb) halo_copy_kernel<double4><<<(nb + 255) / 256, 256, 0, a->stream>>>(
                    (const double4 *)xb, b->halo_send_idx[0], (double4 *)xa, a->halo_recv_idx[1], nb);
            }
            a->launches += (na ? 1 : 0) + (nb ? 1 : 0);
        }
    };
    // one divergence step for the whole group (shard 0's word): every shard
    // retires after the first non-finite step anywhere, like one engine
    for (int k = 1; k < n; ++k) hs[k]->group_div_step = hs[0]->d_div_step;
    const bool rk4 = hs[0]->integrator == SS_RK4;
    for (int k = 0; k < n && rc == SS_OK; ++k)
        if ((hs[k]->integrator == SS_RK4) != rk4) rc = ss::fail(SS_EINVAL, "ss_step_group: mix of RK4 and other integrators");
    for (int64_t s = 0; s < count && rc == SS_OK; ++s) {
        if (rk4) {
            // stage by stage across the shards: each stage's trial positions
            // reach the neighbours' halos before the next stage reads them
            // (stages 1 and 3 write XA, 2 writes XB, 4 the state)
            for (int st = 1; st <= 4 && rc == SS_OK; ++st) {
                for (int k = 0; k < n && rc == SS_OK; ++k) {
                    hs[k]->rk4_stage_only = st;
                    rc = dispatch_steps(hs[k], 1);
                    hs[k]->rk4_stage_only = 0;
                }
                if (!p2p)                                  // (peer-linked: the stage kernels pushed them)
                    copy_planes([st](ss_engine *e) -> void * {
                        return st == 2 ? e->XB : st == 4 ? e->X[e->cur] : e->XA;
                    });
            }
            for (int k = 0; k < n; ++k) {
                hs[k]->n += 1;
                hs[k]->t = (double)hs[k]->n * hs[k]->dt;
            }
            continue;
        }
        for (int k = 0; k < n && rc == SS_OK; ++k) {
            rc = dispatch_steps(hs[k], 1);
            hs[k]->n += 1;
            hs[k]->t = (double)hs[k]->n * hs[k]->dt;
        }
        if (p2p) continue;           // the step kernels exchanged the planes themselves
        copy_planes([](ss_engine *e) -> void * { return e->X[e->cur]; });
    }
    for (int k = 0; k < n; ++k) hs[k]->group_div_step = nullptr;
    if (diverged_shard) *diverged_shard = -1;
    if (rc == SS_OK) {
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) rc = ss::fail(SS_ECUDA, "ss_step_group: %s", cudaGetErrorString(e));
    }
    if (rc == SS_OK) rc = finish_group(hs, n, count, n0, cur0, res, diverged_shard);
    for (int k = 0; k < n; ++k) hs[k]->stream = saved[k];
    return rc;
}

extern "C" int ss_check_f64_fastpath(int32_t device, const double *a, const double *b, int64_t n, double *out,
                                     int32_t *ok) {
    if (!a || !b || !out || !ok || n < 0 || n > (1ll << 28)) return ss::fail(SS_EINVAL, "ss_check_f64_fastpath: bad arguments");
    if (n == 0) return SS_OK;
    CK(cudaSetDevice(device));
    double *da = nullptr, *db = nullptr, *dout = nullptr;
    int *dok = nullptr;
    const size_t nb = (size_t)n * sizeof(double);
    cudaError_t e = cudaMalloc(&da, nb);
    if (e == cudaSuccess) e = cudaMalloc(&db, nb);
    if (e == cudaSuccess) e = cudaMalloc(&dout, 4 * nb);
    if (e == cudaSuccess) e = cudaMalloc(&dok, (size_t)n * sizeof(int));
    if (e == cudaSuccess) e = cudaMemcpy(da, a, nb, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(db, b, nb, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) {
        f64_fastpath_check<<<(unsigned)((n + 255) / 256), 256>>>(da, db, (int)n, dout, dok);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpy(out, dout, 4 * nb, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess) e = cudaMemcpy(ok, dok, (size_t)n * sizeof(int), cudaMemcpyDeviceToHost);
    cudaFree(da);
    cudaFree(db);
    cudaFree(dout);
    cudaFree(dok);
    if (e != cudaSuccess) return ss::fail(SS_ECUDA, "ss_check_f64_fastpath: %s", cudaGetErrorString(e));
    return SS_OK;
}

