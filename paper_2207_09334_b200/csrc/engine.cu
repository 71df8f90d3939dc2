// Engine object and C ABI (include/springsim_b200.h).
//
// Host side of the relaxation loop: freezes a scene description into device
// buffers (engine.py:182-246), builds the incidence layout, and drives the
// per-step kernels of kernels.cuh on a private CUDA stream.  A batch of
// `count` steps is enqueued back-to-back (CUDA graph per batch length) with
// the divergence check fused into each step's epilogue, so a batch costs one
// host synchronisation, not one per step (engine.py:366-373 syncs per step).

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <type_traits>
#include <vector>

#include "common.h"
#include "kernels.cuh"
#include "layout.h"
#include "springsim_b200.h"

using namespace ss;

#define CK(expr)                                                                         \
    do {                                                                                 \
        cudaError_t _e = (expr);                                                         \
        if (_e != cudaSuccess)                                                           \
            return ss::fail(SS_ECUDA, "%s failed: %s", #expr, cudaGetErrorString(_e));   \
    } while (0)

namespace {

constexpr int kBlock = 256;

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
    size_t elem = 8;               // sizeof(T)
    size_t vec = 32;               // sizeof(T4)

    // host-side scalars (engine.py:190-194, 222-224)
    double dt = 1e-4, damping = 0.0, gravity[3] = {0, 0, 0};
    std::vector<Group> groups;
    std::vector<double> planes;    // 6 per plane
    std::vector<double> m;         // masses
    std::vector<uint8_t> fixed;
    double t = 0.0;
    int64_t n = 0;
    bool has_prev = false;
    bool has_fext = false;
    int64_t degenerate_host = 0;   // folded-in count

    // device state
    std::vector<DevBuf> bufs;
    void *X[2] = {nullptr, nullptr};
    int cur = 0;
    void *V = nullptr;
    void *P = nullptr;             // fp32 base positions
    void *F = nullptr;             // f_ext
    void *XA = nullptr, *XB = nullptr, *VS = nullptr, *SV = nullptr, *SA = nullptr;  // RK4
    void *scale = nullptr;
    size_t scale_cap = 0;
    unsigned long long *d_degenerate = nullptr;
    long long *d_div_step = nullptr;
    int *d_div_mass = nullptr;
    void *d_acc = nullptr;         // forces scratch (double3 x N)
    void *d_tmp[2] = {nullptr, nullptr};

    // topology
    Layout lay;
    void *k = nullptr, *l0 = nullptr, *e_k = nullptr, *e_l0 = nullptr;
    int *row = nullptr, *grp = nullptr, *e_other = nullptr, *e_grp = nullptr, *r_pos = nullptr,
        *cnt = nullptr;
    int2 *inc = nullptr;
    int64_t device_bytes = 0;
    int64_t launches = 0;
    int64_t pending = 0;           // steps enqueued by ss_step_async and not yet synced
    int64_t pending_n0 = 0;
    int pending_cur0 = 0;
    double pending_t0 = 0.0;

    ~ss_engine() {
        if (device >= 0) cudaSetDevice(device);
        for (auto &b : bufs) cudaFree(b.p);
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
};

namespace {

// ------------------------------------------------------------ conversions

// Pack (N,3) f64 host positions into the device T4 representation.
//   fp64: (x, y, z, +-m)             fp32: r = float(x - P), .w = +-m
template <typename T, typename T4>
void pack_positions(const ss_engine *h, const double *x, const float *base, T4 *out) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < h->N; ++i) {
        T4 o;
        const double w = h->fixed[i] ? -h->m[i] : h->m[i];
        if constexpr (std::is_same<T, float>::value) {
            o.x = (float)(x[3 * i + 0] - (double)base[4 * i + 0]);
            o.y = (float)(x[3 * i + 1] - (double)base[4 * i + 1]);
            o.z = (float)(x[3 * i + 2] - (double)base[4 * i + 2]);
            o.w = (float)w;
        } else {
            o.x = x[3 * i + 0];
            o.y = x[3 * i + 1];
            o.z = x[3 * i + 2];
            o.w = w;
        }
        out[i] = o;
    }
}

template <typename T, typename T4>
void pack_vec(int64_t N, const double *v, T4 *out) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < N; ++i) {
        T4 o;
        o.x = (T)v[3 * i + 0];
        o.y = (T)v[3 * i + 1];
        o.z = (T)v[3 * i + 2];
        o.w = (T)0;
        out[i] = o;
    }
}

template <typename T, typename T4>
void unpack_positions(const ss_engine *h, const T4 *in, const float *base, double *x) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < h->N; ++i) {
        if constexpr (std::is_same<T, float>::value) {
            x[3 * i + 0] = (double)base[4 * i + 0] + (double)in[i].x;
            x[3 * i + 1] = (double)base[4 * i + 1] + (double)in[i].y;
            x[3 * i + 2] = (double)base[4 * i + 2] + (double)in[i].z;
        } else {
            x[3 * i + 0] = in[i].x;
            x[3 * i + 1] = in[i].y;
            x[3 * i + 2] = in[i].z;
        }
    }
}

template <typename T, typename T4>
void unpack_vec(int64_t N, const T4 *in, double *v) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < N; ++i) {
        v[3 * i + 0] = (double)in[i].x;
        v[3 * i + 1] = (double)in[i].y;
        v[3 * i + 2] = (double)in[i].z;
    }
}

// The fp32 base positions live on the host too (needed to pack/unpack).
struct HostBase {
    std::vector<float> p;   // 4 per mass
};
std::mutex g_base_mu;
std::map<const ss_engine *, HostBase> g_base;

const float *host_base(const ss_engine *h) {
    std::lock_guard<std::mutex> lk(g_base_mu);
    auto it = g_base.find(h);
    return it == g_base.end() ? nullptr : it->second.p.data();
}

// Upload a host array (pageable) into a device buffer on the engine stream.
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

// ----------------------------------------------------------- actuation

// Scale table for `count` steps starting at (t0, n0): the exact Python
// expression of engine.py:250-259 (math.sin is libm sin).
// Euler/Verlet: one evaluation time per step (self.t, which is t0 for the
// first step and n*dt afterwards); RK4: t, t+dt/2, t+dt/2, t+dt.
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
        for (int q = 0; q < stages; ++q)
            for (size_t g = 0; g < G; ++g) {
                const Group &gr = h->groups[g];
                double sc;
                if (gr.mode == SS_CONSTANT_EXPANSION) sc = 1.0 + gr.amplitude;
                else sc = 1.0 + gr.amplitude * std::sin(2.0 * M_PI * gr.frequency * st[q] + gr.phase);
                out[((size_t)s * stages + q) * G + g] = sc;
            }
    }
}

template <typename T>
int upload_scales(ss_engine *h, const std::vector<double> &tab) {
    if (tab.empty()) return SS_OK;
    const size_t bytes = tab.size() * sizeof(T);
    if (bytes > h->scale_cap) {
        if (h->scale) {
            cudaFree(h->scale);
            for (auto &b : h->bufs)
                if (b.p == h->scale) { h->device_bytes -= (int64_t)b.bytes; b.p = nullptr; b.bytes = 0; }
        }
        void *p;
        int rc = h->alloc(&p, std::max<size_t>(bytes, 4096));
        if (rc) return rc;
        h->scale = p;
        h->scale_cap = std::max<size_t>(bytes, 4096);
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
    p.n = (int)h->N;
    p.P = reinterpret_cast<const T4 *>(h->P);
    p.F = h->has_fext ? reinterpret_cast<const T4 *>(h->F) : nullptr;
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
    p.div_step = h->d_div_step;
    p.div_mass = h->d_div_mass;
    return p;
}

template <bool F32, int LAYOUT>
int launch_steps(ss_engine *h, int64_t count) {
    using T = typename Prec<F32>::T;
    using T4 = typename Prec<F32>::T4;
    const int stages = h->integrator == SS_RK4 ? 4 : 1;
    const size_t G = h->groups.size();
    std::vector<double> tab;
    if (G) {
        build_scales(h, count, stages, h->t, h->n, tab);
        int rc = upload_scales<T>(h, tab);
        if (rc) return rc;
    }
    const int grid = (int)((h->N + kBlock - 1) / kBlock);
    Params<T> p = base_params<T>(h);
    const T *scale = reinterpret_cast<const T *>(h->scale);
    for (int64_t s = 0; s < count; ++s) {
        p.step = h->n + s + 1;
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
            p.bootstrap = (h->integrator == SS_VERLET && !h->has_prev) ? 1 : 0;
            if (h->integrator == SS_EULER) step_kernel<F32, 0, LAYOUT><<<grid, kBlock, 0, h->stream>>>(p);
            else step_kernel<F32, 1, LAYOUT><<<grid, kBlock, 0, h->stream>>>(p);
            h->launches += 1;
            h->cur ^= 1;
            if (h->integrator == SS_VERLET) h->has_prev = true;
        } else {
            T4 *XA = reinterpret_cast<T4 *>(h->XA), *XB = reinterpret_cast<T4 *>(h->XB);
            T4 *VS = reinterpret_cast<T4 *>(h->VS);
            p.X0 = Xc;
            p.V0 = V;
            p.SV = reinterpret_cast<T4 *>(h->SV);
            p.SA = reinterpret_cast<T4 *>(h->SA);
            // stage 1: (x0, v0) -> (XA, VS)
            p.scale = G ? scale + ((size_t)s * 4 + 0) * G : nullptr;
            p.X = Xc; p.V = V; p.Xout = XA; p.Vout = VS;
            rk4_kernel<F32, 1, LAYOUT><<<grid, kBlock, 0, h->stream>>>(p);
            // stage 2: (XA, VS) -> (XB, VS)
            p.scale = G ? scale + ((size_t)s * 4 + 1) * G : nullptr;
            p.X = XA; p.V = VS; p.Xout = XB; p.Vout = VS;
            rk4_kernel<F32, 2, LAYOUT><<<grid, kBlock, 0, h->stream>>>(p);
            // stage 3: (XB, VS) -> (XA, VS)
            p.scale = G ? scale + ((size_t)s * 4 + 2) * G : nullptr;
            p.X = XB; p.V = VS; p.Xout = XA; p.Vout = VS;
            rk4_kernel<F32, 3, LAYOUT><<<grid, kBlock, 0, h->stream>>>(p);
            // stage 4: (XA, VS) -> (x0, v0) in place
            p.scale = G ? scale + ((size_t)s * 4 + 3) * G : nullptr;
            p.X = XA; p.V = VS; p.Xout = Xc; p.Vout = V;
            rk4_kernel<F32, 4, LAYOUT><<<grid, kBlock, 0, h->stream>>>(p);
            h->launches += 4;
        }
    }
    CK(cudaGetLastError());
    return SS_OK;
}

int dispatch_steps(ss_engine *h, int64_t count) {
    if (h->precision == SS_F32) {
        return h->layout == SS_LAYOUT_ELL ? launch_steps<true, 2>(h, count) : launch_steps<true, 1>(h, count);
    }
    return h->layout == SS_LAYOUT_ELL ? launch_steps<false, 2>(h, count) : launch_steps<false, 1>(h, count);
}

int reset_divergence(ss_engine *h) {
    const long long none = LLONG_MAX;
    const int nonei = INT_MAX;
    CK(cudaMemcpyAsync(h->d_div_step, &none, sizeof none, cudaMemcpyHostToDevice, h->stream));
    CK(cudaMemcpyAsync(h->d_div_mass, &nonei, sizeof nonei, cudaMemcpyHostToDevice, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    return SS_OK;
}

// After an enqueued batch: read the divergence record, fix up n/t/cur.
int finish_batch(ss_engine *h, int64_t count, int64_t n0, int cur0, ss_step_result *res) {
    CK(cudaStreamSynchronize(h->stream));
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

template <bool F32>
int create_impl(ss_engine *h, const ss_scene_desc *d) {
    using T = typename Prec<F32>::T;
    using T4 = typename Prec<F32>::T4;
    const int64_t N = h->N, S = h->S;
    int rc;
    // fp32 base positions
    std::vector<float> base;
    if (F32) {
        base.resize((size_t)N * 4);
        for (int64_t i = 0; i < N; ++i) {
            for (int c = 0; c < 3; ++c) base[4 * i + c] = (float)d->x[3 * i + c];
            base[4 * i + 3] = 0.f;
        }
        if ((rc = h->alloc(&h->P, (size_t)N * sizeof(T4)))) return rc;
        if ((rc = upload(h, h->P, base.data(), (size_t)N * sizeof(T4)))) return rc;
        std::lock_guard<std::mutex> lk(g_base_mu);
        g_base[h].p = base;
    }
    for (int b = 0; b < 2; ++b)
        if ((rc = h->alloc(&h->X[b], (size_t)N * sizeof(T4)))) return rc;
    if ((rc = h->alloc(&h->V, (size_t)N * sizeof(T4)))) return rc;
    if ((rc = h->alloc(&h->F, (size_t)N * sizeof(T4)))) return rc;
    if (h->integrator == SS_RK4) {
        if ((rc = h->alloc(&h->XA, (size_t)N * sizeof(T4)))) return rc;
        if ((rc = h->alloc(&h->XB, (size_t)N * sizeof(T4)))) return rc;
        if ((rc = h->alloc(&h->VS, (size_t)N * sizeof(T4)))) return rc;
        if ((rc = h->alloc(&h->SV, (size_t)N * sizeof(T4)))) return rc;
        if ((rc = h->alloc(&h->SA, (size_t)N * sizeof(T4)))) return rc;
    }
    {
        std::vector<T4> tmp((size_t)N);
        pack_positions<T, T4>(h, d->x, F32 ? base.data() : nullptr, tmp.data());
        if ((rc = upload(h, h->X[0], tmp.data(), (size_t)N * sizeof(T4)))) return rc;
        pack_vec<T, T4>(N, d->v, tmp.data());
        if ((rc = upload(h, h->V, tmp.data(), (size_t)N * sizeof(T4)))) return rc;
        if (d->f_ext) {
            pack_vec<T, T4>(N, d->f_ext, tmp.data());
            for (int64_t i = 0; i < 3 * N && !h->has_fext; ++i) h->has_fext = d->f_ext[i] != 0.0;
        } else {
            std::memset(tmp.data(), 0, (size_t)N * sizeof(T4));
        }
        if ((rc = upload(h, h->F, tmp.data(), (size_t)N * sizeof(T4)))) return rc;
    }
    // topology
    LayoutInput li{N, S, d->si, d->sj};
    int want = d->layout;
    if ((rc = build_layout(li, want, h->lay))) return rc;
    h->layout = h->lay.kind;
    auto up_typed = [&](void **dst, const std::vector<double> &src) -> int {
        std::vector<T> tv(src.begin(), src.end());
        int r = h->alloc(dst, tv.size() * sizeof(T));
        if (r) return r;
        return upload(h, *dst, tv.data(), tv.size() * sizeof(T));
    };
    auto up_int = [&](int **dst, const std::vector<int> &src) -> int {
        int r = h->alloc(dst, src.size() * sizeof(int));
        if (r) return r;
        return upload(h, *dst, src.data(), src.size() * sizeof(int));
    };
    if (h->layout == SS_LAYOUT_CSR) {
        if ((rc = up_int(&h->row, h->lay.row))) return rc;
        if ((rc = h->alloc(&h->inc, h->lay.inc.size() * sizeof(int2)))) return rc;
        if ((rc = upload(h, h->inc, h->lay.inc.data(), h->lay.inc.size() * sizeof(int2)))) return rc;
        std::vector<double> kv(d->k, d->k + S), lv(d->l0, d->l0 + S);
        if ((rc = up_typed(&h->k, kv))) return rc;
        if ((rc = up_typed(&h->l0, lv))) return rc;
        if (d->group && h->groups.size()) {
            std::vector<int> g(d->group, d->group + S);
            if ((rc = up_int(&h->grp, g))) return rc;
        }
    } else {
        const auto &L = h->lay;
        std::vector<double> ek(L.e_spring.size(), 0.0), el(L.e_spring.size(), 0.0);
        std::vector<int> eg;
        const bool has_g = d->group && h->groups.size();
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
    return SS_OK;
}

int64_t algorithmic_bytes(const ss_engine *h) {
    // fp32 16 B/spring + 64 B/mass; fp64 24 B/spring + 128 B/mass.
    const int64_t per_spring = h->precision == SS_F32 ? 16 : 24;
    const int64_t per_mass = h->precision == SS_F32 ? 64 : 128;
    return per_spring * h->S + per_mass * h->N;
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
    int rc;
    if ((rc = h->alloc(&h->d_degenerate, sizeof(unsigned long long)))) return rc;
    if ((rc = h->alloc(&h->d_div_step, sizeof(long long)))) return rc;
    if ((rc = h->alloc(&h->d_div_mass, sizeof(int)))) return rc;
    CK(cudaMemsetAsync(h->d_degenerate, 0, sizeof(unsigned long long), h->stream));
    if ((rc = reset_divergence(h.get()))) return rc;
    rc = h->precision == SS_F32 ? create_impl<true>(h.get(), d) : create_impl<false>(h.get(), d);
    if (rc) {
        std::lock_guard<std::mutex> lk(g_base_mu);
        g_base.erase(h.get());
        return rc;
    }
    CK(cudaStreamSynchronize(h->stream));
    *out = h.release();
    return SS_OK;
}

int ss_destroy(ss_engine *h) {
    if (!h) return SS_OK;
    {
        std::lock_guard<std::mutex> lk(g_base_mu);
        g_base.erase(h);
    }
    delete h;
    return SS_OK;
}

int ss_step(ss_engine *h, int64_t count, ss_step_result *res) {
    if (!h) return ss::fail(SS_EINVAL, "null engine");
    CK(cudaSetDevice(h->device));
    if (h->pending) {
        int rc = ss_sync(h, nullptr);
        if (rc) return rc;
    }
    if (count <= 0) {
        if (res) *res = {0, h->n, h->t, -1, -1};
        return SS_OK;
    }
    const int64_t n0 = h->n;
    const int cur0 = h->cur;
    const bool had_prev = h->has_prev;
    int rc = dispatch_steps(h, count);
    if (rc) return rc;
    rc = finish_batch(h, count, n0, cur0, res);
    if (rc == SS_EDIVERGED && h->integrator == SS_VERLET) {
        // history exists iff at least one step committed
        h->has_prev = had_prev || (h->n > n0);
    }
    return rc;
}

int ss_step_async(ss_engine *h, int64_t count) {
    if (!h) return ss::fail(SS_EINVAL, "null engine");
    if (count <= 0) return SS_OK;
    CK(cudaSetDevice(h->device));
    if (!h->pending) {
        h->pending_n0 = h->n;
        h->pending_cur0 = h->cur;
        h->pending_t0 = h->t;
    }
    // time bookkeeping for the scale table: advance n/t as if committed
    int rc = dispatch_steps(h, count);
    if (rc) return rc;
    h->pending += count;
    h->n += count;
    h->t = (double)h->n * h->dt;
    return SS_OK;
}

int ss_sync(ss_engine *h, ss_step_result *res) {
    if (!h) return ss::fail(SS_EINVAL, "null engine");
    CK(cudaSetDevice(h->device));
    const int64_t count = h->pending;
    h->pending = 0;
    if (count == 0) {
        CK(cudaStreamSynchronize(h->stream));
        if (res) *res = {0, h->n, h->t, -1, -1};
        return SS_OK;
    }
    return finish_batch(h, count, h->pending_n0, h->pending_cur0, res);
}

void *ss_stream(ss_engine *h) { return h ? (void *)h->stream : nullptr; }

int ss_forces(ss_engine *h, const double *x, const double *v, double t, double *acc_out,
              int64_t *degenerate_out) {
    if (!h || !x || !v || !acc_out) return ss::fail(SS_EINVAL, "ss_forces: null argument");
    CK(cudaSetDevice(h->device));
    if (h->pending) {
        int rc = ss_sync(h, nullptr);
        if (rc) return rc;
    }
    int rc;
    const size_t vec = h->precision == SS_F32 ? sizeof(float4) : sizeof(double4);
    for (int b = 0; b < 2; ++b)
        if (!h->d_tmp[b] && (rc = h->alloc(&h->d_tmp[b], (size_t)h->N * vec))) return rc;
    if (!h->d_acc && (rc = h->alloc(&h->d_acc, (size_t)h->N * 3 * sizeof(double)))) return rc;
    unsigned long long before = 0;
    CK(cudaMemcpy(&before, h->d_degenerate, sizeof before, cudaMemcpyDeviceToHost));
    // scale table at time t
    std::vector<double> tab;
    if (!h->groups.empty()) {
        ss_engine tmp_view = {};
        (void)tmp_view;
        const size_t G = h->groups.size();
        tab.resize(G);
        for (size_t g = 0; g < G; ++g) {
            const Group &gr = h->groups[g];
            tab[g] = gr.mode == SS_CONSTANT_EXPANSION
                         ? 1.0 + gr.amplitude
                         : 1.0 + gr.amplitude * std::sin(2.0 * M_PI * gr.frequency * t + gr.phase);
        }
    }
    const int grid = (int)((h->N + kBlock - 1) / kBlock);
    if (h->precision == SS_F32) {
        if ((rc = upload_scales<float>(h, tab))) return rc;
        std::vector<float4> tx((size_t)h->N), tv((size_t)h->N);
        pack_positions<float, float4>(h, x, host_base(h), tx.data());
        pack_vec<float, float4>(h->N, v, tv.data());
        if ((rc = upload(h, h->d_tmp[0], tx.data(), tx.size() * sizeof(float4)))) return rc;
        if ((rc = upload(h, h->d_tmp[1], tv.data(), tv.size() * sizeof(float4)))) return rc;
        Params<float> p = base_params<float>(h);
        p.X = (const float4 *)h->d_tmp[0];
        p.V = (const float4 *)h->d_tmp[1];
        p.scale = tab.empty() ? nullptr : (const float *)h->scale;
        p.acc_out = (V3<double> *)h->d_acc;
        if (h->layout == SS_LAYOUT_ELL) forces_kernel<true, 2><<<grid, kBlock, 0, h->stream>>>(p);
        else forces_kernel<true, 1><<<grid, kBlock, 0, h->stream>>>(p);
    } else {
        if ((rc = upload_scales<double>(h, tab))) return rc;
        std::vector<double4> tx((size_t)h->N), tv((size_t)h->N);
        pack_positions<double, double4>(h, x, nullptr, tx.data());
        pack_vec<double, double4>(h->N, v, tv.data());
        if ((rc = upload(h, h->d_tmp[0], tx.data(), tx.size() * sizeof(double4)))) return rc;
        if ((rc = upload(h, h->d_tmp[1], tv.data(), tv.size() * sizeof(double4)))) return rc;
        Params<double> p = base_params<double>(h);
        p.X = (const double4 *)h->d_tmp[0];
        p.V = (const double4 *)h->d_tmp[1];
        p.scale = tab.empty() ? nullptr : (const double *)h->scale;
        p.acc_out = (V3<double> *)h->d_acc;
        if (h->layout == SS_LAYOUT_ELL) forces_kernel<false, 2><<<grid, kBlock, 0, h->stream>>>(p);
        else forces_kernel<false, 1><<<grid, kBlock, 0, h->stream>>>(p);
    }
    h->launches += 1;
    CK(cudaGetLastError());
    if ((rc = download(h, acc_out, h->d_acc, (size_t)h->N * 3 * sizeof(double)))) return rc;
    unsigned long long after = 0;
    CK(cudaMemcpy(&after, h->d_degenerate, sizeof after, cudaMemcpyDeviceToHost));
    if (degenerate_out) *degenerate_out = (int64_t)(after - before);
    return SS_OK;
}

int ss_get_state(ss_engine *h, double *x, double *v, double *x_prev, int *has_prev) {
    if (!h) return ss::fail(SS_EINVAL, "null engine");
    CK(cudaSetDevice(h->device));
    if (h->pending) {
        int rc = ss_sync(h, nullptr);
        if (rc && rc != SS_EDIVERGED) return rc;
    }
    int rc;
    const int64_t N = h->N;
    if (has_prev) *has_prev = h->has_prev ? 1 : 0;
    if (h->precision == SS_F32) {
        std::vector<float4> tmp((size_t)N);
        const float *base = host_base(h);
        if (x) {
            if ((rc = download(h, tmp.data(), h->X[h->cur], N * sizeof(float4)))) return rc;
            unpack_positions<float, float4>(h, tmp.data(), base, x);
        }
        if (v) {
            if ((rc = download(h, tmp.data(), h->V, N * sizeof(float4)))) return rc;
            unpack_vec<float, float4>(N, tmp.data(), v);
        }
        if (x_prev && h->has_prev) {
            if ((rc = download(h, tmp.data(), h->X[h->cur ^ 1], N * sizeof(float4)))) return rc;
            unpack_positions<float, float4>(h, tmp.data(), base, x_prev);
        }
    } else {
        std::vector<double4> tmp((size_t)N);
        if (x) {
            if ((rc = download(h, tmp.data(), h->X[h->cur], N * sizeof(double4)))) return rc;
            unpack_positions<double, double4>(h, tmp.data(), nullptr, x);
        }
        if (v) {
            if ((rc = download(h, tmp.data(), h->V, N * sizeof(double4)))) return rc;
            unpack_vec<double, double4>(N, tmp.data(), v);
        }
        if (x_prev && h->has_prev) {
            if ((rc = download(h, tmp.data(), h->X[h->cur ^ 1], N * sizeof(double4)))) return rc;
            unpack_positions<double, double4>(h, tmp.data(), nullptr, x_prev);
        }
    }
    return SS_OK;
}

int ss_get_positions(ss_engine *h, double *x) { return ss_get_state(h, x, nullptr, nullptr, nullptr); }

int ss_set_state(ss_engine *h, const double *x, const double *v, const double *x_prev) {
    if (!h) return ss::fail(SS_EINVAL, "null engine");
    CK(cudaSetDevice(h->device));
    if (h->pending) {
        int rc = ss_sync(h, nullptr);
        if (rc && rc != SS_EDIVERGED) return rc;
    }
    int rc;
    const int64_t N = h->N;
    if (h->precision == SS_F32) {
        std::vector<float4> tmp((size_t)N);
        const float *base = host_base(h);
        if (x) {
            pack_positions<float, float4>(h, x, base, tmp.data());
            if ((rc = upload(h, h->X[h->cur], tmp.data(), N * sizeof(float4)))) return rc;
        }
        if (v) {
            pack_vec<float, float4>(N, v, tmp.data());
            if ((rc = upload(h, h->V, tmp.data(), N * sizeof(float4)))) return rc;
        }
        if (x_prev) {
            pack_positions<float, float4>(h, x_prev, base, tmp.data());
            if ((rc = upload(h, h->X[h->cur ^ 1], tmp.data(), N * sizeof(float4)))) return rc;
        }
    } else {
        std::vector<double4> tmp((size_t)N);
        if (x) {
            pack_positions<double, double4>(h, x, nullptr, tmp.data());
            if ((rc = upload(h, h->X[h->cur], tmp.data(), N * sizeof(double4)))) return rc;
        }
        if (v) {
            pack_vec<double, double4>(N, v, tmp.data());
            if ((rc = upload(h, h->V, tmp.data(), N * sizeof(double4)))) return rc;
        }
        if (x_prev) {
            pack_positions<double, double4>(h, x_prev, nullptr, tmp.data());
            if ((rc = upload(h, h->X[h->cur ^ 1], tmp.data(), N * sizeof(double4)))) return rc;
        }
    }
    if (x_prev) h->has_prev = true;
    return SS_OK;
}

int ss_clear_prev(ss_engine *h) {
    if (!h) return ss::fail(SS_EINVAL, "null engine");
    if (h->pending) {
        int rc = ss_sync(h, nullptr);
        if (rc && rc != SS_EDIVERGED) return rc;
    }
    h->has_prev = false;
    return SS_OK;
}

int ss_get_time(ss_engine *h, double *t, int64_t *n) {
    if (!h) return ss::fail(SS_EINVAL, "null engine");
    if (t) *t = h->t;
    if (n) *n = h->n;
    return SS_OK;
}

int ss_set_time(ss_engine *h, double t, int64_t n) {
    if (!h) return ss::fail(SS_EINVAL, "null engine");
    if (h->pending) {
        int rc = ss_sync(h, nullptr);
        if (rc && rc != SS_EDIVERGED) return rc;
    }
    h->t = t;
    h->n = n;
    return SS_OK;
}

int ss_set_f_ext(ss_engine *h, const double *f) {
    if (!h || !f) return ss::fail(SS_EINVAL, "ss_set_f_ext: null argument");
    CK(cudaSetDevice(h->device));
    if (h->pending) {
        int rc = ss_sync(h, nullptr);
        if (rc && rc != SS_EDIVERGED) return rc;
    }
    bool any = false;
    for (int64_t i = 0; i < 3 * h->N && !any; ++i) any = f[i] != 0.0;
    h->has_fext = any;
    if (h->precision == SS_F32) {
        std::vector<float4> tmp((size_t)h->N);
        pack_vec<float, float4>(h->N, f, tmp.data());
        return upload(h, h->F, tmp.data(), h->N * sizeof(float4));
    }
    std::vector<double4> tmp((size_t)h->N);
    pack_vec<double, double4>(h->N, f, tmp.data());
    return upload(h, h->F, tmp.data(), h->N * sizeof(double4));
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
    info->n_masses = h->N;
    info->n_springs = h->S;
    info->precision = h->precision;
    info->layout = h->layout;
    info->integrator = h->integrator;
    info->device = h->device;
    info->device_bytes = h->device_bytes;
    info->algorithmic_bytes_per_step = (double)algorithmic_bytes(h);
    info->ell_width_own = h->lay.W;
    info->ell_width_ref = h->lay.Wr;
    info->canonical_order = h->lay.canonical ? 1 : 0;
    return SS_OK;
}

int64_t ss_launch_count(ss_engine *h) { return h ? h->launches : 0; }

}  // extern "C"
