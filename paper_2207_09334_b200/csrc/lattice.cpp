// Array-native voxel lattice builder (host, C++/OpenMP).
//
// Restates build_voxel_lattice (reference lattice.py:89-136) for box meshes
// without the Python object model:
//   counts = floor((hi-lo)/dim + 1e-9) + 1                 (lattice.py:104-107)
//   node (i,j,k) -> id (i*ny + j)*nz + k, x = lo + idx*dim  (lattice.py:109-119)
//   springs = the unique unordered pairs of nodes sharing a cell, i.e. the
//   26-neighbour stencil, sorted by (min id, max id)        (lattice.py:121-134)
//   l0 = np.linalg.norm(x_b - x_a) = OpenBLAS ddot = sqrt(fma(dz,dz,fma(dy,dy,dx*dx)))
//                                                         (lattice.py:84)
//   k  = (k0 * l_ref) / l0                                  (model.py:87-92)
// Every grid node of a box lies inside or on box_mesh's surface, so no node
// is culled (mesh.py:75-132 counts on-surface points as inside).
//
// Because springs come out sorted by (i, j), mass a's "upper" springs are the
// 13 forward stencil offsets in increasing linear offset, and the id of each
// spring is (#upper springs of all masses < a) + its rank: both computed in
// closed form so a spatial slab can be emitted with global ids.

#include <cmath>
#include <cstdint>
#include <cstring>
#include <algorithm>
#include <vector>
#include <string>

#include "springsim_b200.h"
#include "common.h"

namespace {

struct Offset { int di, dj, dk; int64_t lin; };

// The 13 neighbour offsets with positive linear offset, sorted ascending.
std::vector<Offset> upper_offsets(int64_t ny, int64_t nz) {
    std::vector<Offset> out;
    for (int di = -1; di <= 1; ++di)
        for (int dj = -1; dj <= 1; ++dj)
            for (int dk = -1; dk <= 1; ++dk) {
                int64_t lin = (int64_t)di * ny * nz + (int64_t)dj * nz + dk;
                if (lin > 0) out.push_back({di, dj, dk, lin});
            }
    std::stable_sort(out.begin(), out.end(),
                     [](const Offset &a, const Offset &b) { return a.lin < b.lin; });
    return out;
}

inline bool inb(int64_t v, int64_t n) { return v >= 0 && v < n; }

}  // namespace

extern "C" int ss_lattice_box(const double lo[3], const double hi[3], double dim,
                              double k0, double l_ref,
                              int64_t i_lo, int64_t i_hi,
                              int64_t counts_out[3], int64_t *n_masses_out,
                              int64_t *n_springs_out,
                              double *x_out, int64_t *si_out, int64_t *sj_out,
                              double *k_out, double *l0_out, int64_t *spring_id_out) {
    if (!lo || !hi || !(dim > 0.0)) return ss::fail(SS_EINVAL, "ss_lattice_box: need lo, hi and dim > 0");
    int64_t c[3];
    for (int a = 0; a < 3; ++a) {
        if (!(hi[a] > lo[a])) return ss::fail(SS_EINVAL, "box must have positive extent on every axis");
        const double q = (hi[a] - lo[a]) / dim;   // built with -ffp-contract=off
        const double q2 = q + 1e-9;
        c[a] = (int64_t)std::floor(q2) + 1;
    }
    const int64_t nx = c[0], ny = c[1], nz = c[2];
    if (counts_out) { counts_out[0] = nx; counts_out[1] = ny; counts_out[2] = nz; }
    if (i_hi <= i_lo) { i_lo = 0; i_hi = nx; }
    i_lo = std::max<int64_t>(0, i_lo);
    i_hi = std::min<int64_t>(nx, i_hi);
    if (i_hi <= i_lo) return ss::fail(SS_EINVAL, "empty slab");

    const auto offs = upper_offsets(ny, nz);
    const int64_t plane = ny * nz;

    // upper degree of node (i,j,k)
    auto updeg = [&](int64_t i, int64_t j, int64_t k) {
        int d = 0;
        for (const auto &o : offs)
            d += inb(i + o.di, nx) && inb(j + o.dj, ny) && inb(k + o.dk, nz);
        return d;
    };
    // springs whose lower endpoint lies in plane i: same for every interior plane
    auto plane_springs = [&](int64_t i) {
        int64_t s = 0;
        for (int64_t j = 0; j < ny; ++j)
            for (int64_t k = 0; k < nz; ++k) s += updeg(i, j, k);
        return s;
    };
    const int64_t s_first = plane_springs(0);
    const int64_t s_mid = nx > 2 ? plane_springs(1) : 0;
    const int64_t s_last = nx > 1 ? plane_springs(nx - 1) : 0;
    auto springs_before_plane = [&](int64_t i) -> int64_t {   // ids of springs with lower endpoint in planes < i
        if (i <= 0) return 0;
        int64_t s = s_first;                                  // plane 0
        if (i - 1 >= 1) s += (std::min(i, nx - 1) - 1) * s_mid;  // planes 1 .. min(i,nx-1)-1
        if (i == nx) s += (nx > 1 ? s_last : 0);
        return s;
    };
    const int64_t total_springs = springs_before_plane(nx);

    // slab: masses in planes [i_lo, i_hi); springs with >=1 endpoint there.
    // Lower endpoints of those springs lie in planes [i_lo-1, i_hi).
    const int64_t m_lo = i_lo * plane, m_hi = i_hi * plane;
    const int64_t p_lo = std::max<int64_t>(0, i_lo - 1);
    const int64_t n_masses = m_hi - m_lo;

    // per-plane emitted counts (for the lower-neighbour plane only springs
    // reaching into the slab are emitted)
    std::vector<int64_t> pcount(i_hi - p_lo + 1, 0);
    for (int64_t i = p_lo; i < i_hi; ++i) {
        int64_t s = 0;
        if (i >= i_lo) {
            s = (i == 0) ? s_first : (i == nx - 1 ? s_last : s_mid);
            if (nx == 1) s = s_first;
        } else {  // plane i_lo-1: only offsets with di == 1
            for (int64_t j = 0; j < ny; ++j)
                for (int64_t k = 0; k < nz; ++k)
                    for (const auto &o : offs)
                        s += o.di == 1 && inb(i + 1, nx) && inb(j + o.dj, ny) && inb(k + o.dk, nz);
        }
        pcount[i - p_lo + 1] = s;
    }
    for (size_t q = 1; q < pcount.size(); ++q) pcount[q] += pcount[q - 1];
    const int64_t n_springs = pcount.back();
    if (n_masses_out) *n_masses_out = n_masses;
    if (n_springs_out) *n_springs_out = n_springs;
    (void)total_springs;
    if (!x_out && !si_out) return SS_OK;   // size query

    if (x_out) {
#pragma omp parallel for schedule(static)
        for (int64_t a = m_lo; a < m_hi; ++a) {
            int64_t i = a / plane, j = (a / nz) % ny, k = a % nz;
            const int64_t idx[3] = {i, j, k};
            for (int d = 0; d < 3; ++d) {
                const double step = (double)idx[d] * dim;
                x_out[(a - m_lo) * 3 + d] = lo[d] + step;
            }
        }
    }
    if (!si_out) return SS_OK;

#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t i = p_lo; i < i_hi; ++i) {
        int64_t w = pcount[i - p_lo];                 // emit cursor
        int64_t gid = springs_before_plane(i);        // global id cursor
        const bool halo_plane = i < i_lo;
        for (int64_t j = 0; j < ny; ++j)
            for (int64_t k = 0; k < nz; ++k) {
                const int64_t a = (i * ny + j) * nz + k;
                double xa[3] = {lo[0] + (double)i * dim, lo[1] + (double)j * dim,
                                lo[2] + (double)k * dim};
                for (const auto &o : offs) {
                    int64_t bi = i + o.di, bj = j + o.dj, bk = k + o.dk;
                    if (!(inb(bi, nx) && inb(bj, ny) && inb(bk, nz))) continue;
                    const int64_t id = gid++;
                    if (halo_plane && o.di != 1) continue;
                    const int64_t b = a + o.lin;
                    double xb[3] = {lo[0] + (double)bi * dim, lo[1] + (double)bj * dim,
                                    lo[2] + (double)bk * dim};
                    const double dx = xb[0] - xa[0], dy = xb[1] - xa[1], dz = xb[2] - xa[2];
                    double l0 = std::sqrt(std::fma(dz, dz, std::fma(dy, dy, dx * dx)));
                    const double kk = k0 * l_ref;
                    si_out[w] = a;
                    sj_out[w] = b;
                    if (l0_out) l0_out[w] = l0;
                    if (k_out) k_out[w] = kk / l0;
                    if (spring_id_out) spring_id_out[w] = id;
                    ++w;
                }
            }
    }
    return SS_OK;
}
