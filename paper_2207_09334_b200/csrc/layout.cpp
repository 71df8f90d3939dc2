// Incidence layouts for the mass-centric gather.
//
// The reference accumulates spring forces in spring-id order
// (_kernels.py:51-70); parallel-det mode reproduces that per mass by sorting
// slots by spring id (_kernels.py:128-144).  Both layouts below encode, per
// mass, a fixed summation order equal to that spring-id order, so fp64 sums
// are bitwise identical to the serial oracle.
//
// CSR: per mass, (other endpoint, spring id) in spring-id order.  Any graph.
//
// ELL: each spring is stored once, in the row of its lower-id endpoint (its
// "owner"), in sliced-ELL order (32 masses per slice, position
// (slice*W + q)*32 + lane, so the q-th record of 32 consecutive masses is one
// 128-byte line per field).  The other endpoint reaches the record through a
// 4-byte reverse reference.  For a mass whose incident springs with a lower
// partner all precede those with a higher partner in id order ("canonical":
// always true for lattice builders, which sort springs by (i, j),
// lattice.py:133-134) the kernel sums refs then own records; for any other
// mass every incidence is emitted as a ref in spring-id order, so the
// result is still exact.
//
// DRAM bytes per spring per step (fp32): 12 B own record + 4 B ref = 16 B,
// the SURVEY §8d algorithmic figure; the ref's second touch of the record is
// an L2 hit because the owner's warp streamed it moments earlier.

#include "layout.h"

#include <algorithm>
#include <cstring>

#include "common.h"
#include "springsim_b200.h"

namespace ss {

static int build_csr(const LayoutInput &in, Layout &L) {
    const int64_t N = in.N, S = in.S;
    L.kind = SS_LAYOUT_CSR;
    L.row.assign((size_t)N + 1, 0);
    for (int64_t s = 0; s < S; ++s) {
        L.row[in.si[s] + 1]++;
        L.row[in.sj[s] + 1]++;
    }
    for (int64_t m = 0; m < N; ++m) L.row[m + 1] += L.row[m];
    L.inc.resize((size_t)2 * S);
    std::vector<int> cur(L.row.begin(), L.row.end() - 1);
    for (int64_t s = 0; s < S; ++s) {   // ascending s => rows sorted by spring id
        const int i = (int)in.si[s], j = (int)in.sj[s];
        L.inc[cur[i]++] = make_int2(j, (int)s);
        L.inc[cur[j]++] = make_int2(i, (int)s);
    }
    return SS_OK;
}

static int build_ell(const LayoutInput &in, Layout &L) {
    const int64_t N = in.N, S = in.S;
    L.kind = SS_LAYOUT_ELL;
    std::vector<int> n_own((size_t)N, 0), n_low((size_t)N, 0);
    for (int64_t s = 0; s < S; ++s) {
        const int64_t a = std::min(in.si[s], in.sj[s]), b = std::max(in.si[s], in.sj[s]);
        n_own[a]++;
        n_low[b]++;
    }
    // canonical per mass: max id of springs where m is the upper endpoint
    // < min id of springs m owns.
    std::vector<int64_t> max_ref((size_t)N, -1), min_own((size_t)N, INT64_MAX);
    for (int64_t s = 0; s < S; ++s) {
        const int64_t a = std::min(in.si[s], in.sj[s]), b = std::max(in.si[s], in.sj[s]);
        if (s < min_own[a]) min_own[a] = s;
        if (s > max_ref[b]) max_ref[b] = s;
    }
    std::vector<char> canon((size_t)N);
    int W = 1, Wr = 1;
    L.canonical = true;
    for (int64_t m = 0; m < N; ++m) {
        canon[m] = max_ref[m] < min_own[m];
        if (!canon[m]) L.canonical = false;
        W = std::max(W, n_own[m]);
        const int nref = canon[m] ? n_low[m] : n_low[m] + n_own[m];
        Wr = std::max(Wr, nref);
        if (n_own[m] >= 65536 || nref >= 65536)
            return fail(SS_EINVAL, "mass %lld has too many springs for the ELL layout", (long long)m);
    }
    L.W = W;
    L.Wr = Wr;
    L.slices = (N + 31) / 32;
    const size_t own_sz = (size_t)L.slices * W * 32, ref_sz = (size_t)L.slices * Wr * 32;
    if (own_sz >= (size_t)INT32_MAX || ref_sz >= (size_t)INT32_MAX)
        return fail(SS_EINVAL, "ELL layout exceeds 2^31 entries");
    L.e_other.assign(own_sz, 0);
    L.e_spring.assign(own_sz, -1);
    L.r_pos.assign(ref_sz, -1);
    L.cnt.assign((size_t)N, 0);
    auto own_pos = [&](int64_t m, int q) -> int64_t { return ((m >> 5) * W + q) * 32 + (m & 31); };
    auto ref_pos = [&](int64_t m, int q) -> int64_t { return ((m >> 5) * Wr + q) * 32 + (m & 31); };
    std::vector<int> oc((size_t)N, 0), rc((size_t)N, 0);
    for (int64_t s = 0; s < S; ++s) {   // ascending s => every list in spring-id order
        const int64_t a = std::min(in.si[s], in.sj[s]), b = std::max(in.si[s], in.sj[s]);
        const int64_t p = own_pos(a, oc[a]++);
        L.e_other[p] = (int)b;
        L.e_spring[p] = s;
        if (!canon[a]) L.r_pos[ref_pos(a, rc[a]++)] = (int)p;   // own record referenced in order
        L.r_pos[ref_pos(b, rc[b]++)] = (int)p;
    }
    for (int64_t m = 0; m < N; ++m)
        L.cnt[m] = (canon[m] ? oc[m] : 0) | (rc[m] << 16);
    return SS_OK;
}

int build_layout(const LayoutInput &in, int want, Layout &out) {
    out = Layout{};
    if (want == SS_LAYOUT_CSR) return build_csr(in, out);
    if (want == SS_LAYOUT_ELL) return build_ell(in, out);
    // AUTO: ELL unless its padding more than doubles the record storage.
    int rc = build_ell(in, out);
    if (rc == SS_OK) {
        const double used = (double)in.S;
        const double padded = (double)out.slices * out.W * 32;
        if (in.S == 0 || padded <= 2.0 * used + 64.0 * 32.0) return SS_OK;
    }
    out = Layout{};
    return build_csr(in, out);
}

}  // namespace ss
