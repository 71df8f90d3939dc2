// Host builder of the fp64 (bit-parity) tiled incidence layout;
// fp32 builds are dispatched to tiles_f32.cpp.
//
// Masses are renumbered into 4x8x8 bricks of the lattice (generic scenes:
// bricks of quantised coordinates), and consecutive runs of kTile=256 new
// ids form a tile, processed by one CTA.  Each spring is owned by its
// endpoint with the lower ORIGINAL id and stored once, in the owner's tile,
// as a record (other-endpoint local index u16, k, l0[, group]) in
// sliced-ELL order.  The other endpoint reaches it through a 2-byte
// reference: a slot in the same tile's record array, or (owner outside the
// tile) an entry of the tile's short "foreign" record list.  Per mass the
// kernel sums references then own records, both in ascending spring id —
// the reference's serial summation order (_kernels.py:51-70) for every
// "canonical" mass; a non-canonical mass lists all its incidences as
// references in spring-id order.  The tile's halo (partners outside the
// tile) is a list of global ids whose states the CTA stages into shared
// memory once, so the hot loop reads nothing but shared memory.
//
// DRAM bytes per spring ~ 10 (own record) + 2 (ref) + ~0.3 x 10 (foreign
// copy) + halo ids ~ 16 B in fp32: the SURVEY §8d algorithmic figure.

#include "tiles.h"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <tuple>

#include "common.h"
#include "springsim_b200.h"

namespace ss {

namespace {

inline uint32_t align16(uint32_t v) { return (v + 15u) & ~15u; }

}  // namespace

// Device slot order: tile t owns slots [256t, 256t+256); real masses fill a
// tile's first n slots, the rest are padding (-1).  With order == 1 the
// masses are sorted into 4x8x8 bricks of quantised coordinates and whole
// bricks are packed into tiles, so tiles never straddle brick boundaries.
void tile_order(const TileInput &in, std::vector<int32_t> &orig_of, std::vector<int32_t> *zcell) {
    const int64_t N = in.N;
    std::vector<int32_t> sorted(N);
    std::iota(sorted.begin(), sorted.end(), 0);
    std::vector<uint64_t> brick_of;
    bool bricks = false;
    if (in.order == 1 && in.x && N > kTile) {
        // cell size: shortest spring (the lattice pitch for voxel lattices)
        double h = INFINITY;
        for (int64_t s = 0; s < in.S; ++s) {
            const double *a = in.x + 3 * in.si[s], *b = in.x + 3 * in.sj[s];
            const double d = std::sqrt((b[0] - a[0]) * (b[0] - a[0]) + (b[1] - a[1]) * (b[1] - a[1]) +
                                       (b[2] - a[2]) * (b[2] - a[2]));
            if (d > 0 && d < h) h = d;
        }
        if (h > 0 && std::isfinite(h)) {
            double lo[3] = {INFINITY, INFINITY, INFINITY};
            for (int64_t i = 0; i < N; ++i)
                for (int c = 0; c < 3; ++c) lo[c] = std::min(lo[c], in.x[3 * i + c]);
            std::vector<int64_t> cell((size_t)N * 3);
            if (zcell) zcell->assign(N, 0);
            int64_t mx[3] = {0, 0, 0};
            for (int64_t i = 0; i < N; ++i)
                for (int c = 0; c < 3; ++c) {
                    const double q = std::floor((in.x[3 * i + c] - lo[c]) / h + 0.5);
                    const int64_t v = q < 0 ? 0 : (int64_t)q;
                    cell[3 * i + c] = v;
                    if (zcell && c == 2) (*zcell)[i] = (int32_t)(v & 0x7fffffff);
                    mx[c] = std::max(mx[c], v);
                }
            const int64_t B[3] = {4, 8, 8};
            const int64_t nb1 = mx[1] / B[1] + 1, nb2 = mx[2] / B[2] + 1;
            std::vector<uint64_t> key((size_t)N);
            brick_of.resize(N);
            for (int64_t i = 0; i < N; ++i) {
                const int64_t *c = &cell[3 * i];
                const uint64_t brick = ((uint64_t)(c[0] / B[0]) * nb1 + (uint64_t)(c[1] / B[1])) * nb2 +
                                       (uint64_t)(c[2] / B[2]);
                const uint64_t inner =
                    (uint64_t)((c[0] % B[0]) * B[1] + (c[1] % B[1])) * B[2] + (c[2] % B[2]);
                brick_of[i] = brick;
                key[i] = (brick << 8) | inner;
            }
            std::stable_sort(sorted.begin(), sorted.end(),
                             [&](int32_t a, int32_t b) { return key[a] < key[b]; });
            bricks = true;
        }
    }
    orig_of.clear();
    orig_of.reserve((size_t)N + N / 4 + kTile);
    auto pad_tile = [&]() {
        while (orig_of.size() % kTile) orig_of.push_back(-1);
    };
    if (!bricks) {
        orig_of.assign(sorted.begin(), sorted.end());
        pad_tile();
        return;
    }
    int64_t i = 0;
    while (i < N) {
        int64_t j = i;
        while (j < N && brick_of[sorted[j]] == brick_of[sorted[i]]) ++j;
        const int64_t size = j - i;
        const int64_t fill = (int64_t)(orig_of.size() % kTile);
        if (size > kTile) {
            pad_tile();
            for (int64_t q = i; q < j; ++q) orig_of.push_back(sorted[q]);
            pad_tile();
        } else {
            if (fill && fill + size > kTile) pad_tile();
            for (int64_t q = i; q < j; ++q) orig_of.push_back(sorted[q]);
        }
        i = j;
    }
    pad_tile();
}

namespace {

template <typename T>
void put(std::vector<uint8_t> &blob, uint32_t off, const T &v) {
    std::memcpy(blob.data() + off, &v, sizeof(T));
}

}  // namespace

// fp64 compact format (tiles.h): one incidence list per mass in ascending
// spring id -- the reference's serial summation order for every mass, no
// canonical-order condition -- of u16 = partner slot | dictionary index << 10
// over a per-tile dictionary of distinct (k, l0, group).  SS_EAGAIN_DICT when
// a tile does not fit (more than 64 dictionary entries, more than 768 halo
// slots, a mass of degree > 255, a self spring).
int build_tiles_f64_compact(const TileInput &in, TileLayout &L, bool inline_kl) {
    const int64_t N = in.N, S = in.S;
    if (N >= (1ll << 30) || S >= (1ll << 31)) return fail(SS_EINVAL, "scene too large for the tiled layout");
    for (int64_t s = 0; s < S; ++s)
        if (in.si[s] == in.sj[s]) return SS_EAGAIN_SHAPE;
    L = TileLayout{};
    std::vector<int32_t> zcell;
    tile_order(in, L.orig_of, &zcell);
    const char *bank_env = getenv("SS_TILE_BANK");           // 0: dense halo slots (A/B experiments)
    const bool bank_aware = !zcell.empty() && !(bank_env && atoi(bank_env) == 0);
    const int64_t D = (int64_t)L.orig_of.size();
    L.new_of.assign(N, -1);
    for (int64_t i = 0; i < D; ++i)
        if (L.orig_of[i] >= 0) L.new_of[L.orig_of[i]] = (int32_t)i;
    // incidences per device slot, ascending spring id
    std::vector<int64_t> ptr(D + 1, 0);
    for (int64_t s = 0; s < S; ++s) {
        ptr[L.new_of[in.si[s]] + 1]++;
        ptr[L.new_of[in.sj[s]] + 1]++;
    }
    for (int64_t m = 0; m < D; ++m) ptr[m + 1] += ptr[m];
    std::vector<int32_t> inc_s((size_t)2 * S), inc_o((size_t)2 * S);
    {
        std::vector<int64_t> fill(ptr.begin(), ptr.end() - 1);
        for (int64_t s = 0; s < S; ++s) {
            const int32_t a = L.new_of[in.si[s]], b = L.new_of[in.sj[s]];
            inc_s[fill[a]] = (int32_t)s;
            inc_o[fill[a]++] = b;
            inc_s[fill[b]] = (int32_t)s;
            inc_o[fill[b]++] = a;
        }
    }
    const int64_t n_tiles = D / kTile;
    L.n_tiles = n_tiles;
    std::vector<std::vector<uint8_t>> parts(n_tiles);
    std::vector<uint32_t> tW(n_tiles), tH(n_tiles), tSplit(n_tiles), tN(n_tiles);
    std::vector<double> tRatio(n_tiles);
    std::vector<std::vector<double>> tKL(inline_kl ? n_tiles : 0);
    std::vector<std::vector<int8_t>> tG(inline_kl && in.group ? n_tiles : 0);
    const bool has_g = in.group != nullptr;
    int err = 0;        // 3: a tile's shape does not fit (degree, halo); 4: its dictionary does not

#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t t = 0; t < n_tiles; ++t) {
        if (err) continue;
        const int64_t base = t * kTile;
        int n = 0;
        while (n < kTile && L.orig_of[base + n] >= 0) ++n;
        uint32_t W = 1;
        std::vector<int32_t> halo;
        for (int l = 0; l < n; ++l) {
            const int64_t m = base + l;
            W = std::max<uint32_t>(W, (uint32_t)(ptr[m + 1] - ptr[m]));
            for (int64_t q = ptr[m]; q < ptr[m + 1]; ++q)
                if (inc_o[q] < base || inc_o[q] >= base + n) halo.push_back(inc_o[q]);
        }
        std::sort(halo.begin(), halo.end());
        halo.erase(std::unique(halo.begin(), halo.end()), halo.end());
        // bank-aware halo slots (as tiles_f32.cpp): a halo mass sits at
        // 8 * (its rank among the halo masses of its z class) + (z mod 8), so
        // the partners of 8 consecutive z (one warp phase of a 16-byte
        // gather) land in 8 distinct bank groups; holes hold id -1
        std::vector<int32_t> halo_ids;
        std::vector<uint32_t> halo_slot(halo.size());
        uint32_t cnt[8] = {0, 0, 0, 0, 0, 0, 0, 0}, maxc = 0;
        std::vector<uint32_t> cls(halo.size());
        if (bank_aware) {
            for (size_t i = 0; i < halo.size(); ++i) cls[i] = cnt[zcell[L.orig_of[halo[i]]] & 7]++;
            for (int r = 0; r < 8; ++r) maxc = std::max(maxc, cnt[r]);
        }
        if (bank_aware && 8 * maxc <= 768) {          // (else: dense slots, the tile still fits)
            halo_ids.assign((size_t)8 * maxc, -1);
            for (size_t i = 0; i < halo.size(); ++i) {
                const uint32_t sl = 8 * cls[i] + ((uint32_t)zcell[L.orig_of[halo[i]]] & 7u);
                halo_ids[sl] = halo[i];
                halo_slot[i] = (uint32_t)kTile + sl;
            }
        } else {
            halo_ids = halo;
            for (size_t i = 0; i < halo.size(); ++i) halo_slot[i] = (uint32_t)(kTile + i);
        }
        if (W > 255 || halo_ids.size() > 768) {
#pragma omp atomic write
            err = 3;
            continue;
        }
        // dictionary of distinct (k, l0, group), in first-use order; inline
        // format: (k, l0) and the group per incidence instead
        std::vector<std::tuple<uint64_t, uint64_t, int32_t>> keys;
        std::vector<uint16_t> incs((size_t)W * kTile, 0);
        if (inline_kl) {
            tKL[t].assign((size_t)2 * W * kTile, 0.0);
            if (has_g) tG[t].assign((size_t)W * kTile, (int8_t)-1);
        }
        bool fits = true;
        for (int l = 0; l < n && fits; ++l) {
            const int64_t m = base + l;
            for (int64_t q = ptr[m]; q < ptr[m + 1]; ++q) {
                const int32_t s = inc_s[q], o = inc_o[q];
                const size_t at = (size_t)(q - ptr[m]) * kTile + l;
                size_t di = 0;
                if (inline_kl) {
                    tKL[t][2 * at] = in.k[s];
                    tKL[t][2 * at + 1] = in.l0[s];
                    if (has_g) tG[t][at] = (int8_t)in.group[s];
                } else {
                    uint64_t kb, lb;
                    std::memcpy(&kb, &in.k[s], 8);
                    std::memcpy(&lb, &in.l0[s], 8);
                    const auto key = std::make_tuple(kb, lb, has_g ? in.group[s] : -1);
                    while (di < keys.size() && keys[di] != key) ++di;
                    if (di == keys.size()) {
                        if (keys.size() == 64) { fits = false; break; }
                        keys.push_back(key);
                    }
                }
                const uint32_t slot = (o >= base && o < base + n)
                                          ? (uint32_t)(o - base)
                                          : halo_slot[std::lower_bound(halo.begin(), halo.end(), o) - halo.begin()];
                incs[at] = (uint16_t)(slot | (di << 10));
            }
        }
        if (!fits) {
            if (err != 3) {
#pragma omp atomic write
                err = 4;
            }
            continue;
        }
        const uint32_t nd = (uint32_t)keys.size();
        TileHdr h{};
        h.n = n; h.W = W; h.Wr = W; h.n_halo = (uint32_t)halo_ids.size();
        h.canonical = 1u | 2u | (inline_kl ? 4u : 0u);   // bit 1: compact format; bit 2: inline (k, l0)
        h.slice_log2 = 8;
        h.n_dict = nd;
        uint32_t off = align16(sizeof(TileHdr));
        h.off_halo = off; off = align16(off + (uint32_t)halo_ids.size() * 4);
        h.off_cnt = off;  off = align16(off + kTile * 2);
        h.off_oo = off;   off = align16(off + W * kTile * 2);
        h.off_okl = off;  off = align16(off + nd * 16);
        h.off_og = 0;
        if (has_g) { h.off_og = off; off = align16(off + nd); }
        h.off_ref = h.off_fo = h.off_fkl = h.off_fg = 0;
        h.bytes = off;
        std::vector<uint8_t> &blob = parts[t];
        blob.assign(off, 0);
        std::memcpy(blob.data(), &h, sizeof h);
        std::memcpy(blob.data() + h.off_halo, halo_ids.data(), halo_ids.size() * 4);
        for (int l = 0; l < n; ++l)
            put<uint16_t>(blob, h.off_cnt + 2 * l, (uint16_t)((ptr[base + l + 1] - ptr[base + l]) << 8));
        std::memcpy(blob.data() + h.off_oo, incs.data(), incs.size() * 2);
        for (uint32_t d = 0; d < nd; ++d) {
            uint64_t kb = std::get<0>(keys[d]), lb = std::get<1>(keys[d]);
            std::memcpy(blob.data() + h.off_okl + 16 * d, &kb, 8);
            std::memcpy(blob.data() + h.off_okl + 16 * d + 8, &lb, 8);
            if (has_g) put<int8_t>(blob, h.off_og + d, (int8_t)std::get<2>(keys[d]));
        }
        tW[t] = W; tH[t] = (uint32_t)halo_ids.size(); tN[t] = n;
        tSplit[t] = h.off_cnt | ((uint32_t)(n - 1) << 24);
        tRatio[t] = (double)(n + halo.size()) / n;
    }
    if (err == 3) return SS_EAGAIN_SHAPE;
    if (err) return SS_EAGAIN_DICT;
    if (in.group) {
        for (int64_t s = 0; s < S; ++s)
            if (in.group[s] > 127) return fail(SS_EINVAL, "at most 128 actuation groups in the tiled layout");
    }
    L.canonical = true;
    L.compact = true;
    L.inline_kl = inline_kl;
    if (inline_kl) {
        L.kl_off.assign(n_tiles + 1, 0);
        for (int64_t t = 0; t < n_tiles; ++t) L.kl_off[t + 1] = L.kl_off[t] + tKL[t].size() / 2;
        L.kl_inline.resize(2 * L.kl_off[n_tiles]);
        if (has_g) L.g_inline.resize(L.kl_off[n_tiles]);
#pragma omp parallel for schedule(static)
        for (int64_t t = 0; t < n_tiles; ++t) {
            std::memcpy(L.kl_inline.data() + 2 * L.kl_off[t], tKL[t].data(), tKL[t].size() * 8);
            if (has_g) std::memcpy(L.g_inline.data() + L.kl_off[t], tG[t].data(), tG[t].size());
        }
    }
    L.split = tSplit;
    L.off.assign(n_tiles + 1, 0);
    for (int64_t t = 0; t < n_tiles; ++t) L.off[t + 1] = L.off[t] + parts[t].size();
    L.blob.resize(L.off[n_tiles]);
#pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < n_tiles; ++t)
        std::memcpy(L.blob.data() + L.off[t], parts[t].data(), parts[t].size());
    double hsum = 0;
    for (int64_t t = 0; t < n_tiles; ++t) {
        L.max_tile_bytes = std::max<uint32_t>(L.max_tile_bytes, (uint32_t)parts[t].size());
        L.max_tile_smem = L.max_tile_bytes;
        const uint32_t head = tSplit[t] & 0xffffffu;
        L.max_head_bytes = std::max<uint32_t>(L.max_head_bytes, head);
        L.max_rest_bytes = std::max<uint32_t>(L.max_rest_bytes, (uint32_t)parts[t].size() - head);
        L.max_halo = std::max(L.max_halo, tH[t]);
        L.max_W = std::max<int>(L.max_W, (int)tW[t]);
        L.max_Wr = L.max_W;
        hsum += tRatio[t];
    }
    L.halo_ratio = hsum / (double)n_tiles;
    L.foreign_frac = 0.0;
    return SS_OK;
}

int build_tiles(const TileInput &in, TileLayout &L) {
    if (in.f32) return build_tiles_f32(in, L);
    {
        // SS_TILE_DICT: unset -> dictionary, else inline, else explicit;
        // "0" -> inline (the general-graph format); "explicit" -> explicit
        const char *env = getenv("SS_TILE_DICT");
        const bool explicit_only = env && std::strcmp(env, "explicit") == 0;
        const bool inline_only = env && !explicit_only && atoi(env) == 0;
        if (!explicit_only) {
            int rc = inline_only ? SS_EAGAIN_DICT : build_tiles_f64_compact(in, L, false);
            if (rc == SS_EAGAIN_DICT) rc = build_tiles_f64_compact(in, L, true);
            if (rc != SS_EAGAIN_DICT && rc != SS_EAGAIN_SHAPE) return rc;
        }
    }
    const int64_t N = in.N, S = in.S;
    if (N >= (1ll << 30) || S >= (1ll << 31)) return fail(SS_EINVAL, "scene too large for the tiled layout");
    L = TileLayout{};
    tile_order(in, L.orig_of);
    const int64_t D = (int64_t)L.orig_of.size();          // device slots, multiple of kTile
    L.new_of.assign(N, -1);
    for (int64_t i = 0; i < D; ++i)
        if (L.orig_of[i] >= 0) L.new_of[L.orig_of[i]] = (int32_t)i;

    // per-slot own / ref lists, each ascending in spring id
    std::vector<int64_t> own_ptr(D + 1, 0), ref_ptr(D + 1, 0);
    std::vector<int32_t> owner_new(S), other_new(S);
    for (int64_t s = 0; s < S; ++s) {
        const int64_t a = std::min(in.si[s], in.sj[s]), b = std::max(in.si[s], in.sj[s]);
        owner_new[s] = L.new_of[a];
        other_new[s] = L.new_of[b];
        own_ptr[owner_new[s] + 1]++;
        ref_ptr[other_new[s] + 1]++;
    }
    for (int64_t m = 0; m < D; ++m) {
        own_ptr[m + 1] += own_ptr[m];
        ref_ptr[m + 1] += ref_ptr[m];
    }
    std::vector<int32_t> own_sp(S), ref_sp(S);
    std::vector<uint8_t> q_of(S);
    {
        std::vector<int64_t> oc(own_ptr.begin(), own_ptr.end() - 1), rc(ref_ptr.begin(), ref_ptr.end() - 1);
        for (int64_t s = 0; s < S; ++s) {
            const int64_t o = owner_new[s];
            const int64_t q = oc[o] - own_ptr[o];
            if (q > 255) return fail(SS_EINVAL, "a mass owns more than 255 springs (tiled layout)");
            q_of[s] = (uint8_t)q;
            own_sp[oc[o]++] = (int32_t)s;
            ref_sp[rc[other_new[s]]++] = (int32_t)s;
        }
    }
    std::vector<uint8_t> canon(D);
    bool all_canon = true;
    for (int64_t m = 0; m < D; ++m) {
        const bool c = (ref_ptr[m + 1] == ref_ptr[m]) || (own_ptr[m + 1] == own_ptr[m]) ||
                       ref_sp[ref_ptr[m + 1] - 1] < own_sp[own_ptr[m]];
        canon[m] = c;
        all_canon = all_canon && c;
    }
    L.canonical = all_canon;
    for (int64_t s = 0; s < S && !L.has_self; ++s) L.has_self = in.si[s] == in.sj[s];

    const int64_t n_tiles = D / kTile;
    L.n_tiles = n_tiles;
    std::vector<std::vector<uint8_t>> parts(n_tiles);
    std::vector<uint32_t> tW(n_tiles), tWr(n_tiles), tH(n_tiles), tF(n_tiles), tSplit(n_tiles), tN(n_tiles);
    std::vector<int64_t> tRefs(n_tiles);
    const bool has_g = in.group != nullptr;
    const size_t rs = 8;                   // fp64 records (fp32 builds: tiles_f32.cpp)
    int err = 0;

#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t t = 0; t < n_tiles; ++t) {
        if (err) continue;
        const int64_t base = t * kTile;
        int n = 0;
        while (n < kTile && L.orig_of[base + n] >= 0) ++n;
        int W = 1, Wr = 1;
        std::vector<int32_t> halo;
        for (int l = 0; l < n; ++l) {
            const int64_t m = base + l;
            const int no = (int)(own_ptr[m + 1] - own_ptr[m]);
            const int nr = (int)(ref_ptr[m + 1] - ref_ptr[m]) + (canon[m] ? 0 : no);
            W = std::max(W, no);
            Wr = std::max(Wr, nr);
            for (int64_t q = own_ptr[m]; q < own_ptr[m + 1]; ++q) {
                const int32_t o = other_new[own_sp[q]];
                if (o < base || o >= base + n) halo.push_back(o);
            }
            for (int64_t q = ref_ptr[m]; q < ref_ptr[m + 1]; ++q) {
                const int32_t o = owner_new[ref_sp[q]];
                if (o < base || o >= base + n) halo.push_back(o);
            }
        }
        std::sort(halo.begin(), halo.end());
        halo.erase(std::unique(halo.begin(), halo.end()), halo.end());
        if (W > 127 || Wr > 255 || halo.size() + kTile > 65535) {
#pragma omp atomic write
            err = 1;
            continue;
        }
        auto local_of = [&](int32_t g) -> uint16_t {
            if (g >= base && g < base + n) return (uint16_t)(g - base);
            const auto it = std::lower_bound(halo.begin(), halo.end(), g);
            return (uint16_t)(kTile + (it - halo.begin()));
        };
        const uint32_t sl = 5u;                // 32-wide slices
        const int slices = (n + (1 << sl) - 1) >> sl;
        const uint32_t own_n = ((uint32_t)slices * W) << sl, ref_n = ((uint32_t)slices * Wr) << sl;
        // foreign references (owner outside the tile)
        std::vector<int32_t> foreign;          // spring ids
        std::vector<uint16_t> refs(ref_n, 0xffff);
        int64_t n_refs = 0;
        for (int l = 0; l < n; ++l) {
            const int64_t m = base + l;
            // merged list for non-canonical masses
            int q = 0;
            auto emit = [&](int32_t s) {
                const int32_t o = owner_new[s];
                uint16_t v;
                if (o >= base && o < base + n) {
                    v = (uint16_t)(((uint32_t)q_of[s] << 8) | (uint32_t)(o - base));
                } else {
                    v = (uint16_t)(0x8000 | foreign.size());
                    foreign.push_back(s);
                }
                refs[ell_slot(l, q, Wr, sl)] = v;
                ++q;
                ++n_refs;
            };
            if (canon[m]) {
                for (int64_t r = ref_ptr[m]; r < ref_ptr[m + 1]; ++r) emit(ref_sp[r]);
            } else {
                int64_t a = ref_ptr[m], b = own_ptr[m];
                while (a < ref_ptr[m + 1] || b < own_ptr[m + 1]) {
                    if (b >= own_ptr[m + 1] || (a < ref_ptr[m + 1] && ref_sp[a] < own_sp[b])) emit(ref_sp[a++]);
                    else emit(own_sp[b++]);
                }
            }
        }
        if (foreign.size() >= 0x8000) {
#pragma omp atomic write
            err = 2;
            continue;
        }
        const uint32_t nf = (uint32_t)foreign.size();
        bool tile_canon = true;
        for (int l = 0; l < n; ++l) tile_canon = tile_canon && canon[base + l];
        TileHdr h{};
        h.n = n; h.W = W; h.Wr = Wr; h.n_halo = (uint32_t)halo.size(); h.n_foreign = nf;
        h.canonical = tile_canon ? 1u : 0u;
        h.slice_log2 = sl;
        uint32_t off = align16(sizeof(TileHdr));
        h.off_halo = off; off = align16(off + (uint32_t)halo.size() * 4);
        h.off_cnt = off; off = align16(off + kTile * 2);
        h.off_oo = off;  off = align16(off + own_n * 2);
        h.off_okl = off; off = align16(off + own_n * 2 * rs);
        h.off_og = 0;
        if (has_g) { h.off_og = off; off = align16(off + own_n); }
        h.off_ref = off; off = align16(off + ref_n * 2);
        h.off_fo = off;  off = align16(off + nf * 2);
        h.off_fkl = off; off = align16(off + nf * 2 * rs);
        h.off_fg = 0;
        if (has_g) { h.off_fg = off; off = align16(off + nf); }
        h.bytes = off;
        std::vector<uint8_t> &blob = parts[t];
        blob.assign(off, 0);
        std::memcpy(blob.data(), &h, sizeof h);
        for (int l = 0; l < n; ++l) {
            const int64_t m = base + l;
            const int no = canon[m] ? (int)(own_ptr[m + 1] - own_ptr[m]) : 0;
            const int nr = (int)(ref_ptr[m + 1] - ref_ptr[m]) + (canon[m] ? 0 : (int)(own_ptr[m + 1] - own_ptr[m]));
            put<uint16_t>(blob, h.off_cnt + 2 * l, (uint16_t)(no | (nr << 8)));
            for (int64_t q = own_ptr[m]; q < own_ptr[m + 1]; ++q) {
                const int32_t s = own_sp[q];
                const uint32_t slot = ell_slot(l, (uint32_t)(q - own_ptr[m]), W, sl);
                put<uint16_t>(blob, h.off_oo + 2 * slot, local_of(other_new[s]));
                put<double>(blob, h.off_okl + 16 * slot, in.k[s]);
                put<double>(blob, h.off_okl + 16 * slot + 8, in.l0[s]);
                if (has_g) put<int8_t>(blob, h.off_og + slot, (int8_t)in.group[s]);
            }
        }
        std::memcpy(blob.data() + h.off_ref, refs.data(), refs.size() * 2);
        for (uint32_t f = 0; f < nf; ++f) {
            const int32_t s = foreign[f];
            put<uint16_t>(blob, h.off_fo + 2 * f, local_of(owner_new[s]));
            put<double>(blob, h.off_fkl + 16 * f, in.k[s]);
            put<double>(blob, h.off_fkl + 16 * f + 8, in.l0[s]);
            if (has_g) put<int8_t>(blob, h.off_fg + f, (int8_t)in.group[s]);
        }
        std::memcpy(blob.data() + h.off_halo, halo.data(), halo.size() * 4);
        tW[t] = W; tWr[t] = Wr; tH[t] = (uint32_t)halo.size(); tF[t] = nf; tRefs[t] = n_refs;
        tSplit[t] = h.off_cnt | ((uint32_t)(n - 1) << 24);   // n-1 in the top byte
        tN[t] = n;
    }
    if (err == 1) return fail(SS_EINVAL, "tile exceeds layout limits (degree or halo too large)");
    if (err == 2) return fail(SS_EINVAL, "tile has too many foreign references");
    if (in.group) {
        for (int64_t s = 0; s < S; ++s)
            if (in.group[s] > 127) return fail(SS_EINVAL, "at most 128 actuation groups in the tiled layout");
    }

    L.split = tSplit;
    L.off.assign(n_tiles + 1, 0);
    for (int64_t t = 0; t < n_tiles; ++t) L.off[t + 1] = L.off[t] + parts[t].size();
    L.blob.resize(L.off[n_tiles]);
#pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < n_tiles; ++t)
        std::memcpy(L.blob.data() + L.off[t], parts[t].data(), parts[t].size());
    double hsum = 0, fsum = 0, rsum = 0;
    for (int64_t t = 0; t < n_tiles; ++t) {
        L.max_tile_bytes = std::max<uint32_t>(L.max_tile_bytes, (uint32_t)parts[t].size());
        L.max_tile_smem = std::max<uint32_t>(L.max_tile_smem, (uint32_t)parts[t].size());
        const uint32_t head = tSplit[t] & 0xffffffu;
        L.max_head_bytes = std::max<uint32_t>(L.max_head_bytes, head);
        L.max_rest_bytes = std::max<uint32_t>(L.max_rest_bytes, (uint32_t)parts[t].size() - head);
        L.max_halo = std::max(L.max_halo, tH[t]);
        L.max_W = std::max<int>(L.max_W, (int)tW[t]);
        L.max_Wr = std::max<int>(L.max_Wr, (int)tWr[t]);
        const int n = (int)tN[t];
        hsum += (double)(n + tH[t]) / n;
        fsum += tF[t];
        rsum += (double)tRefs[t];
    }
    L.halo_ratio = hsum / (double)n_tiles;
    L.foreign_frac = rsum > 0 ? fsum / rsum : 0.0;
    return SS_OK;
}

}  // namespace ss
