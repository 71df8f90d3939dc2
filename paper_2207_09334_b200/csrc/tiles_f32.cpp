// Host builder of the fp32 (production) tiled layout (tiles.h).
//
// Same tiles as the fp64 builder (4x8x8 bricks of the lattice packed into
// 256-slot tiles, spring owner = endpoint with the lower caller id), but
// organised for the spring-once kernels of tile_f32.cuh instead of the
// reference's summation order (fp32 is a tolerance mode):
//
//  * own records of mass l at slot q*256 + l (one 256-wide ELL slice);
//  * foreign copies: a spring whose owner lies in another tile is copied
//    into the partner's tile (owner halo index, local partner, k, k*l0);
//  * reference list of mass l: foreign references first (0x8000 | copy),
//    then in-tile ones, whose value is the owner's slot (q*256 + owner);
//  * inside a tile the masses are ordered by (foreign, own, in-tile
//    reference) counts, so the 32 lanes of a warp walk lists of equal length;
//  * records hold k and k*l0 in fp32, as two planar arrays (k, then k*l0),
//    so the c written over k and read by the partners is a dense array.

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <numeric>
#include <tuple>

#include "common.h"
#include "springsim_b200.h"
#include "tiles.h"

namespace ss {

namespace {

inline uint32_t al16(uint32_t v) { return (v + 15u) & ~15u; }

template <typename T>
void put_at(std::vector<uint8_t> &blob, uint32_t off, const T &v) {
    std::memcpy(blob.data() + off, &v, sizeof(T));
}

}  // namespace

// mode: 0 explicit, 1 compact with the dictionary, 2 compact with inline records
int build_tiles_f32_fmt(const TileInput &in, TileLayout &L, int mode);

namespace {
size_t own_total(const std::vector<std::vector<int32_t>> &own) {
    size_t n = 0;
    for (const auto &o : own) n += o.size();
    return n;
}
}  // namespace

// Compact format when every tile has at most 64 distinct (k, k*l0, group, D)
// records and at most 768 halo slots; compact lists with inline records when
// only the dictionary overflows (SS_TILE_DICT=0 forces it); the explicit
// format otherwise (SS_TILE_DICT=explicit forces it).
int build_tiles_f32(const TileInput &in, TileLayout &L) {
    const char *env = getenv("SS_TILE_DICT");
    const bool explicit_only = env && std::strcmp(env, "explicit") == 0;
    const bool inline_only = env && !explicit_only && atoi(env) == 0;
    if (!explicit_only) {
        // the D-keyed dictionary, then a (k, k*l0, group) dictionary with the
        // rest vectors formed from X0 on the device, then inline records
        int rc = inline_only ? SS_EAGAIN_DICT : build_tiles_f32_fmt(in, L, 1);
        if (rc == SS_EAGAIN_DICT && !inline_only) rc = build_tiles_f32_fmt(in, L, 3);
        if (rc == SS_EAGAIN_DICT) rc = build_tiles_f32_fmt(in, L, 2);
        if (rc != SS_EAGAIN_DICT && rc != SS_EAGAIN_SHAPE) return rc;
    }
    return build_tiles_f32_fmt(in, L, 0);
}

int build_tiles_f32_fmt(const TileInput &in, TileLayout &L, int mode) {
    const bool use_dict = mode != 0, inline_rec = mode == 2, dict_x0 = mode == 3;
    const int64_t N = in.N, S = in.S;
    if (N >= (1ll << 30) || S >= (1ll << 31)) return fail(SS_EINVAL, "scene too large for the tiled layout");
    L = TileLayout{};
    std::vector<int32_t> zcell;
    tile_order(in, L.orig_of, &zcell);
    const bool bank_aware = !zcell.empty();
    const int64_t D = (int64_t)L.orig_of.size();
    const int64_t n_tiles = D / kTile;
    // per caller mass: own springs and springs referencing it, ascending id
    std::vector<int64_t> own_ptr(N + 1, 0), ref_ptr(N + 1, 0);
    for (int64_t s = 0; s < S; ++s) {
        const int64_t a = std::min(in.si[s], in.sj[s]), b = std::max(in.si[s], in.sj[s]);
        own_ptr[a + 1]++;
        ref_ptr[b + 1]++;
        if (a == b) L.has_self = true;
    }
    for (int64_t m = 0; m < N; ++m) {
        own_ptr[m + 1] += own_ptr[m];
        ref_ptr[m + 1] += ref_ptr[m];
    }
    std::vector<int32_t> own_sp(S), ref_sp(S);
    {
        std::vector<int64_t> oc(own_ptr.begin(), own_ptr.end() - 1), rc(ref_ptr.begin(), ref_ptr.end() - 1);
        for (int64_t s = 0; s < S; ++s) {
            const int64_t a = std::min(in.si[s], in.sj[s]), b = std::max(in.si[s], in.sj[s]);
            own_sp[oc[a]++] = (int32_t)s;
            ref_sp[rc[b]++] = (int32_t)s;
        }
    }
    std::vector<int32_t> tile_of(N);
    for (int64_t i = 0; i < D; ++i)
        if (L.orig_of[i] >= 0) tile_of[L.orig_of[i]] = (int32_t)(i / kTile);
    auto owner_of = [&](int32_t s) { return std::min(in.si[s], in.sj[s]); };
    auto other_of = [&](int32_t s) { return std::max(in.si[s], in.sj[s]); };

    // 1) optionally order the masses inside each tile by work: (foreign,
    // own, in-tile) counts (SS_TILE_SORT=1).  Off by default: the brick
    // order keeps in-tile neighbour gathers bank-conflict free.
    const char *sort_env = getenv("SS_TILE_SORT");
    const bool work_sort = sort_env && atoi(sort_env) != 0;
#pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < (work_sort ? n_tiles : 0); ++t) {
        int32_t *slot = L.orig_of.data() + t * kTile;
        int n = 0;
        while (n < kTile && slot[n] >= 0) ++n;
        std::vector<std::pair<uint32_t, int32_t>> key(n);
        for (int l = 0; l < n; ++l) {
            const int64_t m = slot[l];
            const uint32_t own = (uint32_t)(own_ptr[m + 1] - own_ptr[m]);
            uint32_t in_t = 0, fr = 0;
            for (int64_t r = ref_ptr[m]; r < ref_ptr[m + 1]; ++r) {
                if (tile_of[owner_of(ref_sp[r])] == t) ++in_t;
                else ++fr;
            }
            key[l] = {(std::min(fr, 255u) << 16) | (std::min(own, 255u) << 8) | std::min(in_t, 255u), (int32_t)m};
        }
        std::stable_sort(key.begin(), key.end(),
                         [](const auto &a, const auto &b) { return a.first > b.first; });
        for (int l = 0; l < n; ++l) slot[l] = key[l].second;
    }
    L.new_of.assign(N, -1);
    for (int64_t i = 0; i < D; ++i)
        if (L.orig_of[i] >= 0) L.new_of[L.orig_of[i]] = (int32_t)i;
    // index of each spring in its owner's compute list (own records come first)
    std::vector<uint8_t> q_of(S);
    for (int64_t m = 0; m < N; ++m) {
        if (own_ptr[m + 1] - own_ptr[m] > 255) return fail(SS_EINVAL, "a mass owns more than 255 springs (tiled layout)");
        for (int64_t q = own_ptr[m]; q < own_ptr[m + 1]; ++q) q_of[own_sp[q]] = (uint8_t)(q - own_ptr[m]);
    }

    // 2) per-tile blobs
    L.n_tiles = n_tiles;
    std::vector<std::vector<uint8_t>> parts(n_tiles);
    std::vector<uint32_t> tH(n_tiles), tHr(n_tiles), tSplit(n_tiles), tN(n_tiles), tW(n_tiles), tWr(n_tiles);
    std::vector<int64_t> tFor(n_tiles), tRefs(n_tiles);
    const bool has_g = in.group != nullptr;
    std::vector<std::vector<float>> tKD(inline_rec ? n_tiles : 0);
    std::vector<std::vector<int8_t>> tG(inline_rec && has_g ? n_tiles : 0);
    int err = 0;        // 1 hard limit, 3 dictionary overflow, 4 compact shape overflow
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t t = 0; t < n_tiles; ++t) {
        if (err) continue;
        const int64_t base = t * kTile;
        int n = 0;
        while (n < kTile && L.orig_of[base + n] >= 0) ++n;
        auto local = [&](int64_t caller) -> int64_t { return (int64_t)L.new_of[caller] - base; };
        // own records (spring ids), foreign copies and reference lists
        std::vector<std::vector<int32_t>> own(n), refs(n);
        std::vector<uint8_t> n_for(kTile, 0);
        std::vector<int32_t> halo, foreign;      // foreign: spring ids of the copies
        std::vector<uint8_t> foreign_l;          // their local partner
        for (int l = 0; l < n; ++l) {
            const int64_t m = L.orig_of[base + l];
            for (int64_t q = own_ptr[m]; q < own_ptr[m + 1]; ++q) {
                own[l].push_back(own_sp[q]);
                const int64_t ol = local(other_of(own_sp[q]));
                if (ol < 0 || ol >= n) halo.push_back(L.new_of[other_of(own_sp[q])]);
            }
            for (int pass = 0; pass < 2; ++pass) {          // foreign references first
                for (int64_t r = ref_ptr[m]; r < ref_ptr[m + 1]; ++r) {
                    const int32_t s = ref_sp[r];
                    const int64_t ol = local(owner_of(s));
                    const bool in_tile = ol >= 0 && ol < n;
                    if (in_tile != (pass == 1)) continue;
                    if (in_tile) {
                        refs[l].push_back((int32_t)(((uint32_t)q_of[s] << 8) | (uint32_t)ol));
                    } else {
                        refs[l].push_back((int32_t)(0x8000u | (uint32_t)foreign.size()));
                        foreign.push_back(s);
                        foreign_l.push_back((uint8_t)l);
                        halo.push_back(L.new_of[owner_of(s)]);
                        n_for[l]++;
                    }
                }
            }
        }
        std::sort(halo.begin(), halo.end());
        halo.erase(std::unique(halo.begin(), halo.end()), halo.end());
        // Bank-aware halo slots: slot = 256 + 8j + (z mod 8), so every staged
        // mass (own ones sit at l == z mod 8 in a brick) has slot == z (mod 8)
        // and the 8 lanes of a 128-bit shared-memory phase (8 consecutive z
        // of one brick row) gather 8 distinct bank groups, in-tile or halo.
        std::vector<uint16_t> halo_slot(halo.size());
        std::vector<int32_t> halo_ids;            // per slot, -1 = hole
        bool pad_ok = bank_aware;
        if (pad_ok && use_dict) {                 // the compact format addresses <= 768 halo slots
            uint32_t cnt[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            for (size_t i = 0; i < halo.size(); ++i) cnt[(uint32_t)zcell[L.orig_of[halo[i]]] & 7u]++;
            uint32_t maxc = 0;
            for (int r = 0; r < 8; ++r) maxc = std::max(maxc, cnt[r]);
            pad_ok = kTile + 8 * maxc <= 1024;    // else: plain sorted halo for this tile
        }
        if (pad_ok) {
            uint32_t cnt[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            std::vector<uint32_t> cls(halo.size());
            for (size_t i = 0; i < halo.size(); ++i) {
                const uint32_t r = (uint32_t)zcell[L.orig_of[halo[i]]] & 7u;
                cls[i] = cnt[r]++;
            }
            uint32_t maxc = 0;
            for (int r = 0; r < 8; ++r) maxc = std::max(maxc, cnt[r]);
            halo_ids.assign((size_t)8 * maxc, -1);
            for (size_t i = 0; i < halo.size(); ++i) {
                const uint32_t slot = 8 * cls[i] + ((uint32_t)zcell[L.orig_of[halo[i]]] & 7u);
                halo_ids[slot] = halo[i];
                halo_slot[i] = (uint16_t)(kTile + slot);
            }
        } else {
            halo_ids = halo;
            for (size_t i = 0; i < halo.size(); ++i) halo_slot[i] = (uint16_t)(kTile + i);
        }
        int W = 1, Wr = 1;
        for (int l = 0; l < n; ++l) {
            W = std::max(W, (int)own[l].size());
            Wr = std::max(Wr, (int)refs[l].size());
        }
        if (W > 255 || Wr > 255 || halo_ids.size() + kTile > 65535 || foreign.size() >= 0x8000) {
#pragma omp atomic write
            err = 1;
            continue;
        }
        auto slot_of_local = [&](int64_t dev) -> uint16_t {
            const int64_t ol = dev - base;
            if (ol >= 0 && ol < n) return (uint16_t)ol;
            const auto it = std::lower_bound(halo.begin(), halo.end(), (int32_t)dev);
            return halo_slot[it - halo.begin()];
        };
        const uint32_t own_n = (uint32_t)W << 8, ref_n = (uint32_t)Wr << 8, nf = (uint32_t)foreign.size();
        if (use_dict) {
            // compact format: per mass one incidence list (own springs, then
            // the springs it references), u16 = partner slot | dict index << 10
            // dictionary key: (k, k*l0, group, rest vector D = fp32(X0_other - X0_me))
            using Key = std::tuple<float, float, int, float, float, float>;
            std::map<Key, uint32_t> dict;
            auto key_of = [&](int32_t s, int64_t m) {
                const int64_t o = (int64_t)in.si[s] + in.sj[s] - m;
                if (dict_x0)                                  // D formed on the device from X0
                    return std::make_tuple((float)in.k[s], (float)(in.k[s] * in.l0[s]),
                                           has_g ? (int)in.group[s] : -1, 0.f, 0.f, 0.f);
                return std::make_tuple((float)in.k[s], (float)(in.k[s] * in.l0[s]), has_g ? (int)in.group[s] : -1,
                                       (float)(in.x[3 * o] - in.x[3 * m]), (float)(in.x[3 * o + 1] - in.x[3 * m + 1]),
                                       (float)(in.x[3 * o + 2] - in.x[3 * m + 2]));
            };
            std::vector<std::vector<int32_t>> inc(n);
            int Wi = 1;
            for (int l = 0; l < n; ++l) {
                const int64_t m = L.orig_of[base + l];
                for (const int32_t s : own[l]) inc[l].push_back(s);
                for (int64_t r = ref_ptr[m]; r < ref_ptr[m + 1]; ++r) inc[l].push_back(ref_sp[r]);
                if (!inline_rec)
                    for (const int32_t s : inc[l]) dict.emplace(key_of(s, m), 0u);
                Wi = std::max(Wi, (int)inc[l].size());
            }
            if (kTile + halo_ids.size() > 1024 || Wi > 255) {
#pragma omp atomic write
                err = 4;                                       // the shape does not fit: explicit format
                continue;
            }
            if (dict.size() > 64) {
                if (err != 4) {
#pragma omp atomic write
                    err = 3;                                   // only the dictionary overflows: inline records
                }
                continue;
            }
            uint32_t di = 0;
            for (auto &kv : dict) kv.second = di++;
            const uint32_t D = (uint32_t)dict.size(), inc_n = (uint32_t)Wi << 8;
            TileHdr h{};
            h.n = n; h.W = Wi; h.Wr = 0; h.n_halo = (uint32_t)halo_ids.size(); h.n_foreign = 0;
            h.canonical = 1 | 2 | (inline_rec ? 4 : 0) | (dict_x0 ? 8 : 0);   // bit 1: compact; 2: inline; 3: D from X0
            h.slice_log2 = 8;
            h.n_dict = D;
            uint32_t off = al16(sizeof(TileHdr));
            h.off_halo = off; off = al16(off + (uint32_t)halo_ids.size() * 4);
            h.off_cnt = off;  off = al16(off + kTile * 2);       // n_own | n_inc << 8
            h.off_oo = off;   off = al16(off + inc_n * 2);       // incidences
            h.off_okl = off;  off = al16(off + D * 32);          // dictionary: float4 (k, k*l0, Dx, Dy), float4 (Dz, grp bits, 0, 0)
            h.off_og = 0;
            if (has_g) { h.off_og = off; off = al16(off + D); } // dictionary groups
            h.off_nf = h.off_ref = h.off_fo = h.off_fkl = h.off_fl = h.off_fg = 0;
            h.bytes = off;
            std::vector<uint8_t> &blob = parts[t];
            blob.assign(off, 0);
            std::memcpy(blob.data(), &h, sizeof h);
            std::memcpy(blob.data() + h.off_halo, halo_ids.data(), halo_ids.size() * 4);
            for (const auto &kv : dict) {
                const uint32_t e = kv.second;
                put_at<float>(blob, h.off_okl + 32 * e, std::get<0>(kv.first));
                put_at<float>(blob, h.off_okl + 32 * e + 4, std::get<1>(kv.first));
                put_at<float>(blob, h.off_okl + 32 * e + 8, std::get<3>(kv.first));
                put_at<float>(blob, h.off_okl + 32 * e + 12, std::get<4>(kv.first));
                put_at<float>(blob, h.off_okl + 32 * e + 16, std::get<5>(kv.first));
                put_at<int32_t>(blob, h.off_okl + 32 * e + 20, (int32_t)std::get<2>(kv.first));
                if (has_g) put_at<int8_t>(blob, h.off_og + e, (int8_t)std::get<2>(kv.first));
            }
            if (inline_rec) {
                tKD[t].assign((size_t)2 * inc_n, 0.f);
                if (has_g) tG[t].assign((size_t)inc_n, (int8_t)-1);
            }
            int64_t n_inc = 0;
            for (int l = 0; l < n; ++l) {
                const int64_t m = L.orig_of[base + l];
                put_at<uint16_t>(blob, h.off_cnt + 2 * l, (uint16_t)(own[l].size() | (inc[l].size() << 8)));
                for (size_t q = 0; q < inc[l].size(); ++q) {
                    const int32_t s = inc[l][q];
                    const int64_t o = (int64_t)in.si[s] + in.sj[s] - m;   // the other endpoint
                    const uint32_t at = ((uint32_t)q << 8) | (uint32_t)l;
                    uint32_t di = 0;
                    if (inline_rec) {                          // (k, k*l0); D from X0 on the device
                        tKD[t][2 * at] = (float)in.k[s];
                        tKD[t][2 * at + 1] = (float)(in.k[s] * in.l0[s]);
                        if (has_g) tG[t][at] = (int8_t)in.group[s];
                    } else {
                        di = dict.at(key_of(s, m));
                    }
                    const uint32_t v = (uint32_t)slot_of_local(L.new_of[o]) | (di << 10);
                    put_at<uint16_t>(blob, h.off_oo + 2 * at, (uint16_t)v);
                }
                n_inc += (int64_t)inc[l].size();
            }
            tH[t] = (uint32_t)halo_ids.size();
            tHr[t] = (uint32_t)halo.size();
            tSplit[t] = h.off_cnt | ((uint32_t)(n - 1) << 24);
            tN[t] = n; tW[t] = Wi; tWr[t] = 0;
            tFor[t] = nf;
            tRefs[t] = n_inc - (int64_t)own_total(own);
            continue;
        }
        TileHdr h{};
        h.n = n; h.W = W; h.Wr = Wr; h.n_halo = (uint32_t)halo_ids.size(); h.n_foreign = nf;
        h.canonical = 1;
        h.slice_log2 = 8;
        uint32_t off = al16(sizeof(TileHdr));
        h.off_halo = off; off = al16(off + (uint32_t)halo_ids.size() * 4);
        h.off_cnt = off;  off = al16(off + kTile * 2);
        h.off_nf = off;   off = al16(off + kTile);
        h.off_oo = off;   off = al16(off + own_n * 2);
        h.off_okl = off;  off = al16(off + own_n * 20);         // planar k, k*l0, Dx, Dy, Dz
        h.off_og = 0;
        if (has_g) { h.off_og = off; off = al16(off + own_n); }
        h.off_ref = off;  off = al16(off + ref_n * 2);
        h.off_fo = off;   off = al16(off + nf * 2);
        h.off_fl = off;   off = al16(off + nf);
        h.off_fkl = off;  off = al16(off + nf * 20);            // planar k, k*l0, Dx, Dy, Dz
        h.off_fg = 0;
        if (has_g) { h.off_fg = off; off = al16(off + nf); }
        h.bytes = off;
        std::vector<uint8_t> &blob = parts[t];
        blob.assign(off, 0);
        std::memcpy(blob.data(), &h, sizeof h);
        std::memcpy(blob.data() + h.off_halo, halo_ids.data(), halo_ids.size() * 4);
        for (uint32_t l = 0; l < (uint32_t)kTile; ++l)          // padding: self, k = 0
            for (int q = 0; q < W; ++q) put_at<uint16_t>(blob, h.off_oo + 2 * (((uint32_t)q << 8) | l), (uint16_t)l);
        if (has_g) std::memset(blob.data() + h.off_og, 0xff, own_n);
        std::memset(blob.data() + h.off_ref, 0xff, ref_n * 2);
        std::memcpy(blob.data() + h.off_nf, n_for.data(), kTile);
        int64_t n_refs = 0;
        for (int l = 0; l < n; ++l) {
            const int64_t m = L.orig_of[base + l];
            put_at<uint16_t>(blob, h.off_cnt + 2 * l, (uint16_t)(own[l].size() | (refs[l].size() << 8)));
            for (size_t q = 0; q < own[l].size(); ++q) {
                const int32_t s = own[l][q];
                const uint32_t slot = ((uint32_t)q << 8) | (uint32_t)l;
                put_at<uint16_t>(blob, h.off_oo + 2 * slot, slot_of_local(L.new_of[other_of(s)]));
                const int64_t o = other_of(s);                  // D = X0_other - X0_owner
                put_at<float>(blob, h.off_okl + 4 * slot, (float)in.k[s]);
                put_at<float>(blob, h.off_okl + 4 * (own_n + slot), (float)(in.k[s] * in.l0[s]));
                for (int c = 0; c < 3; ++c)
                    put_at<float>(blob, h.off_okl + 4 * ((2 + c) * own_n + slot), (float)(in.x[3 * o + c] - in.x[3 * m + c]));
                if (has_g) put_at<int8_t>(blob, h.off_og + slot, (int8_t)in.group[s]);
            }
            for (size_t q = 0; q < refs[l].size(); ++q)
                put_at<uint16_t>(blob, h.off_ref + 2 * (((uint32_t)q << 8) | (uint32_t)l), (uint16_t)refs[l][q]);
            n_refs += (int64_t)refs[l].size();
        }
        for (uint32_t f = 0; f < nf; ++f) {
            const int32_t s = foreign[f];
            put_at<uint16_t>(blob, h.off_fo + 2 * f, slot_of_local(L.new_of[owner_of(s)]));
            put_at<uint8_t>(blob, h.off_fl + f, foreign_l[f]);
            put_at<float>(blob, h.off_fkl + 4 * f, (float)in.k[s]);
            put_at<float>(blob, h.off_fkl + 4 * (nf + f), (float)(in.k[s] * in.l0[s]));
            {                                                   // D = X0_owner - X0_partner
                const int64_t ow = owner_of(s), pa = other_of(s);
                for (int c = 0; c < 3; ++c)
                    put_at<float>(blob, h.off_fkl + 4 * ((2 + c) * nf + f), (float)(in.x[3 * ow + c] - in.x[3 * pa + c]));
            }
            if (has_g) put_at<int8_t>(blob, h.off_fg + f, (int8_t)in.group[s]);
        }
        const int64_t n_for_t = nf;
        tH[t] = (uint32_t)halo_ids.size();
            tHr[t] = (uint32_t)halo.size();
        tSplit[t] = h.off_cnt | ((uint32_t)(n - 1) << 24);
        tN[t] = n; tW[t] = W; tWr[t] = Wr;
        tFor[t] = n_for_t;
        tRefs[t] = n_refs;
    }
    if (err == 1) return fail(SS_EINVAL, "tile exceeds layout limits (degree or halo too large)");
    if (err == 4) return SS_EAGAIN_SHAPE;
    if (err == 3) return SS_EAGAIN_DICT;
    L.compact = use_dict;
    L.inline_kl = inline_rec;
    L.dict_x0 = dict_x0;
    if (inline_rec) {
        L.kl_off.assign(n_tiles + 1, 0);
        for (int64_t t = 0; t < n_tiles; ++t) L.kl_off[t + 1] = L.kl_off[t] + tKD[t].size() / 2;
        L.kd_inline.resize(2 * L.kl_off[n_tiles]);
        if (has_g) L.g_inline.resize(L.kl_off[n_tiles]);
#pragma omp parallel for schedule(static)
        for (int64_t t = 0; t < n_tiles; ++t) {
            std::memcpy(L.kd_inline.data() + 2 * L.kl_off[t], tKD[t].data(), tKD[t].size() * 4);
            if (has_g) std::memcpy(L.g_inline.data() + L.kl_off[t], tG[t].data(), tG[t].size());
        }
    }
    if (in.group) {
        for (int64_t s = 0; s < S; ++s)
            if (in.group[s] > 127) return fail(SS_EINVAL, "at most 128 actuation groups in the tiled layout");
    }
    L.canonical = true;
    L.split = tSplit;
    L.off.assign(n_tiles + 1, 0);
    for (int64_t t = 0; t < n_tiles; ++t) L.off[t + 1] = L.off[t] + parts[t].size();
    L.blob.resize(L.off[n_tiles]);
#pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < n_tiles; ++t) std::memcpy(L.blob.data() + L.off[t], parts[t].data(), parts[t].size());
    double hsum = 0, fsum = 0, rsum = 0;
    for (int64_t t = 0; t < n_tiles; ++t) {
        L.max_tile_bytes = std::max<uint32_t>(L.max_tile_bytes, (uint32_t)parts[t].size());
        {
            TileHdr th;
            std::memcpy(&th, parts[t].data(), sizeof th);
            L.max_tile_smem = std::max<uint32_t>(L.max_tile_smem, (uint32_t)parts[t].size());
        }
        const uint32_t head = tSplit[t] & 0xffffffu;
        L.max_head_bytes = std::max<uint32_t>(L.max_head_bytes, head);
        L.max_rest_bytes = std::max<uint32_t>(L.max_rest_bytes, (uint32_t)parts[t].size() - head);
        L.max_halo = std::max(L.max_halo, tH[t]);
        L.max_W = std::max<int>(L.max_W, (int)tW[t]);
        L.max_Wr = std::max<int>(L.max_Wr, (int)tWr[t]);
        hsum += (double)(tN[t] + tHr[t]) / tN[t];
        fsum += (double)tFor[t];
        rsum += (double)tRefs[t];
    }
    L.halo_ratio = hsum / (double)n_tiles;
    L.foreign_frac = rsum > 0 ? fsum / rsum : 0.0;
    return SS_OK;
}

}  // namespace ss
