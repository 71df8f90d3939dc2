// Tiled incidence layout (SS_LAYOUT_TILE): host builder.
#pragma once

#include <cstdint>
#include <vector>

namespace ss {

constexpr int kTile = 256;            // masses per tile == threads per CTA

// Per-tile blob header (all offsets in bytes from the tile start, 16-B aligned).
// [0, off_cnt) (header + halo ids) is copied first so the halo gather
// overlaps the record stream.
//
// fp64 builds (bit parity, tiles.cpp build_tiles): 32-wide ELL slices.
//   Section order: header | halo ids | counts | own other | own (k,l0) |
//   own grp | refs | foreign owner | foreign (k,l0) | foreign grp.
//   counts: n_own | n_ref << 8.  A mass sums references then own records,
//   both in ascending spring id (the reference's serial order).
//   ref value: bit 15 set  -> foreign record index (bits 0-14)
//              bit 15 clear-> in-tile record: owner local id (bits 0-7), slot q (bits 8-14)
//
// fp32 builds (production, tiles_f32.cpp build_tiles_f32): one 256-wide ELL
// slice, slot = q*256 + l, records (other local u16, k f32, k*l0 f32
// [, grp i8]) as planar arrays (the okl section is k[W*256] then
// k*l0[W*256]; fkl likewise over the n_foreign copies); padding slots
// point at their own mass with k = 0.  A
// spring whose owner lies in another tile is copied into the partner's
// tile (foreign owner, foreign local partner off_fl, (k, k*l0), grp).  A
// mass's reference list holds its foreign references first (0x8000 | copy;
// their count per mass in off_nf) and then its in-tile ones, whose value
// is the owner's slot.  counts: n_own | n_ref << 8.
struct TileHdr {
    uint32_t n, W, Wr, n_halo;
    uint32_t n_foreign, bytes, off_cnt, off_oo;
    uint32_t off_okl, off_og, off_ref, off_fo;
    uint32_t off_fkl, off_fg, off_halo, canonical;
    uint32_t off_nf;       // fp32 builds: u8 per mass, leading foreign references
    uint32_t slice_log2;   // sliced-ELL slice of 2^slice_log2 masses (fp64 builds 5, fp32 builds 8)
    uint32_t off_fl;       // fp32 builds: u8 per foreign copy, its local partner
    uint32_t pad3;
};
static_assert(sizeof(TileHdr) == 80, "TileHdr must stay 80 bytes");

struct TileInput {
    int64_t N, S;
    const int64_t *si, *sj;
    const double *x;             // (N,3) positions for the brick renumbering (may be null: identity)
    const double *k, *l0;
    const int32_t *group;        // may be null
    bool f32;                    // record precision
    int order;                   // 0 identity, 1 brick
};

// Sliced-ELL position of entry q of tile mass l (slices of 2^sl masses, W
// entries per slice row).  fp32 builds use sl = 8 (one slice per tile), so
// slot = q*256 + l and an in-tile reference value (q << 8 | owner) IS the
// owner's record slot.
#if defined(__CUDACC__)
__host__ __device__
#endif
inline uint32_t ell_slot(uint32_t l, uint32_t q, uint32_t W, uint32_t sl) {
    return (((l >> sl) * W + q) << sl) | (l & ((1u << sl) - 1u));
}

struct TileLayout {
    std::vector<int32_t> orig_of;   // new id -> original id (empty: identity)
    std::vector<int32_t> new_of;    // original id -> new id
    std::vector<uint8_t> blob;      // concatenated tiles
    std::vector<uint64_t> off;      // n_tiles + 1 byte offsets into blob
    std::vector<uint32_t> split;    // per tile: bytes of the first copy (header + halo ids)
    int64_t n_tiles = 0;
    uint32_t max_tile_bytes = 0;
    uint32_t max_head_bytes = 0;    // [0, split): header + halo ids
    uint32_t max_rest_bytes = 0;    // [split, bytes): counts + records + refs
    uint32_t max_halo = 0;
    int max_W = 0, max_Wr = 0;
    bool canonical = true;
    bool has_self = false;          // a spring joins a mass to itself
    double halo_ratio = 0.0;        // mean (n + n_halo) / n
    double foreign_frac = 0.0;      // refs whose owner lies in another tile
};

int build_tiles(const TileInput &in, TileLayout &out);      // fp64; dispatches fp32 builds to:
int build_tiles_f32(const TileInput &in, TileLayout &out);
// Device slot order (brick renumbering, tiles padded to kTile slots).
void tile_order(const TileInput &in, std::vector<int32_t> &orig_of);

}  // namespace ss
