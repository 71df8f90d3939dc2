// Tiled incidence layout (SS_LAYOUT_TILE): host builder.
#pragma once

#include <cstdint>
#include <vector>

namespace ss {

constexpr int kTile = 256;            // masses per tile == threads per CTA

// Per-tile blob header (all offsets in bytes from the tile start, 16-B aligned).
// Section order: header | halo ids | counts | own other | own (k,l0) | own grp |
// refs | foreign owner | foreign (k,l0) | foreign grp.  [0, off_cnt) is copied
// first so the halo gather overlaps the record stream.
//   ref value: bit 15 set  -> foreign record index (bits 0-14)
//              bit 15 clear-> in-tile record: owner local id (bits 0-7), slot q (bits 8-14)
struct TileHdr {
    uint32_t n, W, Wr, n_halo;
    uint32_t n_foreign, bytes, off_cnt, off_oo;
    uint32_t off_okl, off_og, off_ref, off_fo;
    uint32_t off_fkl, off_fg, off_halo, canonical;
    uint32_t pad0, pad1, pad2, pad3;
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
    double halo_ratio = 0.0;        // mean (n + n_halo) / n
    double foreign_frac = 0.0;      // refs whose owner lies in another tile
};

int build_tiles(const TileInput &in, TileLayout &out);

}  // namespace ss
