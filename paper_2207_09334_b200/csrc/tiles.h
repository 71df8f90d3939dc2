// Tiled incidence layout (SS_LAYOUT_TILE): host builder.
#pragma once

#include <cstdint>
#include <vector>

namespace ss {

constexpr int kTile = 256;            // masses per tile == threads per CTA

// Per-tile blob header (all offsets in bytes from the tile start, 16-B aligned).
struct TileHdr {
    uint32_t n, W, Wr, n_halo;
    uint32_t n_foreign, bytes, off_cnt, off_oo;
    uint32_t off_ok, off_ol, off_og, off_ref;
    uint32_t off_fo, off_fk, off_fl, off_fg;
    uint32_t off_halo, pad0, pad1, pad2;
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
    int64_t n_tiles = 0;
    uint32_t max_tile_bytes = 0;
    uint32_t max_halo = 0;
    int max_W = 0, max_Wr = 0;
    bool canonical = true;
    double halo_ratio = 0.0;        // mean (n + n_halo) / n
    double foreign_frac = 0.0;      // refs whose owner lies in another tile
};

int build_tiles(const TileInput &in, TileLayout &out);

}  // namespace ss
