// Tiled incidence layout (SS_LAYOUT_TILE): host builder.
#pragma once

#include <cstdint>
#include <vector>

namespace ss {

constexpr int kTile = 256;            // masses per tile == threads per CTA
constexpr int SS_EAGAIN_DICT = -1000;  // internal: a tile's (k, l0, group) dictionary does not fit the compact format
constexpr int SS_EAGAIN_SHAPE = -1001; // internal: a tile's degree or halo (or a self spring) does not fit it at all

// Per-tile blob header (all offsets in bytes from the tile start, 16-B aligned).
// [0, off_cnt) (header + halo ids) is copied first so the halo gather
// overlaps the record stream.
//
// fp64 compact builds (bit parity, the default; tiles.cpp
// build_tiles_f64_compact): canonical bit 1 set, one 256-wide ELL slice.
//   header | halo ids | counts (n_inc << 8) | incidences u16 at off_oo,
//   slot q*256 + l, = partner slot (10 bits) | dictionary index << 10, in
//   ascending spring id (the reference's serial order for every mass) |
//   dictionary of n_dict (k, l0) double pairs at off_okl | int8 groups at
//   off_og.
//
// fp64 inline builds (canonical bits 1|2|4; the general-graph format, used
// when some tile has more than 64 distinct (k, l0, group) -- jittered
// robot populations, irregular meshes -- or with SS_TILE_DICT=0): the
// compact layout without a dictionary.  Incidences are the partner slot
// only, and each incidence's (k, l0) double pair (and int8 group) sits in
// the separate global arrays TileLayout::kl_inline / g_inline at
// kl_off[tile] + q*256 + l, streamed by the kernel instead of staged.
//
// fp64 explicit builds (the old fallback, SS_TILE_DICT=explicit; tiles.cpp build_tiles): 32-wide ELL slices.
//   Section order: header | halo ids | counts | own other | own (k,l0) |
//   own grp | refs | foreign owner | foreign (k,l0) | foreign grp.
//   counts: n_own | n_ref << 8.  A mass sums references then own records,
//   both in ascending spring id (the reference's serial order).
//   ref value: bit 15 set  -> foreign record index (bits 0-14)
//              bit 15 clear-> in-tile record: owner local id (bits 0-7), slot q (bits 8-14)
//
// fp32 builds (production, tiles_f32.cpp build_tiles_f32): one 256-wide ELL
// slice, slot = q*256 + l.  fp32 tile engines keep the state as the
// displacement r = x - X0 from the caller's fp64 rest positions, and every
// record carries the fp32 rest vector D = X0_partner - X0_me, so a spring
// vector is d = D + (r_partner - r_me): the small r differences keep the
// strain resolution.  Two record formats:
//  * compact (canonical bit 1 set, the default when every tile has <= 64
//    distinct (k, k*l0, group, D) records and <= 768 halo slots -- a voxel
//    lattice has one per material and stencil direction): every mass has
//    ONE incidence list -- its own springs first, then the springs it
//    references -- of u16 = partner slot (10 bits) | dictionary index << 10;
//    counts = n_own | n_inc << 8 (off_cnt), incidences at off_oo (W = max
//    n_inc); dictionary of 32-byte entries at off_okl: float4 (k, k*l0, Dx,
//    Dy), float4 (Dz, group as int32 bits (-1 passive), 0, 0); int8 groups
//    also at off_og.  2 B per incidence, 4 B per spring.
//  * inline (canonical bits 1|2|4; the fp32 general-graph format when a tile
//    has more than 64 distinct records, or with SS_TILE_DICT=0): the compact
//    incidence lists with partner slots only, and each incidence's (k, k*l0)
//    float2 and int8 group in TileLayout::kd_inline / g_inline at
//    kl_off[tile] + q*256 + l, streamed from HBM; the rest vector
//    D = fp32(X0_partner - X0_me) is formed on the device from the staged
//    fp64 X0 (the same value the dictionary stores).
//  * explicit (canonical bit 1 clear; SS_TILE_DICT=explicit): counts = n_own | n_ref << 8; own
//    records (other u16 off_oo, then planar k, k*l0, Dx, Dy, Dz [W*256 each]
//    at off_okl, grp i8 off_og); a spring whose owner lies in another tile is
//    copied into the partner's tile (owner u16 off_fo, partner u8 off_fl,
//    planar k, k*l0, D = X0_owner - X0_partner [n_foreign each] off_fkl, grp
//    off_fg); a mass's reference list holds its foreign references first
//    (0x8000 | copy; their count per mass in off_nf) and then its in-tile
//    ones, whose value is the owner's slot (the vector to the owner is -D of
//    that record).
// Padding slots point at their own mass.  Halo slots are bank-aware
// (tiles_f32.cpp): slot == z (mod 8), holes carry id -1.
struct TileHdr {
    uint32_t n, W, Wr, n_halo;
    uint32_t n_foreign, bytes, off_cnt, off_oo;
    uint32_t off_okl, off_og, off_ref, off_fo;
    uint32_t off_fkl, off_fg, off_halo, canonical;
    uint32_t off_nf;       // fp32 builds: u8 per mass, leading foreign references
    uint32_t slice_log2;   // sliced-ELL slice of 2^slice_log2 masses (fp64 builds 5, fp32 builds 8)
    uint32_t off_fl;       // fp32 builds: u8 per foreign copy, its local partner
    uint32_t n_dict;       // fp32 compact format: entries of the tile's (k, k*l0) dictionary
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
    uint32_t max_tile_smem = 0;     // shared memory a tile blob needs
    uint32_t max_head_bytes = 0;    // [0, split): header + halo ids
    uint32_t max_rest_bytes = 0;    // [split, bytes): counts + records + refs
    uint32_t max_halo = 0;
    int max_W = 0, max_Wr = 0;
    bool canonical = true;
    bool has_self = false;          // a spring joins a mass to itself
    bool compact = false;           // compact format (fp32 tiles_f32.cpp, fp64 build_tiles_f64_compact)
    bool inline_kl = false;         // fp64 inline format: (k, l0) per incidence in kl_inline
    std::vector<double> kl_inline;  // inline format: (k, l0) pairs, tile t at kl_off[t] pairs
    std::vector<int8_t> g_inline;   // inline format: group per incidence (empty: no groups)
    std::vector<uint64_t> kl_off;   // inline format: n_tiles + 1 slot offsets (W * 256 per tile)
    std::vector<float> kd_inline;   // fp32 inline format: (k, k*l0) per incidence slot
    bool dict_x0 = false;           // fp32 compact: dictionary of (k, k*l0, group), D formed from X0 (canonical bit 3)
    double halo_ratio = 0.0;        // mean (n + n_halo) / n
    double foreign_frac = 0.0;      // refs whose owner lies in another tile
};

int build_tiles(const TileInput &in, TileLayout &out);      // fp64; dispatches fp32 builds to:
int build_tiles_f32(const TileInput &in, TileLayout &out);
// Device slot order (brick renumbering, tiles padded to kTile slots);
// optionally the quantised z cell of every mass (empty: no positions).
void tile_order(const TileInput &in, std::vector<int32_t> &orig_of, std::vector<int32_t> *zcell = nullptr);

}  // namespace ss
