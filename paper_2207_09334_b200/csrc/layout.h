// Host construction of the device incidence layouts.
#pragma once

#include <cstdint>
#include <vector>

#include <cuda_runtime.h>

namespace ss {

struct LayoutInput {
    int64_t N, S;
    const int64_t *si, *sj;
};

struct Layout {
    int kind = 1;                 // SS_LAYOUT_CSR / SS_LAYOUT_ELL
    // CSR
    std::vector<int> row;         // N+1
    std::vector<int2> inc;        // 2S: (other, spring id), per mass in spring-id order
    // ELL
    int W = 0, Wr = 0;            // own / ref widths (max per-mass counts)
    int64_t slices = 0;
    std::vector<int> e_other;     // slices*W*32
    std::vector<int64_t> e_spring;// slices*W*32, -1 = padding (host only)
    std::vector<int> r_pos;       // slices*Wr*32, -1 = padding
    std::vector<int> cnt;         // N: n_own_inline | n_ref << 16
    bool canonical = true;        // every mass: refs-then-own == spring-id order
};

// want: SS_LAYOUT_AUTO / CSR / ELL.  Returns SS_OK or an error status.
int build_layout(const LayoutInput &in, int want, Layout &out);

}  // namespace ss
