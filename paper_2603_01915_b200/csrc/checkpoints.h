// Long-slice checkpoint index shared by the host builder and the kernels.
#pragma once
#include <cstdint>
#include <vector>

#include "../../include/dtans.h"

namespace dtans {

// One warp task: segments [j0, j1) of a long slice.  ck indexes the
// checkpoint record in the pool ({active lane mask, then per active lane
// w0, w1, w2, d, r, col}); 0xFFFFFFFF = start from the slice's init events.
struct LongTask {
    uint32_t slice, j0, j1, part;  // part: partial-sum slot
    uint32_t cur0, cur1;           // slice-relative cursor at j0 and expected at j1
    uint32_t ck, last;             // last: j1 is the slice's final segment count
};

// Segments [j0, j1) of a long slice whose only active lane is `lane` from
// j0 on: its words are consecutive in the stream, so one thread decodes the
// chunk without the other lanes.  ck indexes {w0, w1, w2, d, r, col}.
struct SoloTask {
    uint32_t slice, lane, j0, j1;
    uint32_t part, cur0, cur1, ck;
};

// A staged task: segments [j0, j1) of a long slice whose words [cur0,
// cur1) fit one staging buffer together with the slice's row_symbols and the
// resume state, so the main kernel decodes it from shared memory like a
// chunk (one TMA bulk copy).  ck indexes {mask, per active lane w0, w1, w2,
// d, r, col} in the pool, or 0xFFFFFFFF (start from the init events).
struct StagedTask {
    uint32_t slice, j0, j1, part;
    uint32_t cur0, cur1, ck, last;
};

struct LongSlice {
    uint32_t slice, part_base, nparts, pad;
};

struct LongIndex {
    std::vector<LongTask> tasks;     // global-memory warp tasks (task kernel)
    std::vector<SoloTask> solo;      // single-lane tasks (solo kernel)
    std::vector<StagedTask> staged;  // shared-memory tasks (main kernel)
    std::vector<uint32_t> pool;
    std::vector<LongSlice> slices;
    uint32_t nparts = 0;
};

// Slices whose longest row has more than seg_threshold segments, or whose
// 16-byte aligned stream window exceeds max_words (does not fit a staging
// buffer), are long.  With stage_words > 0 a long slice is cut into staged
// tasks whose resume state + words fit stage_words (a new task starts at the
// segment where the window would overflow); a slice with a segment larger
// than that falls back to global-memory tasks of `chunk` segments.  Once a
// single lane is left at a task boundary, its remaining segments become solo
// tasks of `chunk` segments.
int build_long_index(const dtans_container_view *c, int seg_threshold, uint64_t max_words, int chunk,
                     uint64_t stage_words, LongIndex &out);

}  // namespace dtans
