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

struct LongSlice {
    uint32_t slice, part_base, nparts, pool_base;  // pool_base: the slice's first resume record
};

struct LongIndex {
    std::vector<LongTask> tasks;     // global-memory warp tasks (task kernel)
    std::vector<SoloTask> solo;      // single-lane tasks (solo kernel)
    std::vector<uint32_t> pool;
    std::vector<LongSlice> slices;
    uint32_t nparts = 0;
};

// Slices whose longest row has more than seg_threshold segments, or whose
// 16-byte aligned stream window exceeds max_words (does not fit a staging
// buffer), are long: they are split into warp tasks of `chunk` segments, and
// once a single lane is left at a task boundary its remaining segments
// become solo tasks of `chunk` segments.
// walk = false: only the structure (tasks, parts, record offsets and masks);
// the cursors and resume records are filled by the GPU walk
// (kernels.cuh dtans_walk_kernel, api.cu).
int build_long_index(const dtans_container_view *c, int seg_threshold, uint64_t max_words, int chunk,
                     bool walk, LongIndex &out);

}  // namespace dtans
