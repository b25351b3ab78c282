// Internal: the host table stage shared by the CPU encoder (encoder.cpp)
// and the GPU encoder (gpu_encoder.cu).
#pragma once
#include <cstdint>
#include <vector>

#include "common.h"

namespace dtans {

// Distributions (container.py:112-114): sorted unique symbols with counts.
struct Dist {
    std::vector<uint64_t> sym;
    std::vector<int64_t> cnt;
    int64_t total = 0;
};

struct SymMap {  // open addressing, symbol -> retained id
    std::vector<uint64_t> keys;
    std::vector<int32_t> vals;
    uint64_t mask = 0;
    int shift = 0;
    void init(size_t n)
    {
        size_t cap = 16;
        while (cap < 4 * n) cap <<= 1;
        keys.assign(cap, 0);
        vals.assign(cap, -1);
        mask = cap - 1;
        shift = 64 - __builtin_ctzll(cap);
    }
    size_t h(uint64_t k) const { return (size_t)((k * 0x9E3779B97F4A7C15ull) >> shift); }
    void put(uint64_t k, int32_t v)
    {
        size_t i = h(k);
        while (vals[i] >= 0) i = (i + 1) & mask;
        keys[i] = k;
        vals[i] = v;
    }
    int32_t get(uint64_t k) const
    {
        size_t i = h(k);
        while (vals[i] >= 0) {
            if (keys[i] == k) return vals[i];
            i = (i + 1) & mask;
        }
        return -1;
    }
};

// One domain's coding table (entropy.py:333-436) with the encoder-side
// inverse maps.
struct Domain {
    // slot arrays (decode view)
    std::vector<uint64_t> sym;
    std::vector<uint8_t> dig;
    std::vector<uint16_t> base;
    std::vector<uint8_t> esc;
    // encoder view
    int32_t esc_base = 0;            // 0: no escape entry
    std::vector<uint16_t> esc_slot;  // (ESCAPE, d) -> slot, full-base run only
    std::vector<uint16_t> id_base;
    std::vector<uint32_t> id_off;
    std::vector<uint16_t> slot_by_digit;
    SymMap map;
    bool has_pad = false;
    int32_t pad_id = -1;
    int payload_words = 1;
    std::vector<uint64_t> ret_sym;  // retained symbols, ascending (id order)
};

// quantize x2 (container.py:155-158), build_tables x2 (entropy.py:404-436)
// and the serialized slot records (container.py:612-625) into `tables`
// (K * 16 or 12 bytes).
int prepare_tables(const Dist &ddist, const Dist &vdist, int prec, const dtans_encode_opts *opts,
                   uint8_t *tables, Domain &Dd, Domain &Dv);

}  // namespace dtans
