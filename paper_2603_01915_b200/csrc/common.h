// Internal helpers shared by the encoder (C++) and the CUDA API (nvcc).
#pragma once
#include <cstdarg>
#include <cstdio>
#include <string>

#include "../../include/dtans.h"

namespace dtans {

// Per-thread last-error text behind dtans_last_error().
void set_error_text(const char *msg);

inline int fail(int code, const char *fmt, ...)
{
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    set_error_text(buf);
    return code;
}

// Shape of an uploaded container (api.cu; used by the multi-GPU driver mg.cu).
void dev_shape(const dtans_dev *h, int64_t *rows, int64_t *cols, int32_t *precision);

constexpr int kSlice = 32;     // rows per slice = lanes per warp (container.py:45)
constexpr int kK = 4096;       // table slots
constexpr int kKLog2 = 12;
constexpr int kL = 8;          // symbols per segment
constexpr int kO = 3;          // words per segment
constexpr int kF = 2;          // conditional checks per segment
constexpr uint64_t kDeltaSentinel = 0xFFFFFFFFull;  // container.py:50

}  // namespace dtans
