// NVTX ranges (header-only NVTX v3, CUDA toolkit): decode calls, per-(token, layer) host steps,
// router syncs and tile copies show up as named ranges in Nsight tools (ncu --nvtx filters on
// them); without an attached tool a range costs a few nanoseconds.
#pragma once

#include <nvtx3/nvToolsExt.h>

#include <cstdarg>
#include <cstdio>

namespace adapmoe {

class NvtxRange {
public:
    explicit NvtxRange(const char* fmt, ...) __attribute__((format(printf, 2, 3))) {
        char buf[96];
        va_list ap;
        va_start(ap, fmt);
        std::vsnprintf(buf, sizeof buf, fmt, ap);
        va_end(ap);
        nvtxRangePushA(buf);
    }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

}  // namespace adapmoe
