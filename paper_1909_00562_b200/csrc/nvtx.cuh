// nvtx.cuh -- NVTX ranges for the library's entry points and marks at the
// stage boundaries of the stage (SURVEY.md §5 "Tracing / profiling").  NVTX 3
// is header-only: without an attached tool (ncu, nsys) each call is one
// function-pointer check.
#pragma once
#include <nvtx3/nvToolsExt.h>

namespace attnsm {
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
}  // namespace attnsm
