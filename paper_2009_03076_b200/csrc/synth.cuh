// synth.cuh — device-resident cell lists (GPU synthetic generator, csrc/synth.cu).
#pragma once
#include "../../include/exabricks.h"
#include "common.cuh"

namespace xb {

struct DevCells {
    int device = 0;
    int64_t n = 0;
    DevBuf<int32_t> i, j, k, level;
    DevBuf<float> vals;  // one field
};

void generate_synthetic_device(const xb_synth_spec& sp, int device, DevCells& out, cudaStream_t s);

}  // namespace xb
