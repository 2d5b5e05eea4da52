// metrics.cuh — device reconstruction diagnostics (metrics.hpp:9-24).
#pragma once

#include "common.cuh"

namespace ptg {

// any subset of relativeError / magnitudeRelError / phaseSSIM (mask of
// PTG_METRIC_*) between two n x n device fields in precision prec
void dev_metrics(int prec, const void* z, const void* z_true, int n, unsigned mask, ptg_metrics* out,
                 cudaStream_t s);
// canonicalPhase (metrics.hpp:15-18) into an n x n fp64 device map
void dev_canonical_phase(int prec, const void* z, int n, double* out, cudaStream_t s);

}  // namespace ptg
