// transfer.cuh — MG/OPT grid-transfer operators (see transfer.cu).
#pragma once

#include "common.cuh"

namespace ptg {

void dev_restrict_field(int prec, const void* fine, int n, void* coarse, cudaStream_t s);
void dev_prolong_field(int prec, const void* coarse, int nH, void* fine, cudaStream_t s);
// scale = 1/16 for intensities (multigrid.cpp:74), 1/4 for amplitudes sqrt(d)
void dev_restrict_data(int dtype, const void* fine, int N, int M, void* coarse, double scale,
                       cudaStream_t s);

// band-decomposition exchange (halo.cu)
size_t halo_bytes(int prec, int n, int ov);
void dev_halo_pack(int prec, const void* g, int n, int ov, const double* val, void* buf, cudaStream_t s);
void dev_halo_unpack(int prec, void* g, int n, int ov, const void* all, int rank, int world, double* val,
                     cudaStream_t s);

}  // namespace ptg
