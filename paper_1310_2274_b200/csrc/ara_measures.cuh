// ara_measures.cuh -- device radix select + tail sort for PML / TVaR.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace ara {

constexpr uint32_t kSortCap = 32768;   // max K (deepest rank needed) per call

struct SelectState {
    uint64_t k_rem;            // rank still to find within the current prefix
    uint32_t prefix, pmask;    // key bits fixed so far
    unsigned long long n_gt;   // keys > T
    unsigned long long n_eq;   // keys == T
};

struct MeasuresScratch {
    float *vals = nullptr;     // [capacity] gathered / rolled-up losses
    uint64_t capacity = 0;
    float *buf = nullptr;      // [kSortCap] losses above the threshold
    unsigned int *hist = nullptr;
    SelectState *state = nullptr;
    double *d_rps = nullptr;   // [64]
    double *d_out = nullptr;   // [128]
    // deep-rank path (K > kSortCap): one select per needed rank + a tail sum
    SelectState *states = nullptr;       // [kMaxRanks]
    double *part_sum = nullptr;          // [kRedBlocks]
    unsigned long long *part_cnt = nullptr;
};

constexpr int kMaxRanks = 3 * 64;

struct RpList {                // return periods, passed by value to the sort kernel
    double v[64];
};
constexpr int kRedBlocks = 592;

cudaError_t launch_measures(const float *ylt, uint32_t n_layers, uint64_t n_total, uint32_t n_shards,
                            int32_t layer, const RpList &rps, uint32_t n_rp, uint64_t k_need,
                            MeasuresScratch &S, double *d_out, cudaStream_t s);

cudaError_t launch_measures_deep(const float *ylt, uint32_t n_layers, uint64_t n_total,
                                 uint32_t n_shards, int32_t layer, const double *rps, uint32_t n_rp,
                                 MeasuresScratch &S, double *d_out, cudaStream_t s);

}  // namespace ara
