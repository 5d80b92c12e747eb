// ara_measures.cuh -- device radix select + tail sort for PML / TVaR.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace ara {

constexpr uint32_t kSortCap = 32768;   // max K (deepest rank needed) per call
constexpr int kMaxPlanRanks = 16;      // joint select: 3 ranks per return period (n_rp <= 4) + L(1), L(N)
// joint select histograms: 12-bit digits for the first pass (one group), 10-bit
// digits per rank group for the second and third, then their chunk sums (32 bins each)
constexpr uint32_t kMultiBinWords = 4096u + 2u * kMaxPlanRanks * 1024u;
constexpr uint32_t kMultiHistWords = kMultiBinWords + kMultiBinWords / 32u;

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
    // joint select (launch_measures_multi)
    unsigned int *mhist = nullptr;       // [4][kMaxPlanRanks][256]
    unsigned long long *macc = nullptr;  // [8]: fixed-point tail sums, counts
};

constexpr int kMaxRanks = 3 * 64;

struct RpList {                // return periods, passed by value to the sort kernel
    double v[64];
};
constexpr int kRedBlocks = 592;

cudaError_t launch_measures(const float *ylt, uint32_t n_layers, uint64_t n_total, uint32_t n_shards,
                            int32_t layer, const RpList &rps, uint32_t n_rp, uint64_t k_need,
                            MeasuresScratch &S, double *d_out, cudaStream_t s);

// every needed rank in one cooperative launch (n_rp <= 4), any depth
cudaError_t launch_measures_multi(const float *ylt, uint32_t n_layers, uint64_t n_total, uint32_t n_shards,
                                  int32_t layer, const double *rps, uint32_t n_rp, MeasuresScratch &S,
                                  double *d_out, cudaStream_t s);

// the YLT (layer or roll-up) sorted descending: the exceedance curve (NEXT-3)
cudaError_t launch_exceedance_curve(const float *ylt, uint32_t n_layers, uint64_t n_total, uint32_t n_shards,
                                    int32_t layer, uint32_t *scratch, float *out, cudaStream_t s, int num_sms);

cudaError_t launch_measures_deep(const float *ylt, uint32_t n_layers, uint64_t n_total,
                                 uint32_t n_shards, int32_t layer, const double *rps, uint32_t n_rp,
                                 MeasuresScratch &S, double *d_out, cudaStream_t s);

}  // namespace ara
