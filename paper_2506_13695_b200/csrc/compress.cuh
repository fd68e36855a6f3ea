// GPU lifelong-history compression (compress.cu): compress_lifelong,
// policy.cpp:447-510, over hierarchical_clusters / kmeans, kmeans.cpp:22-183.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace orx {

struct CompressArgs {  // device pointers
  int D, threshold, n_code_layers;
  int64_t total_points, total_kmax;
  const int64_t *offsets, *out_offsets;
  const int64_t* vid;
  const int32_t* aid;
  const uint32_t* labels;
  const double *tag, *ts, *playtime, *duration;
  const int32_t* sid;
  const double* content;  // [N][D]
  int64_t* out_vid;
  int32_t* out_aid;
  uint32_t* out_labels;
  double *out_tag, *out_ts, *out_playtime, *out_duration;
  int32_t* out_sid;
  double *leaf_tag, *leaf_play, *leaf_dur;  // [N] scratch
};

struct CompressHost {  // host pointers (C-ABI arguments)
  int n_users, D, threshold, max_out, n_code_layers;
  const int64_t* offsets;
  const int64_t* vid;
  const int32_t* aid;
  const uint32_t* labels;
  const double *tag, *ts, *playtime, *duration;
  const int32_t* sid;
  const double* content;
  const uint64_t* rng_seeds;
  int64_t* out_offsets;
  int64_t* out_vid;
  int32_t* out_aid;
  uint32_t* out_labels;
  double *out_tag, *out_ts, *out_playtime, *out_duration;
  int32_t* out_sid;
};

// Runs the whole batch on `device`; outputs min(n_u, max_out) records per user.
void compress_lifelong_gpu(const CompressHost& h, int device);

}  // namespace orx
