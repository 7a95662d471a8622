// Shared helpers for the sm_100a kernels of libsmoe_b200.so.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/smoe_b200.h"

namespace smoe {

// Thread-local last-error message (smoe_get_last_error).
void set_error(const std::string &msg);
int fail(int status, const std::string &msg);
int check_launch(const char *what, int launches = 1);

// ---- dtype helpers --------------------------------------------------------
template <typename T> struct Num;
template <> struct Num<float> {
  static __device__ __forceinline__ float to_f(float v) { return v; }
  static __device__ __forceinline__ float from_f(float v) { return v; }
};
template <> struct Num<__nv_bfloat16> {
  static __device__ __forceinline__ float to_f(__nv_bfloat16 v) { return __bfloat162float(v); }
  static __device__ __forceinline__ __nv_bfloat16 from_f(float v) { return __float2bfloat16_rn(v); }
};

// ---- activations (moe_layers.py:42-65), evaluated in fp32 -----------------
// Exact-erf GELU (not the tanh approximation) to match the reference.
__device__ __forceinline__ float act_fwd(int act, float z) {
  if (act == SMOE_ACT_GELU) return 0.5f * z * (1.0f + erff(z * 0.70710678118654752f));
  if (act == SMOE_ACT_RELU) return z > 0.0f ? z : 0.0f;
  // SiLU
  return z / (1.0f + expf(-z));
}

__device__ __forceinline__ float act_grad(int act, float z) {
  if (act == SMOE_ACT_GELU)
    return 0.5f * (1.0f + erff(z * 0.70710678118654752f)) +
           z * expf(-0.5f * z * z) * 0.39894228040143268f;
  if (act == SMOE_ACT_RELU) return z > 0.0f ? 1.0f : 0.0f;
  float s = 1.0f / (1.0f + expf(-z));
  return s * (1.0f + z * (1.0f - s));
}

inline int num_sms() {
  static int sms = -1;
  if (sms < 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

}  // namespace smoe
