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

// Accumulator of the SIMT / row kernels: the fp32 check mode accumulates in
// 64-bit and rounds once to the storage dtype, the reference's numeric contract
// (core_tensor.py:1-7); the bf16 SIMT cross-check accumulates in fp32 like the
// tensor cores.
template <typename T> struct AccOf { using type = float; };
template <> struct AccOf<float> { using type = double; };
template <> struct AccOf<double> { using type = double; };
// Element type of per-slot weights (combine weights p, group weights) and of
// dp: float32, float64 when the storage is float64 (SMOE_F64).
template <typename T> struct WOf { using type = float; };
template <> struct WOf<double> { using type = double; };

template <typename T> struct Conv;
template <> struct Conv<__nv_bfloat16> {
  static __device__ __forceinline__ float to_acc(__nv_bfloat16 v) { return __bfloat162float(v); }
  static __device__ __forceinline__ __nv_bfloat16 from_acc(float v) { return __float2bfloat16_rn(v); }
};
template <> struct Conv<float> {
  static __device__ __forceinline__ double to_acc(float v) { return (double)v; }
  static __device__ __forceinline__ float from_acc(double v) { return (float)v; }  // round to nearest even
};
template <> struct Conv<double> {
  static __device__ __forceinline__ double to_acc(double v) { return v; }
  static __device__ __forceinline__ double from_acc(double v) { return v; }
};

// Run `...` with T bound to the storage type of a SMOE_* dtype id.
#define SMOE_DTYPE_DISPATCH(dtype, ...)                          \
  do {                                                           \
    switch (dtype) {                                             \
      case SMOE_BF16: { using T = __nv_bfloat16; __VA_ARGS__; } break; \
      case SMOE_F64: { using T = double; __VA_ARGS__; } break;   \
      default: { using T = float; __VA_ARGS__; } break;          \
    }                                                            \
  } while (0)

// ---- activations (moe_layers.py:42-65), evaluated in fp32 -----------------
// Exact-erf GELU (not the tanh approximation) to match the reference.
__device__ __forceinline__ float act_fwd(int act, float z) {
  if (act == SMOE_ACT_GELU) return 0.5f * z * (1.0f + erff(z * 0.70710678118654752f));
  if (act == SMOE_ACT_RELU) return z > 0.0f ? z : 0.0f;
  if (act == SMOE_ACT_IDENTITY) return z;
  // SiLU
  return z / (1.0f + expf(-z));
}

__device__ __forceinline__ float act_grad(int act, float z) {
  if (act == SMOE_ACT_GELU)
    return 0.5f * (1.0f + erff(z * 0.70710678118654752f)) +
           z * expf(-0.5f * z * z) * 0.39894228040143268f;
  if (act == SMOE_ACT_RELU) return z > 0.0f ? 1.0f : 0.0f;
  if (act == SMOE_ACT_IDENTITY) return 1.0f;
  float s = 1.0f / (1.0f + expf(-z));
  return s * (1.0f + z * (1.0f - s));
}

// 64-bit evaluation for the fp32 check mode: the reference evaluates the
// activation in 64-bit on the storage-rounded input and rounds once
// (moe_layers.py:75-83).
__device__ __forceinline__ double act_fwd(int act, double z) {
  if (act == SMOE_ACT_GELU) return 0.5 * z * (1.0 + erf(z * 0.70710678118654752440));
  if (act == SMOE_ACT_RELU) return z > 0.0 ? z : 0.0;
  if (act == SMOE_ACT_IDENTITY) return z;
  const double s = 1.0 / (1.0 + exp(-z));
  return z * s;
}

__device__ __forceinline__ double act_grad(int act, double z) {
  if (act == SMOE_ACT_GELU)
    return 0.5 * (1.0 + erf(z * 0.70710678118654752440)) + z * exp(-0.5 * z * z) * 0.39894228040143272;
  if (act == SMOE_ACT_RELU) return z > 0.0 ? 1.0 : 0.0;
  if (act == SMOE_ACT_IDENTITY) return 1.0;
  const double s = 1.0 / (1.0 + exp(-z));
  return s * (1.0 + z * (1.0 - s));
}

// Fast variants for the bf16 tensor-core epilogues.  erf uses Abramowitz &
// Stegun 7.1.26 (|error| <= 1.5e-7, plus MUFU rcp/ex2 rounding, ~3e-7 total) —
// three orders of magnitude below the bf16 rounding (2^-9) applied to the
// result, so the exact-erf GELU semantics of the reference are kept.  The
// fp32 check mode (SIMT kernels) uses act_fwd/act_grad above.
struct ErfExp {
  float erf;   // erf(z / sqrt(2))
  float gexp;  // exp(-z^2 / 2)
};
__device__ __forceinline__ ErfExp erf_scaled(float z) {
  const float x = fabsf(z) * 0.70710678118654752f;
  const float t = __fdividef(1.0f, fmaf(0.3275911f, x, 1.0f));
  float poly = fmaf(1.061405429f, t, -1.453152027f);
  poly = fmaf(poly, t, 1.421413741f);
  poly = fmaf(poly, t, -0.284496736f);
  poly = fmaf(poly, t, 0.254829592f);
  poly *= t;
  const float e = __expf(-0.5f * z * z);
  const float y = fmaf(-poly, e, 1.0f);
  return {copysignf(y, z), e};
}

__device__ __forceinline__ float act_fwd_fast(int act, float z) {
  if (act == SMOE_ACT_GELU) {
    const ErfExp r = erf_scaled(z);
    return 0.5f * z * (1.0f + r.erf);
  }
  if (act == SMOE_ACT_RELU) return z > 0.0f ? z : 0.0f;
  if (act == SMOE_ACT_IDENTITY) return z;
  return __fdividef(z, 1.0f + __expf(-z));
}

__device__ __forceinline__ float act_grad_fast(int act, float z) {
  if (act == SMOE_ACT_GELU) {
    const ErfExp r = erf_scaled(z);
    return fmaf(z * 0.39894228040143268f, r.gexp, 0.5f * (1.0f + r.erf));
  }
  if (act == SMOE_ACT_RELU) return z > 0.0f ? 1.0f : 0.0f;
  if (act == SMOE_ACT_IDENTITY) return 1.0f;
  const float s = __fdividef(1.0f, 1.0f + __expf(-z));
  return s * (1.0f + z * (1.0f - s));
}

// act(z) and act'(z) together (GELU shares one erf / exp evaluation).
__device__ __forceinline__ void act_both_fast(int act, float z, float &f, float &g) {
  if (act == SMOE_ACT_GELU) {
    const ErfExp r = erf_scaled(z);
    f = 0.5f * z * (1.0f + r.erf);
    g = fmaf(z * 0.39894228040143268f, r.gexp, 0.5f * (1.0f + r.erf));
    return;
  }
  f = act_fwd_fast(act, z);
  g = act_grad_fast(act, z);
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
