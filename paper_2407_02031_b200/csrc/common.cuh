// common.cuh — shared helpers for the sdb C-ABI library (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>
#include <string>

#include "../../include/sdb_api.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "this library is written for sm_100a (B200) only"
#endif

namespace sdb {

// Thread-local error string behind sdb_last_error().
void set_error(const std::string& msg);

inline int fail(int code, const std::string& msg) {
  set_error(msg);
  return code;
}

// Check the launch that was just issued (does not synchronise).
inline int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    return fail(SDB_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
  }
  return SDB_OK;
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// ---- programmatic dependent launch (PDL) ------------------------------------
// Every streaming kernel of this library is launched with the programmatic-
// stream-serialisation attribute and begins with pdl_wait() (griddepcontrol.
// wait) before it touches memory the previous kernel on its stream may read or
// write: the launch and CTA rasterisation of kernel k+1 then overlap the tail
// of kernel k (a cuBLAS / cuDNN kernel or one of ours) instead of following
// its completion.  Inside CUDA graphs the attribute becomes a programmatic
// edge.  Kernels never trigger early (no griddepcontrol.launch_dependents):
// the dependent launches as the last CTA of its predecessor exits, so it can
// never occupy SM slots its predecessor's later waves need, and a kernel that
// starts early has only ever its immediate predecessor in flight.  Only state
// that predecessor cannot touch (weights, gamma / beta, the per-request K/V
// cache, shared memory, tensor maps) is read before the wait.
extern int g_pdl;   // 1 = launch with PDL (default), 0 = plain launches (SDB_PDL=0 / sdb_set_pdl)
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline void launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = g_pdl ? 1 : 0;
  cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// ---- scalar conversions -------------------------------------------------
template <typename T> __device__ __forceinline__ float to_f32(T v);
template <> __device__ __forceinline__ float to_f32<float>(float v) { return v; }
template <> __device__ __forceinline__ float to_f32<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }
template <> __device__ __forceinline__ float to_f32<__half>(__half v) { return __half2float(v); }

template <typename T> __device__ __forceinline__ T from_f32(float v);
template <> __device__ __forceinline__ float from_f32<float>(float v) { return v; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f32<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }
template <> __device__ __forceinline__ __half from_f32<__half>(float v) { return __float2half_rn(v); }

// ---- 8-element vector load/store (16 B for 2-byte types, 2x16 B for fp32) --
template <typename T> struct Vec8;
template <> struct Vec8<float> {
  static __device__ __forceinline__ void load(const float* p, float (&v)[8]) {
    float4 a = *reinterpret_cast<const float4*>(p);
    float4 b = *reinterpret_cast<const float4*>(p + 4);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
    v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  }
  static __device__ __forceinline__ void store(float* p, const float (&v)[8]) {
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
    *reinterpret_cast<float4*>(p + 4) = make_float4(v[4], v[5], v[6], v[7]);
  }
};
template <typename T2> struct Vec8Half {
  template <typename T>
  static __device__ __forceinline__ void load(const T* p, float (&v)[8]) {
    uint4 u = *reinterpret_cast<const uint4*>(p);
    const T* h = reinterpret_cast<const T*>(&u);
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = to_f32<T>(h[i]);
  }
  template <typename T>
  static __device__ __forceinline__ void store(T* p, const float (&v)[8]) {
    uint4 u;
    T* h = reinterpret_cast<T*>(&u);
#pragma unroll
    for (int i = 0; i < 8; ++i) h[i] = from_f32<T>(v[i]);
    *reinterpret_cast<uint4*>(p) = u;
  }
};
template <> struct Vec8<__nv_bfloat16> {
  static __device__ __forceinline__ void load(const __nv_bfloat16* p, float (&v)[8]) { Vec8Half<int>::load(p, v); }
  static __device__ __forceinline__ void store(__nv_bfloat16* p, const float (&v)[8]) { Vec8Half<int>::store(p, v); }
};
template <> struct Vec8<__half> {
  static __device__ __forceinline__ void load(const __half* p, float (&v)[8]) { Vec8Half<int>::load(p, v); }
  static __device__ __forceinline__ void store(__half* p, const float (&v)[8]) { Vec8Half<int>::store(p, v); }
};

// ---- 8 elements held as raw registers until consumed ----------------------
// (loads issued early without unpacking: 4 registers per 16-bit vector)
template <typename T> struct Raw8 { uint4 u; };
template <> struct Raw8<float> { float4 a, b; };

template <typename T>
__device__ __forceinline__ Raw8<T> load_raw(const T* p) {
  Raw8<T> r;
  r.u = *reinterpret_cast<const uint4*>(p);
  return r;
}
template <>
__device__ __forceinline__ Raw8<float> load_raw<float>(const float* p) {
  Raw8<float> r;
  r.a = *reinterpret_cast<const float4*>(p);
  r.b = *reinterpret_cast<const float4*>(p + 4);
  return r;
}
template <typename T>
__device__ __forceinline__ void store_raw(T* p, const Raw8<T>& r) {
  *reinterpret_cast<uint4*>(p) = r.u;
}
template <>
__device__ __forceinline__ void store_raw<float>(float* p, const Raw8<float>& r) {
  *reinterpret_cast<float4*>(p) = r.a;
  *reinterpret_cast<float4*>(p + 4) = r.b;
}
template <typename T>
__device__ __forceinline__ void unpack(const Raw8<T>& r, float (&v)[8]) {
  const T* h = reinterpret_cast<const T*>(&r.u);
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = to_f32<T>(h[i]);
}
template <>
__device__ __forceinline__ void unpack<float>(const Raw8<float>& r, float (&v)[8]) {
  v[0] = r.a.x; v[1] = r.a.y; v[2] = r.a.z; v[3] = r.a.w;
  v[4] = r.b.x; v[5] = r.b.y; v[6] = r.b.z; v[7] = r.b.w;
}

// element pair i (0..3) of a raw vector as float2, and back (round to nearest)
template <typename T> __device__ __forceinline__ float2 get_pair(const Raw8<T>& r, int i);
template <> __device__ __forceinline__ float2 get_pair<__nv_bfloat16>(const Raw8<__nv_bfloat16>& r, int i) {
  const uint32_t u = (&r.u.x)[i];
  return make_float2(__uint_as_float(u << 16), __uint_as_float(u & 0xffff0000u));
}
template <> __device__ __forceinline__ float2 get_pair<__half>(const Raw8<__half>& r, int i) {
  const uint32_t u = (&r.u.x)[i];
  return __half22float2(*reinterpret_cast<const __half2*>(&u));
}
template <> __device__ __forceinline__ float2 get_pair<float>(const Raw8<float>& r, int i) {
  const float4& q = i < 2 ? r.a : r.b;
  return (i & 1) ? make_float2(q.z, q.w) : make_float2(q.x, q.y);
}
template <typename T> __device__ __forceinline__ void set_pair(Raw8<T>& r, int i, float2 v);
template <> __device__ __forceinline__ void set_pair<__nv_bfloat16>(Raw8<__nv_bfloat16>& r, int i, float2 v) {
  __nv_bfloat162 h = __floats2bfloat162_rn(v.x, v.y);
  (&r.u.x)[i] = *reinterpret_cast<uint32_t*>(&h);
}
template <> __device__ __forceinline__ void set_pair<__half>(Raw8<__half>& r, int i, float2 v) {
  __half2 h = __floats2half2_rn(v.x, v.y);
  (&r.u.x)[i] = *reinterpret_cast<uint32_t*>(&h);
}
template <> __device__ __forceinline__ void set_pair<float>(Raw8<float>& r, int i, float2 v) {
  float4& q = i < 2 ? r.a : r.b;
  if (i & 1) { q.z = v.x; q.w = v.y; } else { q.x = v.x; q.y = v.y; }
}

// ---- packed fp32x2 arithmetic (sm_100 FFMA2 / FMUL2 / FADD2: two lanes of
// work per issue slot; each lane rounds exactly like the scalar op) ----------
__device__ __forceinline__ uint64_t f2_bits(float2 a) { return *reinterpret_cast<uint64_t*>(&a); }
__device__ __forceinline__ float2 f2_from(uint64_t b) { return *reinterpret_cast<float2*>(&b); }
__device__ __forceinline__ float2 f2fma(float2 a, float2 b, float2 c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(f2_bits(a)), "l"(f2_bits(b)), "l"(f2_bits(c)));
  return f2_from(d);
}
__device__ __forceinline__ float2 f2mul(float2 a, float2 b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2_bits(a)), "l"(f2_bits(b)));
  return f2_from(d);
}
__device__ __forceinline__ float2 f2add(float2 a, float2 b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2_bits(a)), "l"(f2_bits(b)));
  return f2_from(d);
}
__device__ __forceinline__ float2 f2s(float s) { return make_float2(s, s); }

// SiLU of two lanes given nw = -w (callers negate the affine coefficients
// once): w sigmoid(w) = nw * y with y = -1 / (1 + 2^(nw log2 e)).  2^ on the
// MUFU; y from a bit-trick seed (rel. error <= 5.1%) and two PACKED Newton
// steps y <- y (2 + d y) on the FMA pipe (rel. error <= 6.7e-6, far below a
// 16-bit ulp): 17 issue slots per pair where the scalar form took 21.  Bitwise
// equal to w * r with r the positive-seed scalar Newton reciprocal.
__device__ __forceinline__ float2 silu2_neg(float2 nw) {
  float2 t = f2mul(nw, f2s(1.4426950408889634f));
  t.x = fminf(t.x, 126.f);
  t.y = fminf(t.y, 126.f);
  float2 e;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e.x) : "f"(t.x));
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e.y) : "f"(t.y));
  const float2 d = f2add(e, f2s(1.f));
  float2 y = make_float2(__uint_as_float(0xFEF311C3u - __float_as_uint(d.x)),
                         __uint_as_float(0xFEF311C3u - __float_as_uint(d.y)));
  y = f2mul(y, f2fma(d, y, f2s(2.f)));
  y = f2mul(y, f2fma(d, y, f2s(2.f)));
  return f2mul(nw, y);
}

inline int dtype_size(int dt) {
  switch (dt) {
    case SDB_F32: return 4;
    case SDB_BF16: return 2;
    case SDB_F16: return 2;
    default: return 0;
  }
}

constexpr int kNumSMs = 148;

}  // namespace sdb
