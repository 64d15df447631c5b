// Complex arithmetic and compile-time helpers shared by every kernel.
//
// Complex values are interleaved (re, im) pairs -- the layout of
// std::complex<double> in the reference's ComplexField2D (field.hpp:48-91) --
// so host buffers cross the C-ABI without repacking.  cx<float> is one 8-byte
// and cx<double> one 16-byte aligned access.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <utility>

namespace pdd {

template <typename T>
struct alignas(2 * sizeof(T)) cx {
  T x, y;
};

template <typename T>
__host__ __device__ __forceinline__ cx<T> mk(T a, T b) {
  return cx<T>{a, b};
}
template <typename T>
__host__ __device__ __forceinline__ cx<T> operator+(cx<T> a, cx<T> b) {
  return {a.x + b.x, a.y + b.y};
}
template <typename T>
__host__ __device__ __forceinline__ cx<T> operator-(cx<T> a, cx<T> b) {
  return {a.x - b.x, a.y - b.y};
}
template <typename T>
__host__ __device__ __forceinline__ cx<T> operator-(cx<T> a) {
  return {-a.x, -a.y};
}
template <typename T>
__host__ __device__ __forceinline__ cx<T> operator*(cx<T> a, cx<T> b) {
  return {a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x};
}
template <typename T>
__host__ __device__ __forceinline__ cx<T> operator*(cx<T> a, T s) {
  return {a.x * s, a.y * s};
}
template <typename T>
__host__ __device__ __forceinline__ cx<T>& operator+=(cx<T>& a, cx<T> b) {
  a.x += b.x;
  a.y += b.y;
  return a;
}
// a * conj(b)
template <typename T>
__host__ __device__ __forceinline__ cx<T> mul_conj(cx<T> a, cx<T> b) {
  return {a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y};
}
template <typename T>
__host__ __device__ __forceinline__ cx<T> conjg(cx<T> a) {
  return {a.x, -a.y};
}
template <typename T>
__host__ __device__ __forceinline__ T norm2(cx<T> a) {
  return a.x * a.x + a.y * a.y;
}

// ---- complex64 on sm_100 packed FP32 ---------------------------------------
// Blackwell issues FADD2/FMUL2/FFMA2: one instruction on an (re, im) register
// pair.  The frame kernels are issue-bound (FADD/FMUL/FFMA were 65 % of the
// executed instructions of the streamed sweep), so complex64 add/sub is one
// instruction and a complex multiply two (FMUL2 by the broadcast real part,
// FFMA2 of the swapped operand by (-im, im); ptxas folds the swap and the
// partial negation into operand modifiers).  Host code keeps the scalar forms.
#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ >= 1000)
#define PDD_F32X2 1
namespace f32x2 {
__device__ __forceinline__ unsigned long long pk(float x, float y) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(x), "f"(y));
  return r;
}
__device__ __forceinline__ cx<float> up(unsigned long long v) {
  cx<float> r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
  return r;
}
__device__ __forceinline__ unsigned long long add(unsigned long long a, unsigned long long b) {
  unsigned long long d;
  asm("add.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ unsigned long long sub(unsigned long long a, unsigned long long b) {
  unsigned long long d;
  asm("sub.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ unsigned long long mul(unsigned long long a, unsigned long long b) {
  unsigned long long d;
  asm("mul.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ unsigned long long fma(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
}  // namespace f32x2
#endif

__host__ __device__ __forceinline__ cx<float> operator+(cx<float> a, cx<float> b) {
#ifdef PDD_F32X2
  return f32x2::up(f32x2::add(f32x2::pk(a.x, a.y), f32x2::pk(b.x, b.y)));
#else
  return {a.x + b.x, a.y + b.y};
#endif
}
__host__ __device__ __forceinline__ cx<float> operator-(cx<float> a, cx<float> b) {
#ifdef PDD_F32X2
  return f32x2::up(f32x2::sub(f32x2::pk(a.x, a.y), f32x2::pk(b.x, b.y)));
#else
  return {a.x - b.x, a.y - b.y};
#endif
}
__host__ __device__ __forceinline__ cx<float> operator*(cx<float> a, cx<float> b) {
#ifdef PDD_F32X2
  const unsigned long long t = f32x2::mul(f32x2::pk(a.x, a.y), f32x2::pk(b.x, b.x));
  return f32x2::up(f32x2::fma(f32x2::pk(a.y, a.x), f32x2::pk(-b.y, b.y), t));
#else
  return {a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x};
#endif
}
__host__ __device__ __forceinline__ cx<float> operator*(cx<float> a, float s) {
#ifdef PDD_F32X2
  return f32x2::up(f32x2::mul(f32x2::pk(a.x, a.y), f32x2::pk(s, s)));
#else
  return {a.x * s, a.y * s};
#endif
}
__host__ __device__ __forceinline__ cx<float>& operator+=(cx<float>& a, cx<float> b) {
  a = a + b;
  return a;
}
__host__ __device__ __forceinline__ cx<float> mul_conj(cx<float> a, cx<float> b) {
#ifdef PDD_F32X2
  const unsigned long long t = f32x2::mul(f32x2::pk(a.x, a.y), f32x2::pk(b.x, b.x));
  return f32x2::up(f32x2::fma(f32x2::pk(a.y, a.x), f32x2::pk(b.y, -b.y), t));
#else
  return {a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y};
#endif
}

// ---- compile-time loops ----------------------------------------------------
template <int... Is, class F>
__host__ __device__ __forceinline__ void static_for_impl(std::integer_sequence<int, Is...>, F&& f) {
  (f(std::integral_constant<int, Is>{}), ...);
}
template <int N, class F>
__host__ __device__ __forceinline__ void static_for(F&& f) {
  static_for_impl(std::make_integer_sequence<int, N>{}, f);
}

constexpr int ilog2(int n) { return n <= 1 ? 0 : 1 + ilog2(n / 2); }

constexpr int bitrev(int v, int bits) {
  int r = 0;
  for (int b = 0; b < bits; ++b)
    if (v & (1 << b)) r |= 1 << (bits - 1 - b);
  return r;
}

// cos(2*pi*k/64) for k in [0,16]; everything else by symmetry.
constexpr double kCos64[17] = {1.0,
                               0.9951847266721969,
                               0.9807852804032304,
                               0.9569403357322088,
                               0.9238795325112867,
                               0.881921264348355,
                               0.8314696123025452,
                               0.773010453362737,
                               0.7071067811865476,
                               0.6343932841636455,
                               0.5555702330196023,
                               0.4713967368259978,
                               0.38268343236508984,
                               0.29028467725446233,
                               0.19509032201612833,
                               0.09801714032956077,
                               0.0};

constexpr double cos64(int k) {
  k = ((k % 64) + 64) % 64;
  return k <= 16 ? kCos64[k] : k <= 32 ? -kCos64[32 - k] : k <= 48 ? -kCos64[k - 32] : kCos64[64 - k];
}
constexpr double sin64(int k) { return cos64(16 - k); }

}  // namespace pdd
