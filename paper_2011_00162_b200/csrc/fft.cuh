// Register/shared-memory 2-D FFT engine for square power-of-two frames.
//
// Replaces the reference's FFTW call (proj/src/fft.cpp:39-50: unitary DFT2,
// forward sign -1).  The 1/S normalisation is applied by the caller where it
// is folded into other arithmetic.
//
// Decomposition (per axis, length S = R * G):
//   X[k2 + R*k1] = sum_g W_G^{g k1} * ( W_S^{g k2} * sum_m x[g + G m] W_R^{m k2} )
// Step 1: each thread owns one g and R elements (stride G) -> radix-R DFT in
//         registers, twiddle W_S^{g k2}.
// Step 2: radix-G DFTs across the G threads of a line, through shared memory.
// A frame is S lines x G threads = NT threads; every thread holds R complex
// values in registers throughout, so shared memory is touched only at the
// three exchanges of each 2-D transform (row step1->step2, row->column,
// column step1->step2).  The inverse is the exact mirror of the forward and
// starts from the register layout the forward ends in, so the Fourier-domain
// work (ST-AGM prox, Gamma update) sits between them with no extra exchange.
//
// Layouts (t = thread index within the frame):
//   spatial / row layout : y = t / G, g = t % G, v[m] = x(y, g + G m)
//   Fourier / col layout : x = t % S, c = t / S,
//                          v[q G + k1] = X(ky = (c + G q) + R k1, kx = x)
// Fourier-layout global accesses are coalesced along kx (lanes = consecutive x).
//
// Shared memory: one S x P complex tile per frame, P = S + G (or S + 1 when
// G == 1), with a rotation swizzle on the row intermediate; the combination
// was checked bank-conflict-free for every row access pattern (8 and 16 B
// elements) with a bank simulator before being adopted.
#pragma once

#include "cx.cuh"

namespace pdd {

// a * W_N^K; forward W = exp(-2 pi i/N), inverse exp(+2 pi i/N).  N | 64.
template <bool INV, int K, int N, typename T>
__device__ __forceinline__ cx<T> twk(cx<T> a) {
  constexpr int k = ((K % N) + N) % N;
  if constexpr (k == 0) {
    return a;
  } else if constexpr (2 * k == N) {
    return -a;
  } else if constexpr (4 * k == N) {
    if constexpr (INV) return cx<T>{-a.y, a.x};
    else return cx<T>{a.y, -a.x};
  } else if constexpr (4 * k == 3 * N) {
    if constexpr (INV) return cx<T>{a.y, -a.x};
    else return cx<T>{-a.y, a.x};
  } else {
    constexpr int m = k * (64 / N);
    constexpr T c = T(cos64(m));
    constexpr T s = INV ? T(sin64(m)) : T(-sin64(m));
    return a * cx<T>{c, s};
  }
}

// In-register DFT of N (power of two, <= 64) values, natural order in/out.
template <int N, bool INV, typename T>
__device__ __forceinline__ void dft(cx<T>* a) {
  if constexpr (N > 1) {
    constexpr int L = ilog2(N);
    static_for<L>([&](auto S) {
      constexpr int half = N >> (S + 1);
      static_for<N / 2>([&](auto B) {
        constexpr int grp = B / half, k = B % half;
        constexpr int i0 = grp * 2 * half + k, i1 = i0 + half;
        const cx<T> x = a[i0], y = a[i1];
        a[i0] = x + y;
        a[i1] = twk<INV, k*(N / (2 * half)), N>(x - y);
      });
    });
    cx<T> t[N];
    static_for<N>([&](auto I) { t[I] = a[bitrev(I, L)]; });
    static_for<N>([&](auto I) { a[I] = t[I]; });
  }
}

template <typename T, int S_, int R_>
struct Fft2 {
  static constexpr int S = S_;
  static constexpr int R = R_;
  static constexpr int G = S / R;
  static constexpr int NT = S * G;
  static constexpr int P = S + (G > 1 ? G : 1);
  static constexpr int TILE = S * P;  // shared elements per frame
  static_assert(R >= G && R % G == 0, "Fft2: need R >= G, G | R");
  static_assert((S & (S - 1)) == 0, "Fft2: power-of-two S");

  __device__ static __forceinline__ int swz(int k2, int g) { return k2 * G + ((g + k2) & (G - 1)); }

  // v: row layout in, Fourier (col) layout out.  tw[k] = W_S^k (forward).
  __device__ static __forceinline__ void forward(cx<T>* v, cx<T>* buf, const cx<T>* tw, int t) {
    {
      const int y = t / G, g = t % G;
      dft<R, false>(v);
      if constexpr (G == 1) {
        static_for<R>([&](auto K) { buf[y * P + K] = v[K]; });
      } else {
        static_for<R>([&](auto K) {
          buf[y * P + swz(K, g)] = (K == 0) ? v[K] : v[K] * tw[g * K];
        });
        __syncwarp();
        static_for<R / G>([&](auto Q) {
          const int k2 = g + G * Q;
          static_for<G>([&](auto GP) { v[Q * G + GP] = buf[y * P + k2 * G + ((GP + k2) & (G - 1))]; });
          dft<G, false>(v + Q * G);
        });
        __syncwarp();
        static_for<R / G>([&](auto Q) {
          const int k2 = g + G * Q;
          static_for<G>([&](auto K1) { buf[y * P + k2 + R * K1] = v[Q * G + K1]; });
        });
      }
    }
    __syncthreads();
    const int x = t % S, c = t / S;
    static_for<R>([&](auto M) { v[M] = buf[(c + G * M) * P + x]; });
    dft<R, false>(v);
    if constexpr (G > 1) {
      static_for<R>([&](auto K) { buf[(K * G + c) * P + x] = (K == 0) ? v[K] : v[K] * tw[c * K]; });
      __syncthreads();
      static_for<R / G>([&](auto Q) {
        const int k2 = c + G * Q;
        static_for<G>([&](auto GP) { v[Q * G + GP] = buf[(k2 * G + GP) * P + x]; });
        dft<G, false>(v + Q * G);
      });
    }
  }

  // v: Fourier (col) layout in, row layout out (unnormalised inverse).
  __device__ static __forceinline__ void inverse(cx<T>* v, cx<T>* buf, const cx<T>* tw, int t) {
    {
      const int x = t % S, c = t / S;
      if constexpr (G > 1) {
        static_for<R / G>([&](auto Q) {
          const int k2 = c + G * Q;
          dft<G, true>(v + Q * G);
          static_for<G>([&](auto GP) { buf[(k2 * G + GP) * P + x] = v[Q * G + GP]; });
        });
        __syncthreads();
        static_for<R>([&](auto K) {
          const cx<T> a = buf[(K * G + c) * P + x];
          v[K] = (K == 0) ? a : mul_conj(a, tw[c * K]);
        });
      }
      dft<R, true>(v);
      static_for<R>([&](auto M) { buf[(c + G * M) * P + x] = v[M]; });
    }
    __syncthreads();
    const int y = t / G, g = t % G;
    if constexpr (G == 1) {
      static_for<R>([&](auto K) { v[K] = buf[y * P + K]; });
    } else {
      static_for<R / G>([&](auto Q) {
        const int k2 = g + G * Q;
        static_for<G>([&](auto K1) { v[Q * G + K1] = buf[y * P + k2 + R * K1]; });
        dft<G, true>(v + Q * G);
      });
      __syncwarp();
      static_for<R / G>([&](auto Q) {
        const int k2 = g + G * Q;
        static_for<G>([&](auto GP) { buf[y * P + k2 * G + ((GP + k2) & (G - 1))] = v[Q * G + GP]; });
      });
      __syncwarp();
      static_for<R>([&](auto K) {
        const cx<T> a = buf[y * P + swz(K, g)];
        v[K] = (K == 0) ? a : mul_conj(a, tw[g * K]);
      });
    }
    dft<R, true>(v);
  }
};

}  // namespace pdd
