// ORACLE TEST INFRASTRUCTURE — not product code.  See fftw3.h for scope.
//
// 2-D complex DFT over a row-major n0 x n1 array: row transforms in place,
// then column transforms in blocks of kBlock columns gathered into a
// contiguous per-call scratch (so concurrent fftw_execute_dft calls on one
// plan are safe, as FFTW guarantees and the reference relies on:
// proj/src/fft.cpp:9-10).  Power-of-two lengths use an iterative radix-2
// decimation-in-time transform with a precomputed twiddle table; other lengths
// a direct O(n^2) DFT.  Sign convention and lack of normalisation follow FFTW.
#include "fftw3.h"

#include <cmath>
#include <complex>
#include <cstring>
#include <stdexcept>
#include <vector>

namespace {

using cd = std::complex<double>;
constexpr int kBlock = 8;

struct Axis {
  int n = 0;
  bool pow2 = false;
  std::vector<cd> tw;       // exp(sign*2*pi*i*k/n), k in [0,n)
  std::vector<int> bitrev;  // pow2 only

  void init(int len, int sign) {
    n = len;
    pow2 = len > 0 && (len & (len - 1)) == 0;
    tw.resize(static_cast<size_t>(len));
    for (int k = 0; k < len; ++k) {
      const double ang = sign * 2.0 * M_PI * static_cast<double>(k) / static_cast<double>(len);
      tw[k] = cd(std::cos(ang), std::sin(ang));
    }
    if (pow2) {
      bitrev.resize(static_cast<size_t>(len));
      int bits = 0;
      while ((1 << bits) < len) ++bits;
      for (int i = 0; i < len; ++i) {
        int r = 0;
        for (int b = 0; b < bits; ++b)
          if (i & (1 << b)) r |= 1 << (bits - 1 - b);
        bitrev[i] = r;
      }
    }
  }

  // Transform B interleaved sequences: element k of sequence b is a[k*B + b].
  template <int B>
  void run(cd* a, cd* scratch) const {
    if (n <= 1) return;
    if (pow2) {
      for (int i = 0; i < n; ++i) {
        const int r = bitrev[i];
        if (r > i)
          for (int b = 0; b < B; ++b) std::swap(a[i * B + b], a[r * B + b]);
      }
      for (int len = 2; len <= n; len <<= 1) {
        const int half = len >> 1;
        const int stride = n / len;
        for (int i = 0; i < n; i += len)
          for (int k = 0; k < half; ++k) {
            const cd w = tw[static_cast<size_t>(k) * stride];
            cd* p = a + static_cast<size_t>(i + k) * B;
            cd* q = a + static_cast<size_t>(i + k + half) * B;
            for (int b = 0; b < B; ++b) {
              const double vr = q[b].real() * w.real() - q[b].imag() * w.imag();
              const double vi = q[b].real() * w.imag() + q[b].imag() * w.real();
              const double ur = p[b].real(), ui = p[b].imag();
              p[b] = cd(ur + vr, ui + vi);
              q[b] = cd(ur - vr, ui - vi);
            }
          }
      }
      return;
    }
    // Direct DFT for non-power-of-two lengths.
    std::memcpy(static_cast<void*>(scratch), a, sizeof(cd) * static_cast<size_t>(n) * B);
    for (int k = 0; k < n; ++k)
      for (int b = 0; b < B; ++b) {
        cd s(0.0, 0.0);
        for (int t = 0; t < n; ++t)
          s += scratch[static_cast<size_t>(t) * B + b] *
               tw[(static_cast<int64_t>(k) * t) % n];
        a[static_cast<size_t>(k) * B + b] = s;
      }
  }
};

}  // namespace

struct pdd_fftw_plan_s {
  int n0 = 0, n1 = 0;
  Axis rows;  // transform along a row (length n1)
  Axis cols;  // transform along a column (length n0)
  fftw_complex* in = nullptr;
  fftw_complex* out = nullptr;
};

extern "C" {

fftw_plan fftw_plan_dft_2d(int n0, int n1, fftw_complex* in, fftw_complex* out, int sign,
                           unsigned /*flags*/) {
  if (n0 < 1 || n1 < 1) return nullptr;
  auto* p = new pdd_fftw_plan_s;
  p->n0 = n0;
  p->n1 = n1;
  p->rows.init(n1, sign);
  p->cols.init(n0, sign);
  p->in = in;
  p->out = out;
  return p;
}

void fftw_execute_dft(const fftw_plan p, fftw_complex* in, fftw_complex* out) {
  const int n0 = p->n0, n1 = p->n1;
  cd* a = reinterpret_cast<cd*>(out);
  if (in != out)
    std::memcpy(static_cast<void*>(a), in, sizeof(cd) * static_cast<size_t>(n0) * n1);
  const int scratch_len = std::max(n0, n1) * kBlock;
  std::vector<cd> scratch(static_cast<size_t>(scratch_len) * 2);
  cd* blk = scratch.data();
  cd* tmp = scratch.data() + scratch_len;
  for (int r = 0; r < n0; ++r) p->rows.run<1>(a + static_cast<size_t>(r) * n1, tmp);
  int c = 0;
  for (; c + kBlock <= n1; c += kBlock) {
    for (int r = 0; r < n0; ++r)
      for (int b = 0; b < kBlock; ++b) blk[r * kBlock + b] = a[static_cast<size_t>(r) * n1 + c + b];
    p->cols.run<kBlock>(blk, tmp);
    for (int r = 0; r < n0; ++r)
      for (int b = 0; b < kBlock; ++b) a[static_cast<size_t>(r) * n1 + c + b] = blk[r * kBlock + b];
  }
  for (; c < n1; ++c) {
    for (int r = 0; r < n0; ++r) blk[r] = a[static_cast<size_t>(r) * n1 + c];
    p->cols.run<1>(blk, tmp);
    for (int r = 0; r < n0; ++r) a[static_cast<size_t>(r) * n1 + c] = blk[r];
  }
}

void fftw_execute(const fftw_plan p) { fftw_execute_dft(p, p->in, p->out); }

void fftw_destroy_plan(fftw_plan p) { delete p; }

}  // extern "C"
