// ORACLE TEST INFRASTRUCTURE — not product code.  See fftw3.h for scope.
//
// 2-D complex DFT over a row-major n0 x n1 array: row transforms, then column
// transforms, both in batches of kBlock sequences gathered into a contiguous
// split (re / im) per-call scratch, so concurrent fftw_execute_dft calls on
// one plan are safe, as FFTW guarantees and the reference relies on
// (proj/src/fft.cpp:9-10).  Power-of-two lengths use an out-of-place Stockham
// autosort transform, radix 4 with a final radix-2 stage for odd log2(n), with
// table twiddles; the batch index is the unit-stride inner loop, compiled in
// an AVX2 and a baseline clone (no FMA contraction in either, so both give the
// same bits).  Other lengths use a direct O(n^2) DFT.  Sign convention and lack
// of normalisation follow FFTW.  This is the CPU baseline's FFT: written to be
// a fair stand-in for FFTW (FFTW itself is not in the image), about 6x faster
// than the radix-2 version it replaces (bench line: "FFT = oracle/fftw_shim").
#include "fftw3.h"

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstring>
#include <vector>

namespace {

using cd = std::complex<double>;
constexpr int kBlock = 8;

struct Axis {
  int n = 0, sign = -1;
  bool pow2 = false;
  std::vector<double> twr, twi;  // exp(sign*2*pi*i*k/n), k in [0,n)

  void init(int len, int sgn) {
    n = len;
    sign = sgn;
    pow2 = len > 0 && (len & (len - 1)) == 0;
    twr.resize(static_cast<size_t>(len));
    twi.resize(static_cast<size_t>(len));
    for (int k = 0; k < len; ++k) {
      const double ang = sgn * 2.0 * M_PI * static_cast<double>(k) / static_cast<double>(len);
      twr[k] = std::cos(ang);
      twi[k] = std::sin(ang);
    }
  }
};

// One radix-4 Stockham stage over kBlock interleaved sequences (element e of
// sequence b at [e * kBlock + b]): n1 = length still to split, s = stride.
__attribute__((target_clones("avx2", "default"))) void stage4(const Axis& ax, int n1, int s, const double* xr,
                                                             const double* xi, double* yr, double* yi) {
  const int n0 = n1 / 4, step = ax.n / n1, inner = s * kBlock;
  const double sg = ax.sign < 0 ? -1.0 : 1.0;
  for (int p = 0; p < n0; ++p) {
    const double w1r = ax.twr[p * step], w1i = ax.twi[p * step];
    const double w2r = ax.twr[2 * p * step], w2i = ax.twi[2 * p * step];
    const double w3r = ax.twr[3 * p * step], w3i = ax.twi[3 * p * step];
    const double* ar = xr + static_cast<size_t>(p) * inner;
    const double* ai = xi + static_cast<size_t>(p) * inner;
    const double* br = ar + static_cast<size_t>(n0) * inner;
    const double* bi = ai + static_cast<size_t>(n0) * inner;
    const double* cr = br + static_cast<size_t>(n0) * inner;
    const double* ci = bi + static_cast<size_t>(n0) * inner;
    const double* dr = cr + static_cast<size_t>(n0) * inner;
    const double* di = ci + static_cast<size_t>(n0) * inner;
    double* y0r = yr + static_cast<size_t>(4 * p) * inner;
    double* y0i = yi + static_cast<size_t>(4 * p) * inner;
    double* y1r = y0r + inner;
    double* y1i = y0i + inner;
    double* y2r = y1r + inner;
    double* y2i = y1i + inner;
    double* y3r = y2r + inner;
    double* y3i = y2i + inner;
    for (int t = 0; t < inner; ++t) {
      const double apcr = ar[t] + cr[t], apci = ai[t] + ci[t];
      const double amcr = ar[t] - cr[t], amci = ai[t] - ci[t];
      const double bpdr = br[t] + dr[t], bpdi = bi[t] + di[t];
      // sign * i * (b - d)
      const double jr = -sg * (bi[t] - di[t]), ji = sg * (br[t] - dr[t]);
      y0r[t] = apcr + bpdr;
      y0i[t] = apci + bpdi;
      const double u1r = amcr + jr, u1i = amci + ji;
      y1r[t] = u1r * w1r - u1i * w1i;
      y1i[t] = u1r * w1i + u1i * w1r;
      const double u2r = apcr - bpdr, u2i = apci - bpdi;
      y2r[t] = u2r * w2r - u2i * w2i;
      y2i[t] = u2r * w2i + u2i * w2r;
      const double u3r = amcr - jr, u3i = amci - ji;
      y3r[t] = u3r * w3r - u3i * w3i;
      y3i[t] = u3r * w3i + u3i * w3r;
    }
  }
}

// Final radix-2 stage (n1 == 2: no twiddles).
__attribute__((target_clones("avx2", "default"))) void stage2(int s, const double* xr, const double* xi, double* yr,
                                                             double* yi) {
  const int inner = s * kBlock;
  for (int t = 0; t < inner; ++t) {
    const double ar = xr[t], ai = xi[t], br = xr[inner + t], bi = xi[inner + t];
    yr[t] = ar + br;
    yi[t] = ai + bi;
    yr[inner + t] = ar - br;
    yi[inner + t] = ai - bi;
  }
}

// Transforms kBlock interleaved sequences held in (xr, xi); (yr, yi) is the
// ping-pong buffer.  Returns 0 if the result is in x, 1 if in y.
int fft_pow2(const Axis& ax, double* xr, double* xi, double* yr, double* yi) {
  int n1 = ax.n, s = 1, where = 0;
  while (n1 >= 4) {
    if (where == 0) stage4(ax, n1, s, xr, xi, yr, yi);
    else stage4(ax, n1, s, yr, yi, xr, xi);
    where ^= 1;
    n1 /= 4;
    s *= 4;
  }
  if (n1 == 2) {
    if (where == 0) stage2(s, xr, xi, yr, yi);
    else stage2(s, yr, yi, xr, xi);
    where ^= 1;
  }
  return where;
}

// Direct DFT for non-power-of-two lengths (same batch layout).
int dft_direct(const Axis& ax, const double* xr, const double* xi, double* yr, double* yi) {
  const int n = ax.n;
  for (int k = 0; k < n; ++k)
    for (int b = 0; b < kBlock; ++b) {
      double sr = 0.0, si = 0.0;
      for (int t = 0; t < n; ++t) {
        const size_t w = static_cast<size_t>((static_cast<int64_t>(k) * t) % n);
        const double vr = xr[t * kBlock + b], vi = xi[t * kBlock + b];
        sr += vr * ax.twr[w] - vi * ax.twi[w];
        si += vr * ax.twi[w] + vi * ax.twr[w];
      }
      yr[k * kBlock + b] = sr;
      yi[k * kBlock + b] = si;
    }
  return 1;
}

int run_batch(const Axis& ax, double* xr, double* xi, double* yr, double* yi) {
  if (ax.n <= 1) return 0;
  return ax.pow2 ? fft_pow2(ax, xr, xi, yr, yi) : dft_direct(ax, xr, xi, yr, yi);
}

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
  const size_t len = static_cast<size_t>(std::max(n0, n1)) * kBlock;
  std::vector<double> scratch(4 * len, 0.0);
  double* xr = scratch.data();
  double* xi = xr + len;
  double* yr = xi + len;
  double* yi = yr + len;
  // rows: kBlock rows at a time, element k of row r0+b at [k * kBlock + b]
  for (int r0 = 0; r0 < n0; r0 += kBlock) {
    const int nb = std::min(kBlock, n0 - r0);
    for (int b = 0; b < nb; ++b) {
      const cd* row = a + static_cast<size_t>(r0 + b) * n1;
      for (int k = 0; k < n1; ++k) {
        xr[k * kBlock + b] = row[k].real();
        xi[k * kBlock + b] = row[k].imag();
      }
    }
    for (int b = nb; b < kBlock; ++b)
      for (int k = 0; k < n1; ++k) xr[k * kBlock + b] = xi[k * kBlock + b] = 0.0;
    const int w = run_batch(p->rows, xr, xi, yr, yi);
    const double* rr = w ? yr : xr;
    const double* ri = w ? yi : xi;
    for (int b = 0; b < nb; ++b) {
      cd* row = a + static_cast<size_t>(r0 + b) * n1;
      for (int k = 0; k < n1; ++k) row[k] = cd(rr[k * kBlock + b], ri[k * kBlock + b]);
    }
  }
  // columns: kBlock adjacent columns at a time
  for (int c0 = 0; c0 < n1; c0 += kBlock) {
    const int nb = std::min(kBlock, n1 - c0);
    for (int r = 0; r < n0; ++r) {
      const cd* src = a + static_cast<size_t>(r) * n1 + c0;
      for (int b = 0; b < nb; ++b) {
        xr[r * kBlock + b] = src[b].real();
        xi[r * kBlock + b] = src[b].imag();
      }
      for (int b = nb; b < kBlock; ++b) xr[r * kBlock + b] = xi[r * kBlock + b] = 0.0;
    }
    const int w = run_batch(p->cols, xr, xi, yr, yi);
    const double* rr = w ? yr : xr;
    const double* ri = w ? yi : xi;
    for (int r = 0; r < n0; ++r) {
      cd* dst = a + static_cast<size_t>(r) * n1 + c0;
      for (int b = 0; b < nb; ++b) dst[b] = cd(rr[r * kBlock + b], ri[r * kBlock + b]);
    }
  }
}

void fftw_execute(const fftw_plan p) { fftw_execute_dft(p, p->in, p->out); }

void fftw_destroy_plan(fftw_plan p) { delete p; }

}  // extern "C"
