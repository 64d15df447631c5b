// Phase breakdown of the streamed SWEEP kernel (developer tool, not shipped):
// nvcc -DPDD_PHASE_TIMING ... scripts/phase_timing.cu -o scripts/bin/phase_timing
// Runs K1 on synthetic device data (config-4 frame geometry) and prints the
// average SM cycles per frame spent in rows-forward / column groups /
// rows-inverse / reduction+sync.
#include <cstdio>
#include <vector>

#include "../paper_2011_00162_b200/csrc/frame_stream.cuh"

using namespace pdd;

template <class SH, bool USE_TMEM>
void run(int nframes, int W) {
  constexpr int S = SH::S;
  const int64_t SS = static_cast<int64_t>(S) * S;
  const int H = S + 32 * 3;
  cx<float>*img, *probe, *tw, *g0, *g1, *bp;
  float* amp;
  int64_t* off;
  int32_t* pitch;
  double* rf;
  unsigned long long* cyc;
  cudaMalloc(&img, sizeof(cx<float>) * H * W);
  cudaMalloc(&probe, sizeof(cx<float>) * SS);
  cudaMalloc(&tw, sizeof(cx<float>) * S);
  cudaMalloc(&g0, sizeof(cx<float>) * SS * nframes);
  cudaMalloc(&g1, sizeof(cx<float>) * SS * nframes);
  cudaMalloc(&bp, sizeof(cx<float>) * SS * nframes);
  cudaMalloc(&amp, sizeof(float) * SS * nframes);
  cudaMalloc(&off, sizeof(int64_t) * nframes);
  cudaMalloc(&pitch, sizeof(int32_t) * nframes);
  cudaMalloc(&rf, sizeof(double) * nframes);
  cudaMalloc(&cyc, sizeof(unsigned long long) * 4);
  cudaMemset(img, 0, sizeof(cx<float>) * H * W);
  cudaMemset(probe, 0, sizeof(cx<float>) * SS);
  cudaMemset(g0, 0, sizeof(cx<float>) * SS * nframes);
  cudaMemset(amp, 0, sizeof(float) * SS * nframes);
  std::vector<cx<float>> htw(S);
  for (int k = 0; k < S; ++k) htw[k] = {float(cos(-2 * M_PI * k / S)), float(sin(-2 * M_PI * k / S))};
  cudaMemcpy(tw, htw.data(), sizeof(cx<float>) * S, cudaMemcpyHostToDevice);
  std::vector<int64_t> ho(nframes);
  std::vector<int32_t> hp(nframes, W);
  const int per_row = (W - S) / 32 + 1;
  for (int f = 0; f < nframes; ++f) ho[f] = static_cast<int64_t>((f / per_row) % 4) * 32 * W + (f % per_row) * 32;
  cudaMemcpy(off, ho.data(), sizeof(int64_t) * nframes, cudaMemcpyHostToDevice);
  cudaMemcpy(pitch, hp.data(), sizeof(int32_t) * nframes, cudaMemcpyHostToDevice);
  FrameArgs<float> a;
  a.nframes = nframes;
  a.probe = probe;
  a.tw = tw;
  a.img = img;
  a.off = off;
  a.pitch = pitch;
  a.amp = amp;
  a.gamma_in = g0;
  a.gamma_out = g1;
  a.bp_out = bp;
  a.rf_part = rf;
  a.lam = 0.1f;
  a.eps = 0.5f;
  a.scale = 1.f / S;
  auto kern = sweep_stream_kernel<float, SH, true, USE_TMEM>;
  const size_t smem = stream_smem_bytes<float, SH>();
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  int bps = 0, sms = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kern, SH::NT, smem);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int grid = bps * sms;
  for (int rep = 0; rep < 2; ++rep) {
    cudaMemset(cyc, 0, sizeof(unsigned long long) * 4);
    a.phase_cycles = cyc;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    kern<<<grid, SH::NT, smem>>>(a);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long h[4];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    const double tot = double(h[0] + h[1] + h[2] + h[3]);
    printf("tmem=%d S=%d frames=%d grid=%d (%d/SM) %.3f ms  %.2f us/frame/SM | cycles/frame: rows_fwd %.0f  cols %.0f  rows_inv %.0f  tail %.0f (total %.0f) err=%s\n",
           int(USE_TMEM), S, nframes, grid, bps, ms, ms * 1e3 * grid / nframes, h[0] / double(nframes), h[1] / double(nframes),
           h[2] / double(nframes), h[3] / double(nframes), tot / nframes, cudaGetErrorString(cudaGetLastError()));
  }
}

int main() {
  run<StreamShape<128, 512, 8, 8>, false>(16384, 8192);
  run<StreamShape<128, 512, 8, 8>, true>(16384, 8192);
  run<StreamShape<64, 256, 4, 8, 2>, false>(32768, 4096);
  run<StreamShape<64, 256, 4, 8, 2>, true>(32768, 4096);
  return 0;
}
