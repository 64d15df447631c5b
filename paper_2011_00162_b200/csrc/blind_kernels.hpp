// Launchers of the blind probe-side kernels (blind_kernels.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "cx.cuh"

namespace pdd {

template <typename T>
cudaError_t launch_probe_partials(const cx<T>* img, const int64_t* off, const int32_t* pitch, const cx<T>* q,
                                  const int32_t* chunk_f0, const int32_t* chunk_f1, int nchunks, int S, int mode,
                                  cx<T>* num_part, T* den_part, const int* skip, cudaStream_t st);
template <typename T>
cudaError_t launch_chunk_reduce(const cx<T>* num_part, const T* den_part, const int32_t* seg_beg, int nseg, int SS,
                                cx<T>* num, T* den, const int* skip, cudaStream_t st);
template <typename T>
cudaError_t launch_probe_update(const cx<T>* num, const T* den, const cx<T>* w, cx<T>* wc, cx<T>* delta,
                                cx<T>* wd_all, const int* local_map, int nls, int SS, T eta, T mu, const int* skip,
                                cudaStream_t st);
template <typename T>
cudaError_t launch_probe_avg(const cx<T>* wd_all, int D, int SS, cx<T>* avg, const int* skip, cudaStream_t st);
template <typename T>
cudaError_t launch_apply_mask(cx<T>* spec, const T* mask, int SS, const int* skip, cudaStream_t st);
template <typename T>
cudaError_t launch_checker(const T* amp, int64_t nfr, int S, cx<T>* out, cudaStream_t st);
template <typename T>
cudaError_t launch_frame_flux(const T* amp, int64_t nfr, int64_t per, double* out, cudaStream_t st);
template <typename T>
cudaError_t launch_scale_copy(const cx<T>* in, cx<T>* out, int64_t n, double scale, int copies, int64_t stride,
                              cudaStream_t st);

}  // namespace pdd
