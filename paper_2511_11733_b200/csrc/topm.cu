// NormMatch for any top_m (norm_match, verifier.cpp:119-134 over top_ids,
// :40-51): the fused kernel selects up to kMaxTopM (32) ids per row in a warp;
// larger m (the reference accepts any 1 <= m <= V) goes through an exact sort
// of each row by (value desc, id asc) — a stable segmented radix sort of the
// fp64 values with the ids as payload keeps ascending ids among equal values,
// which is top_ids' std::stable_sort order — then a per-position overlap count.
// Used by the C++ drop-in (dsdv_norm_match_rows -> dsdv_window_stats_nm).
#include <cuda_runtime.h>

#include <cub/device/device_segmented_radix_sort.cuh>

#include "common.cuh"

namespace dsdv {

namespace {

__global__ void iota_rows(int32_t *ids, int nrows, int V, int stride) {
  const size_t n = (size_t)nrows * stride;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    ids[i] = (int32_t)(i % (size_t)stride);
}

__global__ void row_offsets(int *begin, int *end, int nrows, int V, int stride) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < nrows) {
    begin[r] = r * stride;
    end[r] = r * stride + V;
  }
}

// One CTA per position: the ids of the target row's top M are marked in a
// position-private byte map, then the draft row's top M ids are counted
// against it (each id appears once per list, so this is |T cap D|).
__global__ void overlap_kernel(const int32_t *sorted_ids, int gamma, int stride, int M,
                               uint8_t *marks, int V, double *nm_out) {
  const int j = blockIdx.x;
  const int32_t *td = sorted_ids + (size_t)j * stride;            // draft row j
  const int32_t *tt = sorted_ids + (size_t)(gamma + j) * stride;  // target row j
  uint8_t *mk = marks + (size_t)j * V;
  for (int i = threadIdx.x; i < V; i += blockDim.x) mk[i] = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < M; i += blockDim.x) mk[tt[i]] = 1;
  __syncthreads();
  int c = 0;
  for (int i = threadIdx.x; i < M; i += blockDim.x) c += mk[td[i]];
  __shared__ int red[32];
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int s = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
    nm_out[j] = (double)s / (double)M;  // verifier.cpp:133
  }
}

}  // namespace

// rows: gamma draft rows then gamma target rows (fp64, [.][stride]); scratch is
// caller-owned device memory of norm_match_scratch_bytes().
size_t norm_match_scratch_bytes(int gamma, int V, int stride) {
  const size_t n = (size_t)2 * gamma * stride;
  size_t temp = 0;
  cub::DeviceSegmentedRadixSort::SortPairsDescending(
      nullptr, temp, (const double *)nullptr, (double *)nullptr, (const int32_t *)nullptr,
      (int32_t *)nullptr, (int)n, 2 * gamma, (const int *)nullptr, (const int *)nullptr);
  auto up = [](size_t b) { return (b + 255) & ~size_t(255); };
  return 2 * up(n * sizeof(double)) + 2 * up(n * sizeof(int32_t)) +
         2 * up(2 * gamma * sizeof(int)) + up((size_t)gamma * V) + up(temp);
}

cudaError_t launch_norm_match(const double *draft, const double *target, int gamma, int V,
                              int stride, int M, void *scratch, double *nm_out,
                              cudaStream_t stream) {
  const int nrows = 2 * gamma;
  const size_t n = (size_t)nrows * stride;
  auto up = [](size_t b) { return (b + 255) & ~size_t(255); };
  char *p = static_cast<char *>(scratch);
  double *keys = reinterpret_cast<double *>(p);
  p += up(n * sizeof(double));
  double *keys_out = reinterpret_cast<double *>(p);
  p += up(n * sizeof(double));
  int32_t *ids_in = reinterpret_cast<int32_t *>(p);
  p += up(n * sizeof(int32_t));
  int32_t *ids_out = reinterpret_cast<int32_t *>(p);
  p += up(n * sizeof(int32_t));
  int *begin = reinterpret_cast<int *>(p);
  p += up(nrows * sizeof(int));
  int *end = reinterpret_cast<int *>(p);
  p += up(nrows * sizeof(int));
  uint8_t *marks = reinterpret_cast<uint8_t *>(p);
  p += up((size_t)gamma * V);
  void *temp = p;
  size_t temp_bytes = 0;
  cudaError_t e = cub::DeviceSegmentedRadixSort::SortPairsDescending(
      nullptr, temp_bytes, keys, keys_out, ids_in, ids_out, (int)n, nrows, begin, end);
  if (e != cudaSuccess) return e;
  // draft rows then target rows, contiguous in the key buffer
  e = cudaMemcpyAsync(keys, draft, (size_t)gamma * stride * sizeof(double),
                      cudaMemcpyDeviceToDevice, stream);
  if (e != cudaSuccess) return e;
  e = cudaMemcpyAsync(keys + (size_t)gamma * stride, target, (size_t)gamma * stride * sizeof(double),
                      cudaMemcpyDeviceToDevice, stream);
  if (e != cudaSuccess) return e;
  iota_rows<<<148, 256, 0, stream>>>(ids_in, nrows, V, stride);
  row_offsets<<<(nrows + 127) / 128, 128, 0, stream>>>(begin, end, nrows, V, stride);
  e = cub::DeviceSegmentedRadixSort::SortPairsDescending(temp, temp_bytes, keys, keys_out, ids_in,
                                                          ids_out, (int)n, nrows, begin, end, 0,
                                                          64, stream);
  if (e != cudaSuccess) return e;
  overlap_kernel<<<gamma, 256, 0, stream>>>(ids_out, gamma, stride, M, marks, V, nm_out);
  return cudaGetLastError();
}

}  // namespace dsdv
