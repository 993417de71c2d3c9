// K4: packed <-> padded bookkeeping of heterogeneous batches on the GPU.
//
//   k_packed_to_padded   packed_to_padded (batching.hpp:48-59): padded[b, j] = packed[first_b + j] for
//                        j < num_b, else the pad row
//   k_padded_to_packed   padded_to_packed (batching.hpp:61-75): packed[first_b + j] = padded[b, j]
//   k_item_to_element    PackedView::item_to_element (batching.hpp:20-27): owning batch element per packed row
//
// Rows are opaque `row_bytes`-byte records (a face, a vertex, a [3,3] face_verts block, ...). Each thread moves
// one 8-byte word (4-byte or 1-byte when the row size does not allow wider words), so consecutive threads touch
// consecutive addresses of a row and of consecutive rows: fully coalesced in both directions.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>

#include "raster_kernels.cuh"

namespace drb {

template <typename W>
__global__ void k_packed_to_padded(const W* __restrict__ packed, const int64_t* __restrict__ first,
                                   const int64_t* __restrict__ num, int64_t N, int64_t max_count, int64_t row_words,
                                   PadRow pad, W* __restrict__ padded) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t total = N * max_count * row_words;
  if (t >= total) return;
  const int64_t w = t % row_words;
  const int64_t row = t / row_words;
  const int64_t b = row / max_count, j = row % max_count;
  W v;
  if (j < num[b]) {
    v = packed[(first[b] + j) * row_words + w];
  } else {
    memcpy(&v, pad.bytes + w * sizeof(W), sizeof(W));
  }
  padded[t] = v;
}

template <typename W>
__global__ void k_padded_to_packed(const W* __restrict__ padded, const int64_t* __restrict__ first,
                                   const int64_t* __restrict__ num, int64_t N, int64_t max_count, int64_t row_words,
                                   W* __restrict__ packed) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t total = N * max_count * row_words;
  if (t >= total) return;
  const int64_t w = t % row_words;
  const int64_t row = t / row_words;
  const int64_t b = row / max_count, j = row % max_count;
  if (j < num[b]) packed[(first[b] + j) * row_words + w] = padded[t];
}

__global__ void k_item_to_element(const int64_t* __restrict__ first, const int64_t* __restrict__ num, int64_t N,
                                  int64_t total, int32_t* __restrict__ out) {
  // one block per batch element, threads stride over its rows (rows owned by no element stay -1)
  const int64_t b = blockIdx.x;
  if (b >= N) return;
  const int64_t f0 = first[b], n = num[b];
  for (int64_t j = threadIdx.x; j < n; j += blockDim.x)
    if (f0 + j >= 0 && f0 + j < total) out[f0 + j] = (int32_t)b;
}

template <typename W>
static cudaError_t p2p(const void* packed, const int64_t* first, const int64_t* num, int64_t N, int64_t max_count,
                       int64_t row_bytes, const PadRow& pad, void* padded, cudaStream_t st) {
  const int64_t rw = row_bytes / (int64_t)sizeof(W);
  const int64_t total = N * max_count * rw;
  if (total == 0) return cudaSuccess;
  k_packed_to_padded<W><<<(unsigned)((total + 255) / 256), 256, 0, st>>>(
      static_cast<const W*>(packed), first, num, N, max_count, rw, pad, static_cast<W*>(padded));
  return cudaGetLastError();
}

template <typename W>
static cudaError_t pd2p(const void* padded, const int64_t* first, const int64_t* num, int64_t N, int64_t max_count,
                        int64_t row_bytes, void* packed, cudaStream_t st) {
  const int64_t rw = row_bytes / (int64_t)sizeof(W);
  const int64_t total = N * max_count * rw;
  if (total == 0) return cudaSuccess;
  k_padded_to_packed<W><<<(unsigned)((total + 255) / 256), 256, 0, st>>>(
      static_cast<const W*>(padded), first, num, N, max_count, rw, static_cast<W*>(packed));
  return cudaGetLastError();
}

static int word_size(int64_t row_bytes, const void* a, const void* b) {
  const uintptr_t m = (uintptr_t)a | (uintptr_t)b;
  if (row_bytes % 8 == 0 && m % 8 == 0) return 8;
  if (row_bytes % 4 == 0 && m % 4 == 0) return 4;
  return 1;
}

cudaError_t launch_packed_to_padded(const void* packed, const int64_t* first, const int64_t* num, int64_t N,
                                    int64_t max_count, int64_t row_bytes, const PadRow& pad, void* padded,
                                    cudaStream_t st) {
  switch (word_size(row_bytes, packed, padded)) {
    case 8: return p2p<uint64_t>(packed, first, num, N, max_count, row_bytes, pad, padded, st);
    case 4: return p2p<uint32_t>(packed, first, num, N, max_count, row_bytes, pad, padded, st);
    default: return p2p<uint8_t>(packed, first, num, N, max_count, row_bytes, pad, padded, st);
  }
}

cudaError_t launch_padded_to_packed(const void* padded, const int64_t* first, const int64_t* num, int64_t N,
                                    int64_t max_count, int64_t row_bytes, void* packed, cudaStream_t st) {
  switch (word_size(row_bytes, packed, padded)) {
    case 8: return pd2p<uint64_t>(padded, first, num, N, max_count, row_bytes, packed, st);
    case 4: return pd2p<uint32_t>(padded, first, num, N, max_count, row_bytes, packed, st);
    default: return pd2p<uint8_t>(padded, first, num, N, max_count, row_bytes, packed, st);
  }
}

cudaError_t launch_item_to_element(const int64_t* first, const int64_t* num, int64_t N, int64_t total, int32_t* out,
                                   cudaStream_t st) {
  if (total > 0) {
    cudaError_t e = cudaMemsetAsync(out, 0xff, sizeof(int32_t) * (size_t)total, st);  // -1
    if (e != cudaSuccess) return e;
  }
  if (N > 0) k_item_to_element<<<(unsigned)N, 256, 0, st>>>(first, num, N, total, out);
  return cudaGetLastError();
}


}  // namespace drb
