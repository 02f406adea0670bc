// K8: weight packing into the device layout of the grouped GEMMs.
//
// Host layout (reference, moe.hpp:39-45): per physical block w1, w3 are
// d_model x width and w2 is width x d_model, row-major.  Device layout, per
// expert unit (an original expert whose P blocks are its sub-blocks):
//   W13  K-major rows of d_model elements: for each sub-block, for each chunk
//        of <= 128 neurons, the chunk's W1 columns then its W3 columns, so one
//        GEMM1 N-tile holds [g | u] for the same neurons (SwiGLU epilogue);
//   W2T  d_model rows of hstride elements (W2 transposed, sub-blocks
//        concatenated along K) so GEMM2 can stop after the major sub-block.
// Widths are zero-padded to multiples of 64 (a zero neuron contributes
// swish(0) * 0 * W2 = 0 exactly).  The same transposing copy also realises
// permute_expert + slice_expert (reconstruct.hpp:173-187, transform.hpp:43-57)
// when given a neuron order (reconstruct_on_device, below).
#include <map>
#include <mutex>
#include <utility>

#include "common.cuh"

namespace dsb {

cudaError_t set_max_dyn_smem(const void* func, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> done;  // (function, device) -> bytes set
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  size_t& cur = done[{func, dev}];
  if (bytes <= cur) return cudaSuccess;
  e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
  if (e == cudaSuccess) cur = bytes;
  return e;
}

template <typename T>
__device__ __forceinline__ float to_f(T v) { return static_cast<float>(v); }
template <typename T>
__device__ __forceinline__ T from_f(float v) { return static_cast<T>(v); }

// dst row of neuron n inside a sub-block packed at `base` with padded width wpad
__device__ __forceinline__ long long w13_row(long long base, int wpad, int n, int which) {
  (void)wpad;
  return w13_row_of(base, n, which);
}

// W13 pack.  src w1/w3: d x ld row-major; neurons are columns order[col0 + n]
// (order == nullptr -> identity) for n < ncols.  grid (ceil(ncols/32), ceil(d/32), 2)
template <typename TS, typename TD>
__global__ void pack_w13_kernel(const TS* __restrict__ w1, const TS* __restrict__ w3, int d, int ld,
                                const int* __restrict__ order, int col0, int ncols, TD* __restrict__ dst,
                                long long base, int wpad) {
  __shared__ float tile[32][33];
  const TS* src = blockIdx.z ? w3 : w1;
  const int n0 = blockIdx.x * 32, k0 = blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int k = k0 + i, n = n0 + threadIdx.x;
    float v = 0.f;
    if (k < d && n < ncols) {
      const int col = order ? order[col0 + n] : col0 + n;
      v = to_f(src[static_cast<long long>(k) * ld + col]);
    }
    tile[i][threadIdx.x] = v;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int n = n0 + i, k = k0 + threadIdx.x;
    if (n < ncols && k < d) dst[w13_row(base, wpad, n, blockIdx.z) * d + k] = from_f<TD>(tile[threadIdx.x][i]);
  }
}

// W2T pack.  src w2: rows x d row-major; neuron n is row order[row0 + n].
// dst[(drow + j) * hstride + hcol0 + n] = src[row(n)][j].  grid (ceil(d/32), ceil(nrows/32))
template <typename TS, typename TD>
__global__ void pack_w2t_kernel(const TS* __restrict__ w2, int d, const int* __restrict__ order, int row0,
                                int nrows, TD* __restrict__ dst, long long drow, int hcol0,
                                long long hstride) {
  __shared__ float tile[32][33];
  const int j0 = blockIdx.x * 32, n0 = blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int n = n0 + i, j = j0 + threadIdx.x;
    float v = 0.f;
    if (n < nrows && j < d) {
      const int row = order ? order[row0 + n] : row0 + n;
      v = to_f(w2[static_cast<long long>(row) * d + j]);
    }
    tile[i][threadIdx.x] = v;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int j = j0 + i, n = n0 + threadIdx.x;
    if (j < d && n < nrows) dst[(drow + j) * hstride + hcol0 + n] = from_f<TD>(tile[threadIdx.x][i]);
  }
}

// gate (d x E) -> gateT (Epad x d, bf16 or fp32) and the exact-mode copy
// gate_exact (d x E fp32 of the layer-dtype-rounded values).
template <typename TS, typename TD>
__global__ void pack_gate_kernel(const TS* __restrict__ gate, int d, int E, TD* __restrict__ gateT,
                                 float* __restrict__ gate_exact) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= static_cast<long long>(d) * E) return;
  const int k = static_cast<int>(i / E), e = static_cast<int>(i - static_cast<long long>(k) * E);
  const TD v = from_f<TD>(to_f(gate[i]));
  gateT[static_cast<long long>(e) * d + k] = v;
  gate_exact[i] = to_f(v);
}

template <typename TS, typename TD>
static int pack_w13_t(const void* w1, const void* w3, int d, int ld, const int* order, int col0,
                      int ncols, void* dst, long long base, int wpad, cudaStream_t s) {
  dim3 grid((ncols + 31) / 32, (d + 31) / 32, 2), block(32, 8);
  pack_w13_kernel<TS, TD><<<grid, block, 0, s>>>(static_cast<const TS*>(w1), static_cast<const TS*>(w3), d,
                                                 ld, order, col0, ncols, static_cast<TD*>(dst), base, wpad);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}
template <typename TS, typename TD>
static int pack_w2t_t(const void* w2, int d, const int* order, int row0, int nrows, void* dst,
                      long long drow, int hcol0, long long hstride, cudaStream_t s) {
  dim3 grid((d + 31) / 32, (nrows + 31) / 32), block(32, 8);
  pack_w2t_kernel<TS, TD><<<grid, block, 0, s>>>(static_cast<const TS*>(w2), d, order, row0, nrows,
                                                 static_cast<TD*>(dst), drow, hcol0, hstride);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}
template <typename TS, typename TD>
static int pack_gate_t(const void* gate, int d, int E, void* gateT, float* gate_exact, cudaStream_t s) {
  const long long n = static_cast<long long>(d) * E;
  pack_gate_kernel<TS, TD><<<static_cast<int>((n + 255) / 256), 256, 0, s>>>(
      static_cast<const TS*>(gate), d, E, static_cast<TD*>(gateT), gate_exact);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

// dtype codes: 0 fp32, 1 bf16
int launch_pack_w13(int src_dt, int dst_dt, const void* w1, const void* w3, int d, int ld, const int* order,
                    int col0, int ncols, void* dst, long long base, int wpad, cudaStream_t s) {
  if (src_dt == 0 && dst_dt == 0) return pack_w13_t<float, float>(w1, w3, d, ld, order, col0, ncols, dst, base, wpad, s);
  if (src_dt == 0 && dst_dt == 1) return pack_w13_t<float, __nv_bfloat16>(w1, w3, d, ld, order, col0, ncols, dst, base, wpad, s);
  if (src_dt == 1 && dst_dt == 1) return pack_w13_t<__nv_bfloat16, __nv_bfloat16>(w1, w3, d, ld, order, col0, ncols, dst, base, wpad, s);
  if (src_dt == 1 && dst_dt == 0) return pack_w13_t<__nv_bfloat16, float>(w1, w3, d, ld, order, col0, ncols, dst, base, wpad, s);
  return -1;
}
int launch_pack_w2t(int src_dt, int dst_dt, const void* w2, int d, const int* order, int row0, int nrows,
                    void* dst, long long drow, int hcol0, long long hstride, cudaStream_t s) {
  if (src_dt == 0 && dst_dt == 0) return pack_w2t_t<float, float>(w2, d, order, row0, nrows, dst, drow, hcol0, hstride, s);
  if (src_dt == 0 && dst_dt == 1) return pack_w2t_t<float, __nv_bfloat16>(w2, d, order, row0, nrows, dst, drow, hcol0, hstride, s);
  if (src_dt == 1 && dst_dt == 1) return pack_w2t_t<__nv_bfloat16, __nv_bfloat16>(w2, d, order, row0, nrows, dst, drow, hcol0, hstride, s);
  if (src_dt == 1 && dst_dt == 0) return pack_w2t_t<__nv_bfloat16, float>(w2, d, order, row0, nrows, dst, drow, hcol0, hstride, s);
  return -1;
}
int launch_pack_gate(int src_dt, int dst_dt, const void* gate, int d, int E, void* gateT, float* gate_exact,
                     cudaStream_t s) {
  if (src_dt == 0 && dst_dt == 0) return pack_gate_t<float, float>(gate, d, E, gateT, gate_exact, s);
  if (src_dt == 0 && dst_dt == 1) return pack_gate_t<float, __nv_bfloat16>(gate, d, E, gateT, gate_exact, s);
  if (src_dt == 1 && dst_dt == 1) return pack_gate_t<__nv_bfloat16, __nv_bfloat16>(gate, d, E, gateT, gate_exact, s);
  if (src_dt == 1 && dst_dt == 0) return pack_gate_t<__nv_bfloat16, float>(gate, d, E, gateT, gate_exact, s);
  return -1;
}

}  // namespace dsb
