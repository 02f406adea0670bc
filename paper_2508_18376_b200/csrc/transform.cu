// K8b: re-grouping of the packed weight layout on the device, and read-back
// into the reference layout.
//
// The packed layout (pack.cu, common.cuh) stores per expert unit a W13 block
// (one K-major row of d_model elements per neuron for W1 and for W3) and a
// W2T block (d_model rows; the unit's neurons are columns).  Every partition
// operation of the reference is a re-grouping of neurons between units:
//   complete_transform  (transform.hpp:66-95)   unit e*p+q <- neurons [q*c, (q+1)*c) of unit e, W2 x p
//   partial_transform   (transform.hpp:100-131) sub-block q of unit e <- the same neurons, unscaled
//   reverse_partial     (transform.hpp:136-170) unit e <- its sub-blocks concatenated
//   block view          (moe.hpp:239-271)       unit b = e*P+p <- sub-block p of unit e (each
//                                               physical block addressable alone, for arbitrary
//                                               RoutingDecisions)
// so two gather kernels serve them all: whole rows of W13 (and of the
// transposed gate) move by a row map, and W2T / the exact-mode gate move by a
// per-unit column map, scaled.  The host (capi.cpp) builds the maps.  A third
// kernel transposes packed rows back into the reference's row-major
// w1 / w3 (d x width), w2 (width x d) and gate (d x E).
#include <algorithm>

#include "kernels.h"

namespace dsb {

// dst row dst_row[i] = src row src_row[i] (or zeros when src_row[i] < 0);
// rows of `vec` 16-byte vectors.  One warp per row.
__global__ void __launch_bounds__(256) row_gather_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst,
                                                         const long long* __restrict__ dst_row,
                                                         const long long* __restrict__ src_row, long long n,
                                                         int vec) {
  const int lane = threadIdx.x & 31;
  const long long w0 = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const long long nw = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
  for (long long i = w0; i < n; i += nw) {
    const long long sr = src_row[i];
    uint4* d = dst + dst_row[i] * vec;
    if (sr < 0) {
      for (int v = lane; v < vec; v += 32) d[v] = make_uint4(0, 0, 0, 0);
    } else {
      const uint4* s = src + sr * vec;
      for (int v = lane; v < vec; v += 32) d[v] = __ldg(s + v);
    }
  }
}

int launch_row_gather(const void* src, void* dst, const long long* dst_row, const long long* src_row, long long n,
                      long long row_bytes, int num_sms, cudaStream_t s) {
  if (row_bytes % 16 != 0) return -1;
  if (n <= 0) return 0;
  const long long blocks = std::min<long long>((n + 7) / 8, static_cast<long long>(num_sms) * 16);
  row_gather_kernel<<<static_cast<int>(blocks), 256, 0, s>>>(static_cast<const uint4*>(src), static_cast<uint4*>(dst),
                                                             dst_row, src_row, n, static_cast<int>(row_bytes / 16));
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

// Column gather: for unit descriptor u (blockIdx.y), rows j in [0, rows):
// dst[(u.dst_row0 + j) * dst_ld + c] = src[(u.src_row0 + j) * src_ld + colmap[u.map_off + c]] * u.scale
// for c in [0, u.ncols) (zeros where the map holds -1).  The scale is applied
// in fp32 and rounded once into the element type — for fp32 layers exactly
// the reference's `w2 * T(p)` (transform.hpp:53).
template <typename TE>
__global__ void __launch_bounds__(256) col_gather_kernel(const TE* __restrict__ src, TE* __restrict__ dst,
                                                         const ColUnit* __restrict__ units, const int* __restrict__ colmap,
                                                         int rows, long long src_ld, long long dst_ld) {
  const ColUnit u = units[blockIdx.y];
  for (int j = blockIdx.x; j < rows; j += gridDim.x) {
    const TE* s = src + (u.src_row0 + j) * src_ld;
    TE* d = dst + (u.dst_row0 + j) * dst_ld;
    for (int c = threadIdx.x; c < u.ncols; c += blockDim.x) {
      const int m = colmap[u.map_off + c];
      float v = 0.0f;
      if (m >= 0) v = __fmul_rn(static_cast<float>(s[m]), u.scale);
      d[c] = static_cast<TE>(v);
    }
  }
}

int launch_col_gather(int bf16, const void* src, void* dst, const ColUnit* units, int nunits, const int* colmap,
                      int rows, long long src_ld, long long dst_ld, cudaStream_t s) {
  if (nunits <= 0 || rows <= 0) return 0;
  const dim3 grid(std::min(rows, 1024), nunits);
  if (bf16)
    col_gather_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(src),
                                                          static_cast<__nv_bfloat16*>(dst), units, colmap, rows,
                                                          src_ld, dst_ld);
  else
    col_gather_kernel<float><<<grid, 256, 0, s>>>(static_cast<const float*>(src), static_cast<float*>(dst), units,
                                                  colmap, rows, src_ld, dst_ld);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

// Transpose read-back: out[c * R + r] = src[row(r) * src_ld + col0 + c] for
// r < R, c < Ccount, row(r) = rows ? rows[r] : row0 + r.  32 x 32 tiles
// through shared memory: coalesced reads along the packed rows, coalesced
// writes along the reference's rows.
template <typename TE>
__global__ void __launch_bounds__(256) transpose_kernel(const TE* __restrict__ src, long long src_ld,
                                                        const long long* __restrict__ rows, long long row0,
                                                        long long col0, int R, int Ccount, TE* __restrict__ out) {
  __shared__ TE tile[32][33];
  const int r0 = blockIdx.x * 32, c0 = blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  for (int i = ty; i < 32; i += 8) {
    const int r = r0 + i, c = c0 + tx;
    if (r < R && c < Ccount) {
      const long long sr = rows ? rows[r] : row0 + r;
      tile[i][tx] = src[sr * src_ld + col0 + c];
    }
  }
  __syncthreads();
  for (int i = ty; i < 32; i += 8) {
    const int c = c0 + i, r = r0 + tx;
    if (r < R && c < Ccount) out[static_cast<long long>(c) * R + r] = tile[tx][i];
  }
}

int launch_transpose(int bf16, const void* src, long long src_ld, const long long* rows, long long row0,
                     long long col0, int R, int Ccount, void* out, cudaStream_t s) {
  if (R <= 0 || Ccount <= 0) return 0;
  const dim3 grid((R + 31) / 32, (Ccount + 31) / 32);
  if (grid.y > 65535) return -1;
  if (bf16)
    transpose_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(src), src_ld, rows, row0,
                                                         col0, R, Ccount, static_cast<__nv_bfloat16*>(out));
  else
    transpose_kernel<float><<<grid, 256, 0, s>>>(static_cast<const float*>(src), src_ld, rows, row0, col0, R, Ccount,
                                                 static_cast<float*>(out));
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

// Row comparison of two T x d outputs (report metrics of the reference C
// ABI: mean_relative_error, dropping.hpp:278-293, and the scaled residual of
// verify_equivalence, transform.hpp:190-198): per token t, out[5t + ...] =
// { sum (a-b)^2, sum b^2, max |a-b|, max |a|, max |b| } in double.  One warp
// per token.
template <typename TE>
__global__ void __launch_bounds__(256) compare_rows_kernel(const TE* __restrict__ a, const TE* __restrict__ b,
                                                           int T, int d, double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (t >= T) return;
  const TE* ra = a + static_cast<long long>(t) * d;
  const TE* rb = b + static_cast<long long>(t) * d;
  double s_d = 0.0, s_b = 0.0, m_d = 0.0, m_a = 0.0, m_b = 0.0;
  for (int j = lane; j < d; j += 32) {
    const double va = static_cast<double>(static_cast<float>(ra[j]));
    const double vb = static_cast<double>(static_cast<float>(rb[j]));
    const double df = va - vb;
    s_d += df * df;
    s_b += vb * vb;
    m_d = fmax(m_d, fabs(df));
    m_a = fmax(m_a, fabs(va));
    m_b = fmax(m_b, fabs(vb));
  }
  for (int o = 16; o > 0; o >>= 1) {
    s_d += __shfl_xor_sync(0xffffffffu, s_d, o);
    s_b += __shfl_xor_sync(0xffffffffu, s_b, o);
    m_d = fmax(m_d, __shfl_xor_sync(0xffffffffu, m_d, o));
    m_a = fmax(m_a, __shfl_xor_sync(0xffffffffu, m_a, o));
    m_b = fmax(m_b, __shfl_xor_sync(0xffffffffu, m_b, o));
  }
  if (lane == 0) {
    double* o5 = out + 5LL * t;
    o5[0] = s_d;
    o5[1] = s_b;
    o5[2] = m_d;
    o5[3] = m_a;
    o5[4] = m_b;
  }
}

int launch_compare_rows(int bf16, const void* a, const void* b, int T, int d, double* out, cudaStream_t s) {
  if (T <= 0) return 0;
  const int blocks = (T + 7) / 8;
  if (bf16)
    compare_rows_kernel<__nv_bfloat16><<<blocks, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(a),
                                                              static_cast<const __nv_bfloat16*>(b), T, d, out);
  else
    compare_rows_kernel<float><<<blocks, 256, 0, s>>>(static_cast<const float*>(a), static_cast<const float*>(b), T,
                                                      d, out);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

}  // namespace dsb
