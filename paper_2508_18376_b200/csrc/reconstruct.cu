// K7 / K8: offline expert partition by neuron importance (north-star item 1).
//
// profile_importance (/root/reference/proj/include/dsmoe/reconstruct.hpp:99-149):
//   for each calibration token t (ascending) and selection j, for each neuron n
//   of the selected expert: g = sum_k x[t][k] * W1[k][n] in float (serial k,
//   one rounding per multiply and per add), likewise u with W3; sg =
//   double(swish(g)) with glibc expf and IEEE division; v = sg | |sg| | sg*u |
//   |sg*u|; acc[e][n] += v in double, in (t, j) order.
// build_reconstruction_map (:151-168): per expert std::stable_sort of the
//   neuron ids by importance descending (ties keep the lower id first).
// reconstruct_experts (:196-230): permute W1/W3 columns and W2 rows by the
//   order, split at ceil(d_ffn/2) into major (block 2e) and minor (2e+1).
//
// Device plan: the calibration routing is imported and permuted exactly like
// the forward (rows of expert e in ascending (t, j) order), so
//   importance_tile_kernel   one 64-row x 64-neuron tile of v per block,
//   importance_reduce_kernel one thread per (e, n) summing v down its rows
//                            in segment order = the reference's (t, j) order,
//   order_sort_kernel        one block per expert: bitonic sort of
//                            (value desc, id asc), a total order whose unique
//                            result is the stable sort's,
//   gather_w13 / gather_w2t  repack the P=1 layout into the P=2 one.
// Compiled with -fmad=false (see build.py).
#include "kernels.h"

namespace dsb {

struct ImpUnit {  // packed-layout facts of one P=1 unit (host computed)
  long long base0, base1;  // W13 row bases of the two virtual sub-blocks
  int h0, wpad0, wpad1;
};

__device__ __forceinline__ long long imp_w13_row(const ImpUnit& u, int n, int which) {
  const bool second = n >= u.h0;
  const int i = second ? n - u.h0 : n;
  const int wpad = second ? u.wpad1 : u.wpad0;
  const long long base = second ? u.base1 : u.base0;
  (void)wpad;
  return w13_row_of(base, i, which);
}

template <typename T>
__global__ void __launch_bounds__(256) importance_tile_kernel(const T* __restrict__ x, const int32_t* __restrict__ row_token,
                                                              int seg_start, int nrows, const T* __restrict__ w13, ImpUnit u,
                                                              int d, int ffn, int metric, double* __restrict__ v) {
  __shared__ float xs[64][33];
  __shared__ float gs[32][65];
  __shared__ float us[32][65];
  const int r0 = blockIdx.x * 64, n0 = blockIdx.y * 64;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const bool need_u = metric >= 2;
  float g[4][4], uu[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) g[i][j] = uu[i][j] = 0.0f;
  for (int k0 = 0; k0 < d; k0 += 32) {
    for (int i = threadIdx.x; i < 64 * 32; i += 256) {
      const int r = i >> 5, c = i & 31;
      float val = 0.0f;
      if (r0 + r < nrows) {
        const long long t = row_token[seg_start + r0 + r];
        val = static_cast<float>(x[t * d + k0 + c]);
      }
      xs[r][c] = val;
    }
    for (int i = threadIdx.x; i < 64 * 32; i += 256) {
      const int nn = i >> 5, c = i & 31;
      float a = 0.0f, b = 0.0f;
      if (n0 + nn < ffn) {
        a = static_cast<float>(w13[imp_w13_row(u, n0 + nn, 0) * d + k0 + c]);
        if (need_u) b = static_cast<float>(w13[imp_w13_row(u, n0 + nn, 1) * d + k0 + c]);
      }
      gs[c][nn] = a;
      us[c][nn] = b;
    }
    __syncthreads();
    for (int k = 0; k < 32; ++k) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float xv = xs[ty + 16 * i][k];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          g[i][j] = __fadd_rn(g[i][j], __fmul_rn(xv, gs[k][tx + 16 * j]));
          if (need_u) uu[i][j] = __fadd_rn(uu[i][j], __fmul_rn(xv, us[k][tx + 16 * j]));
        }
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int r = r0 + ty + 16 * i, n = n0 + tx + 16 * j;
      if (r >= nrows || n >= ffn) continue;
      const float gv = g[i][j];
      const float sw = __fdiv_rn(gv, __fadd_rn(1.0f, glibc_expf(-gv)));  // swish, matrix.hpp:91
      const double sg = static_cast<double>(sw);
      double val;
      switch (metric) {
        case 0: val = sg; break;
        case 1: val = fabs(sg); break;
        case 2: val = __dmul_rn(sg, static_cast<double>(uu[i][j])); break;
        default: val = fabs(__dmul_rn(sg, static_cast<double>(uu[i][j]))); break;
      }
      v[static_cast<long long>(seg_start + r) * ffn + n] = val;
    }
}

__global__ void importance_reduce_kernel(const double* __restrict__ v, const UnitSeg* __restrict__ seg, int ffn,
                                         double* __restrict__ values) {
  const int e = blockIdx.x;
  const int n = blockIdx.y * blockDim.x + threadIdx.x;
  if (n >= ffn) return;
  const UnitSeg s = seg[e];
  double acc = 0.0;
  for (int r = 0; r < s.n_tot; ++r) acc = __dadd_rn(acc, v[static_cast<long long>(s.start + r) * ffn + n]);
  values[static_cast<long long>(e) * ffn + n] = acc;
}

// one block per expert; n_pow2 >= ffn, power of two; smem: n_pow2 x (double + int)
__global__ void order_sort_kernel(const double* __restrict__ values, int ffn, int n_pow2, int32_t* __restrict__ order) {
  extern __shared__ unsigned char sm_raw[];
  double* key = reinterpret_cast<double*>(sm_raw);
  int* id = reinterpret_cast<int*>(key + n_pow2);
  const int e = blockIdx.x;
  for (int i = threadIdx.x; i < n_pow2; i += blockDim.x) {
    key[i] = i < ffn ? values[static_cast<long long>(e) * ffn + i] : 0.0;
    id[i] = i < ffn ? i : ffn + i;  // padding ids sort after every real id
  }
  __syncthreads();
  // "a before b"  <=>  a is real and (b is padding or key_a > key_b or (key_a == key_b and id_a < id_b))
  auto before = [&](int a, int b) {
    const bool pa = id[a] >= ffn, pb = id[b] >= ffn;
    if (pa != pb) return pb;
    if (pa) return id[a] < id[b];
    if (key[a] > key[b]) return true;
    if (key[b] > key[a]) return false;
    return id[a] < id[b];
  };
  for (int size = 2; size <= n_pow2; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < n_pow2; i += blockDim.x) {
        const int j = i ^ stride;
        if (j > i) {
          const bool asc = (i & size) == 0;  // ascending in "before" order
          const bool sw = asc ? before(j, i) : before(i, j);
          if (sw) {
            const double tk = key[i];
            key[i] = key[j];
            key[j] = tk;
            const int ti = id[i];
            id[i] = id[j];
            id[j] = ti;
          }
        }
      }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < ffn; i += blockDim.x) order[static_cast<long long>(e) * ffn + i] = id[i];
}

// new W13 row (unit e, new neuron n', which) <- old row of neuron order[n'];
// the P=2 reconstructed layout has the same sub-block geometry as the P=1
// virtual split (ceil(ffn/2) | rest), so one ImpUnit describes both.
template <typename T>
__global__ void gather_w13_kernel(const T* __restrict__ src, T* __restrict__ dst, const int32_t* __restrict__ order,
                                  ImpUnit u, int ffn, int d) {
  const int n = blockIdx.x;
  const int which = blockIdx.y;
  const long long so = imp_w13_row(u, order[n], which) * d, dof = imp_w13_row(u, n, which) * d;
  for (int k = threadIdx.x; k < d; k += blockDim.x) dst[dof + k] = src[so + k];
}

template <typename T>
__global__ void gather_w2t_kernel(const T* __restrict__ src, T* __restrict__ dst, const int32_t* __restrict__ order,
                                  ImpUnit u, int ffn, long long row0, long long hstride) {
  const long long j = row0 + blockIdx.x;
  for (int n = threadIdx.x; n < ffn; n += blockDim.x) {
    const int o = order[n];
    const int hs = o < u.h0 ? o : u.wpad0 + (o - u.h0);
    const int hd = n < u.h0 ? n : u.wpad0 + (n - u.h0);
    dst[j * hstride + hd] = src[j * hstride + hs];
  }
}

// ---------------------------------------------------------------- launchers
int launch_importance_tiles(int bf16, const void* x, const int32_t* row_token, int seg_start, int nrows,
                            const void* w13, const ImpUnitC& uc, int d, int ffn, int metric, double* v,
                            cudaStream_t s) {
  if (nrows <= 0) return 0;
  ImpUnit u{uc.base0, uc.base1, uc.h0, uc.wpad0, uc.wpad1};
  dim3 grid((nrows + 63) / 64, (ffn + 63) / 64);
  if (bf16)
    importance_tile_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(x), row_token, seg_start,
                                                               nrows, static_cast<const __nv_bfloat16*>(w13), u, d, ffn,
                                                               metric, v);
  else
    importance_tile_kernel<float><<<grid, 256, 0, s>>>(static_cast<const float*>(x), row_token, seg_start, nrows,
                                                       static_cast<const float*>(w13), u, d, ffn, metric, v);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

int launch_importance_reduce(const double* v, const UnitSeg* seg, int E, int ffn, double* values, cudaStream_t s) {
  dim3 grid(E, (ffn + 255) / 256);
  importance_reduce_kernel<<<grid, 256, 0, s>>>(v, seg, ffn, values);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

int launch_order_sort(const double* values, int E, int ffn, int32_t* order, cudaStream_t s) {
  int n = 1;
  while (n < ffn) n <<= 1;
  const size_t smem = static_cast<size_t>(n) * (sizeof(double) + sizeof(int));
  if (smem > 200 * 1024) return -1;
  if (set_max_dyn_smem(order_sort_kernel, smem) != cudaSuccess) return -2;
  order_sort_kernel<<<E, 1024, smem, s>>>(values, ffn, n, order);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

int launch_gather_unit(int bf16, const void* w13_src, void* w13_dst, const void* w2t_src, void* w2t_dst,
                       const int32_t* order, const ImpUnitC& uc, int ffn, int d, long long w2t_row0,
                       long long hstride, cudaStream_t s) {
  ImpUnit u{uc.base0, uc.base1, uc.h0, uc.wpad0, uc.wpad1};
  dim3 g1(ffn, 2);
  if (bf16) {
    gather_w13_kernel<__nv_bfloat16><<<g1, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(w13_src),
                                                        static_cast<__nv_bfloat16*>(w13_dst), order, u, ffn, d);
    gather_w2t_kernel<__nv_bfloat16><<<d, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(w2t_src),
                                                       static_cast<__nv_bfloat16*>(w2t_dst), order, u, ffn, w2t_row0, hstride);
  } else {
    gather_w13_kernel<float><<<g1, 256, 0, s>>>(static_cast<const float*>(w13_src), static_cast<float*>(w13_dst), order,
                                                u, ffn, d);
    gather_w2t_kernel<float><<<d, 256, 0, s>>>(static_cast<const float*>(w2t_src), static_cast<float*>(w2t_dst), order,
                                               u, ffn, w2t_row0, hstride);
  }
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

}  // namespace dsb
