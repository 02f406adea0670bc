// K10: fp32 grouped GEMM for fp32 layers (BASELINE config C1: tiny fp32 layer,
// rel-err 1e-5).  Same work lists (GemmTile) and epilogues as the tcgen05
// kernel (gemm_tc.cu) but true-fp32 FFMA on the SIMT pipes: plain TF32 tensor
// cores would miss the 1e-5 bar.  Replaces accumulate_block
// (/root/reference/proj/include/dsmoe/moe.hpp:213-231) for T = float.
#include "kernels.h"

namespace dsb {

enum { kSimtSwiGLU = 1, kSimtScale = 2 };

template <int MODE>
__global__ void __launch_bounds__(256) gemm_simt_kernel(const SimtArgs a) {
  __shared__ float As[32][kTileM + 4];  // [k][row]
  __shared__ float Bs[32][64 + 4];      // [k][col]
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int ntiles = *a.num_tiles;
  for (int ti = blockIdx.x; ti < ntiles; ti += gridDim.x) {
    const GemmTile tl = a.tiles[ti];
    const bool alt = (tl.m_live & kTileAltA) != 0;
    const float* Ab = alt ? a.A2 : a.A;
    const long long arows = alt ? a.a2_rows : a.a_rows;
    const int K = tl.nkb * kTileK;
    const int nc = tl.n_mma >> 1;
    const int nsub = MODE == kSimtSwiGLU ? nc / 32 : (tl.n_mma + 63) / 64;
    const int live = tl.m_live & 0xFFFFF;
    for (int sb = 0; sb < nsub; ++sb) {
      float acc[8][4];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
      for (int k0 = 0; k0 < K; k0 += 32) {
        for (int i = tid; i < kTileM * 32; i += 256) {
          const int r = i >> 5, c = i & 31;
          const long long row = static_cast<long long>(tl.a_row) + r;
          As[c][r] = row < arows ? Ab[row * a.lda + k0 + c] : 0.f;
        }
        for (int i = tid; i < 64 * 32; i += 256) {
          const int j = i >> 5, c = i & 31;
          int brow;
          bool ok = true;
          if (MODE == kSimtSwiGLU) {
            brow = sb * 64 + j;  // group sb: [32 W1 rows | 32 W3 rows] (w13_row_of)
          } else {
            brow = sb * 64 + j;
            ok = brow < tl.n_mma;
          }
          Bs[c][j] = ok ? a.B[(static_cast<long long>(tl.b_row) + brow) * a.ldb + k0 + c] : 0.f;
        }
        __syncthreads();
#pragma unroll 8
        for (int k = 0; k < 32; ++k) {
          float av[8], bv[4];
#pragma unroll
          for (int i = 0; i < 8; ++i) av[i] = As[k][ty * 8 + i];
#pragma unroll
          for (int j = 0; j < 4; ++j) bv[j] = Bs[k][tx + 16 * j];
#pragma unroll
          for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
        }
        __syncthreads();
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int r = ty * 8 + i;
        if (r >= tl.m_valid) continue;
        const long long orow = static_cast<long long>(tl.out_row) + r;
        float* o = a.out + orow * a.ldo + tl.out_col;
        if (MODE == kSimtSwiGLU) {
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const float g = acc[i][j], u = acc[i][j + 2];
            o[sb * 32 + tx + 16 * j] = r < live ? (g / (1.0f + expf(-g))) * u : 0.f;
          }
        } else {
          const float sc = a.row_scale[orow];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int col = sb * 64 + tx + 16 * j;
            if (col < tl.n_mma) o[col] = acc[i][j] * sc;
          }
        }
      }
    }
  }
}

int launch_gemm_simt(int mode, const SimtArgs& a, int max_tiles, int num_sms, cudaStream_t stream) {
  const int grid = max_tiles < num_sms * 4 ? (max_tiles > 0 ? max_tiles : 1) : num_sms * 4;
  if (mode == kSimtSwiGLU)
    gemm_simt_kernel<kSimtSwiGLU><<<grid, 256, 0, stream>>>(a);
  else
    gemm_simt_kernel<kSimtScale><<<grid, 256, 0, stream>>>(a);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

}  // namespace dsb
