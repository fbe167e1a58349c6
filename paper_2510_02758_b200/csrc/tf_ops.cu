// Small fused ops of the decode forward that sit between the library GEMMs:
// RMSNorm and the SwiGLU activation.  Both are HBM/latency-bound; torch's
// generic layer-norm and two-pass silu/mul kernels cost ~17% of a C2 decode
// step (profiles/r1_bench_window_launches.txt), so these replace them:
//
//   tf_rmsnorm     y[r] = x[r] * rsqrt(mean(x[r]^2) + eps) * w   (one CTA per row,
//                  16-B vector loads, fp32 sum, row held in registers)
//   tf_silu_mul    y = silu(gu[:, :F]) * gu[:, F:]                (one pass, 16-B vectors)
//   tf_residual_rmsnorm  x += y; h = rmsnorm(x) * w                (residual add taken out of
//                  the output-projection GEMM's epilogue, fused with the next norm)
#include <algorithm>

#include "tf_common.cuh"

namespace tf {

__device__ __forceinline__ void unpack8(const uint4& u, float* f) {
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    f[2 * i] = __uint_as_float(w[i] << 16);
    f[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
  }
}

__device__ __forceinline__ uint4 pack8(const float* f) {
  uint32_t w[4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
    w[i] = (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(f[2 * i])) |
           ((uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(f[2 * i + 1])) << 16);
  return make_uint4(w[0], w[1], w[2], w[3]);
}

constexpr int kNormThreads = 256;
constexpr int kNormMaxVec = 4;  // 16-B vectors per thread held in registers: D <= 256*4*8 = 8192

__global__ void __launch_bounds__(kNormThreads) rmsnorm_kernel(const uint16_t* __restrict__ x,
                                                             const uint16_t* __restrict__ w,
                                                             uint16_t* __restrict__ y, int D, float eps) {
  const int64_t row = blockIdx.x;
  const uint4* xr = reinterpret_cast<const uint4*>(x + row * D);
  const uint4* wr = reinterpret_cast<const uint4*>(w);
  uint4* yr = reinterpret_cast<uint4*>(y + row * D);
  const int nv = D / 8;
  float v[kNormMaxVec][8];
  uint4 gw[kNormMaxVec];
  float ss = 0.f;
  // the weight loads are issued with the row's (independent of the reduction)
  // so their latency overlaps instead of following it
#pragma unroll
  for (int k = 0; k < kNormMaxVec; ++k) {
    const int i = threadIdx.x + k * kNormThreads;
    if (i < nv) gw[k] = __ldg(wr + i);
  }
#pragma unroll
  for (int k = 0; k < kNormMaxVec; ++k) {
    const int i = threadIdx.x + k * kNormThreads;
    if (i < nv) {
      unpack8(xr[i], v[k]);
#pragma unroll
      for (int e = 0; e < 8; ++e) ss += v[k][e] * v[k][e];
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  __shared__ float part[kNormThreads / 32];
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = ss;
  __syncthreads();
  float tot = 0.f;
#pragma unroll
  for (int i = 0; i < kNormThreads / 32; ++i) tot += part[i];
  const float r = rsqrtf(tot / (float)D + eps);
#pragma unroll
  for (int k = 0; k < kNormMaxVec; ++k) {
    const int i = threadIdx.x + k * kNormThreads;
    if (i < nv) {
      float g[8], o[8];
      unpack8(gw[k], g);
#pragma unroll
      for (int e = 0; e < 8; ++e) o[e] = __bfloat162float(__float2bfloat16_rn(v[k][e] * r)) * g[e];
      yr[i] = pack8(o);
    }
  }
}

// x[r] <- bf16(x[r] + y[r]); h[r] <- rmsnorm(x[r]) * w  (one CTA per row).  The
// decode step's output projections (o_proj, down_proj) run as plain GEMMs
// into y - 2 us faster per call than cuBLAS addmm with the residual in its
// epilogue at the C2 shapes (profiles/r2_gemm_probe.json) - and this kernel
// takes over the residual add from the epilogue together with the next
// sub-layer's RMSNorm (same arithmetic as rmsnorm_kernel on the new x).
__global__ void __launch_bounds__(kNormThreads) residual_rmsnorm_kernel(uint16_t* __restrict__ x,
                                                                        const uint16_t* __restrict__ y,
                                                                        const uint16_t* __restrict__ w,
                                                                        uint16_t* __restrict__ h, int D, float eps) {
  const int64_t row = blockIdx.x;
  uint4* xr = reinterpret_cast<uint4*>(x + row * D);
  const uint4* yr = reinterpret_cast<const uint4*>(y + row * D);
  const uint4* wr = reinterpret_cast<const uint4*>(w);
  uint4* hr = reinterpret_cast<uint4*>(h + row * D);
  const int nv = D / 8;
  float v[kNormMaxVec][8];
  uint4 gw[kNormMaxVec];
  float ss = 0.f;
#pragma unroll
  for (int k = 0; k < kNormMaxVec; ++k) {
    const int i = threadIdx.x + k * kNormThreads;
    if (i < nv) gw[k] = __ldg(wr + i);
  }
#pragma unroll
  for (int k = 0; k < kNormMaxVec; ++k) {
    const int i = threadIdx.x + k * kNormThreads;
    if (i < nv) {
      float a[8], b[8];
      unpack8(yr[i], a);
      unpack8(xr[i], b);
#pragma unroll
      for (int e = 0; e < 8; ++e) a[e] += b[e];
      const uint4 packed = pack8(a);  // the new residual is a bf16 tensor: round once
      xr[i] = packed;
      unpack8(packed, v[k]);
#pragma unroll
      for (int e = 0; e < 8; ++e) ss += v[k][e] * v[k][e];
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  __shared__ float part[kNormThreads / 32];
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = ss;
  __syncthreads();
  float tot = 0.f;
#pragma unroll
  for (int i = 0; i < kNormThreads / 32; ++i) tot += part[i];
  const float r = rsqrtf(tot / (float)D + eps);
#pragma unroll
  for (int k = 0; k < kNormMaxVec; ++k) {
    const int i = threadIdx.x + k * kNormThreads;
    if (i < nv) {
      float g[8], o[8];
      unpack8(gw[k], g);
#pragma unroll
      for (int e = 0; e < 8; ++e) o[e] = __bfloat162float(__float2bfloat16_rn(v[k][e] * r)) * g[e];
      hr[i] = pack8(o);
    }
  }
}

// blockIdx.y = row, threads stride the row's 16-B vectors (no 64-bit division)
__global__ void silu_mul_kernel(const uint16_t* __restrict__ gu, uint16_t* __restrict__ y, int64_t rows, int F) {
  const int nvr = F / 8;  // vectors per output row
  const int64_t r = blockIdx.y;
  const uint4* gp = reinterpret_cast<const uint4*>(gu + r * 2 * (int64_t)F);
  const uint4* up = reinterpret_cast<const uint4*>(gu + r * 2 * (int64_t)F + F);
  uint4* yp = reinterpret_cast<uint4*>(y + r * (int64_t)F);
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < nvr; c += gridDim.x * blockDim.x) {
    float g[8], u[8], o[8];
    unpack8(__ldg(gp + c), g);
    unpack8(__ldg(up + c), u);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      // torch: silu in fp32, rounded to bf16, then the bf16 product
      const float s = __bfloat162float(__float2bfloat16_rn(g[e] / (1.f + __expf(-g[e]))));
      o[e] = s * u[e];
    }
    yp[c] = pack8(o);
  }
}

}  // namespace tf

using namespace tf;

extern "C" {

int tf_rmsnorm(const void* x, const void* w, void* y, int32_t rows, int32_t dim, float eps, void* stream) {
  TF_CHECK_ARG(rows >= 0 && dim > 0 && dim % 8 == 0 && dim <= kNormThreads * kNormMaxVec * 8,
               "tf_rmsnorm: bad shape %d x %d", rows, dim);
  if (rows == 0) return TF_OK;
  TF_CHECK_ARG(x && w && y, "tf_rmsnorm: NULL pointer");
  rmsnorm_kernel<<<rows, kNormThreads, 0, (cudaStream_t)stream>>>((const uint16_t*)x, (const uint16_t*)w,
                                                                  (uint16_t*)y, dim, eps);
  TF_LAUNCH_CHECK();
  return TF_OK;
}

int tf_residual_rmsnorm(void* x, const void* y, const void* w, void* h, int32_t rows, int32_t dim, float eps,
                        void* stream) {
  TF_CHECK_ARG(rows >= 0 && dim > 0 && dim % 8 == 0 && dim <= kNormThreads * kNormMaxVec * 8,
               "tf_residual_rmsnorm: bad shape %d x %d", rows, dim);
  if (rows == 0) return TF_OK;
  TF_CHECK_ARG(x && y && w && h, "tf_residual_rmsnorm: NULL pointer");
  residual_rmsnorm_kernel<<<rows, kNormThreads, 0, (cudaStream_t)stream>>>((uint16_t*)x, (const uint16_t*)y,
                                                                           (const uint16_t*)w, (uint16_t*)h, dim, eps);
  TF_LAUNCH_CHECK();
  return TF_OK;
}

int tf_silu_mul(const void* gu, void* y, int32_t rows, int32_t ffn, void* stream) {
  TF_CHECK_ARG(rows >= 0 && ffn > 0 && ffn % 8 == 0, "tf_silu_mul: bad shape %d x %d", rows, ffn);
  if (rows == 0) return TF_OK;
  TF_CHECK_ARG(gu && y, "tf_silu_mul: NULL pointer");
  const int nvr = ffn / 8;
  for (int32_t r0 = 0; r0 < rows; r0 += 65535) {  // grid.y limit (prefills of > 64K tokens)
    const int32_t nr = rows - r0 < 65535 ? rows - r0 : 65535;
    dim3 grid((unsigned)std::max(1, std::min((nvr + 255) / 256, 64)), (unsigned)nr);
    silu_mul_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>((const uint16_t*)gu + (int64_t)r0 * 2 * ffn,
                                                            (uint16_t*)y + (int64_t)r0 * ffn, nr, ffn);
    TF_LAUNCH_CHECK();
  }
  return TF_OK;
}

}  // extern "C"
