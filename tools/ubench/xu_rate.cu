// Throughput of MUFU.EX2 vs F2FP.BF16 pack vs FFMA2 on one SM (cycles per
// warp instruction per SM sub-partition), to see which pipe F2FP uses.
#include <cstdio>
#include <cuda_bf16.h>
__device__ __forceinline__ float ex2(float x) { float r; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x)); return r; }
template <int K>
__global__ void k(float* out, long long* cyc, int iters) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 0.001f + i;
  unsigned u[8] = {0};
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (K == 0) a[i] = ex2(a[i]);
      else if (K == 1) { __nv_bfloat162 h = __floats2bfloat162_rn(a[i], a[(i + 1) & 7]); u[i] ^= *reinterpret_cast<unsigned*>(&h); a[i] += 1.0f; }
      else { float2 r = __ffma2_rn(make_float2(a[i], a[(i+1)&7]), make_float2(1.0001f, 1.0001f), make_float2(0.5f, 0.5f)); a[i] = r.x; a[(i+1)&7] += r.y; }
    }
  }
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i] + u[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  float* out; long long* cyc; cudaMalloc(&out, 1 << 20); cudaMalloc(&cyc, 1024);
  const int iters = 4096;
  const char* names[3] = {"MUFU.EX2", "F2FP pack (+FADD)", "FFMA2 (+FADD)"};
  for (int K = 0; K < 3; ++K)
    for (int warps = 4; warps <= 32; warps *= 2) {
      auto f = K == 0 ? k<0> : (K == 1 ? k<1> : k<2>);
      f<<<1, warps * 32>>>(out, cyc, iters); cudaDeviceSynchronize();
      f<<<1, warps * 32>>>(out, cyc, iters);
      long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      double per = (double)c / (iters * 8.0) / (warps / 4.0);  // cycles per warp-instr per SMSP
      printf("%-20s warps/SM %2d: %.2f cycles per op-group per SMSP\n", names[K], warps, per);
    }
  return 0;
}
