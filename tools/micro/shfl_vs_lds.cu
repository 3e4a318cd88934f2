// Microbenchmark: does SHFL consume the same SM throughput as shared-memory loads?
// A: 64 LDS.64 per iteration; B: 32 LDS.64 + 32 SHFL.64; C: 64 SHFL.64.  All lanes active,
// conflict-free smem addresses, results folded into an FMA chain (kept alive).
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void __launch_bounds__(256) k(int iters, double* out) {
  __shared__ double sm[4096];
  const int tid = threadIdx.x, lane = tid & 31;
  for (int i = tid; i < 4096; i += 256) sm[i] = 1.0 + i * 1e-6;
  __syncthreads();
  double acc = 0.0, v = 1.0 + lane;
  int base = ((tid >> 5) * 64) & 1023;  // warp-uniform: 32 consecutive doubles per LDS.64
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int q = 0; q < 64; ++q) {
      double x;
      if (MODE == 3) {          // lanes 2i, 2i+1 read the same double: 16 distinct per warp
        x = sm[(base + q * 32 + (lane >> 1)) & 4095];
      } else if (MODE == 4) {   // 8 distinct doubles per warp (4 lanes each)
        x = sm[(base + q * 32 + (lane >> 2)) & 4095];
      } else if (MODE == 6) {   // 16 distinct doubles, scattered (stride 17: distinct banks)
        x = sm[(base + q * 32 + (lane >> 1) * 17) & 4095];
      } else if (MODE == 7) {   // 8 distinct in one 64-B block + 8 in another 64-B block 1 KB away
        x = sm[(base + q * 32 + (lane & 15) / 2 + (lane >> 4) * 136) & 4095];
      } else if (MODE == 8) {   // 11 groups of ~3 lanes, scattered bases, distinct banks
        x = sm[(base + q * 32 + (lane / 3) * 37) & 4095];
      } else if (MODE == 9) {   // 16 groups of 2 lanes, scattered bases, distinct banks (stride 37)
        x = sm[(base + q * 32 + (lane >> 1) * 37) & 4095];
      } else if (MODE == 10) {  // 16 groups of 2 lanes, each group's pair split across halves
        x = sm[(base + q * 32 + (lane & 15) * 37) & 4095];
      } else if (MODE == 5) {   // one double for the whole warp
        x = sm[(base + q * 32) & 4095];
      } else if (MODE == 0 || (MODE == 1 && (q & 1) == 0)) {
        x = sm[(base + q * 32 + lane) & 4095];
      } else {
        x = __shfl_sync(0xffffffffu, v, (lane + q) & 31);
      }
      acc = fma(acc, 0.999999, x);
      v += 1e-9;
    }
    base = (base + 7) & 1023;
  }
  if (acc == 12345.0) out[0] = acc;
}

int main() {
  double* out;
  cudaMalloc(&out, 8);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int grid = sms * 8, iters = 2000;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const char* names[11] = {"64 LDS.64", "32 LDS.64 + 32 SHFL.64", "64 SHFL.64",
                          "64 LDS.64, 16 distinct/warp", "64 LDS.64, 8 distinct/warp",
                          "64 LDS.64, 1 distinct/warp", "16 distinct, stride 17",
                          "8+8 distinct, two 64-B blocks", "11 groups of 3, stride 37",
                          "16 pairs, stride 37", "16 pairs split across halves"};
  for (int rep = 0; rep < 1; ++rep)
    for (int m = 0; m < 11; ++m) {
      cudaEventRecord(a);
      if (m == 0) k<0><<<grid, 256>>>(iters, out);
      if (m == 1) k<1><<<grid, 256>>>(iters, out);
      if (m == 2) k<2><<<grid, 256>>>(iters, out);
      if (m == 3) k<3><<<grid, 256>>>(iters, out);
      if (m == 4) k<4><<<grid, 256>>>(iters, out);
      if (m == 5) k<5><<<grid, 256>>>(iters, out);
      if (m == 6) k<6><<<grid, 256>>>(iters, out);
      if (m == 7) k<7><<<grid, 256>>>(iters, out);
      if (m == 8) k<8><<<grid, 256>>>(iters, out);
      if (m == 9) k<9><<<grid, 256>>>(iters, out);
      if (m == 10) k<10><<<grid, 256>>>(iters, out);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double warp_iters = (double)grid * 8 * iters;  // per SM: /sms
      printf("%-26s %.3f ms  -> %.2f clk-ish per 64-load warp-iteration per SM (at 1.965 GHz)\n", names[m], ms,
             ms * 1e-3 * 1.965e9 / (warp_iters / sms));
    }
  return 0;
}
