// Microbenchmark: cost of 128-bit shared loads shared by lane groups, vs the 64-bit
// gathers of the extend (open items).  Each mode delivers 64
// doubles per lane per iteration; clk per warp-iteration per SM is printed.
//   0: 64 LDS.64, lane pairs share an address (16 distinct doubles per warp)  [the extend today]
//   1: 32 LDS.128, lane pairs share (16 distinct 16-B per warp)
//   2: 32 LDS.128, lane quads share (8 distinct 16-B per warp)
//   3: 32 LDS.128, all lanes distinct (32 distinct 16-B)
//   4: 64 LDS.64, lane quads share (8 distinct doubles)
//   5: 32 LDS.128, lane quads share, quads' addresses scattered (stride 37 x 16 B)
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void __launch_bounds__(256) k(int iters, double* out) {
  __shared__ __align__(16) double sm[4096];
  const int tid = threadIdx.x, lane = tid & 31;
  for (int i = tid; i < 4096; i += 256) sm[i] = 1.0 + i * 1e-6;
  __syncthreads();
  double acc = 0.0;
  int base = ((tid >> 5) * 64) & 1023;
  const double2* s2 = (const double2*)sm;
  for (int it = 0; it < iters; ++it) {
    if (MODE == 0 || MODE == 4) {
#pragma unroll
      for (int q = 0; q < 64; ++q) {
        const int idx = MODE == 0 ? (base + q * 32 + (lane >> 1)) : (base + q * 32 + (lane >> 2));
        acc = fma(acc, 0.999999, sm[idx & 4095]);
      }
    } else {
#pragma unroll
      for (int q = 0; q < 32; ++q) {
        int i2;
        if (MODE == 1) i2 = base + q * 16 + (lane >> 1);
        else if (MODE == 2) i2 = base + q * 16 + (lane >> 2);
        else if (MODE == 3) i2 = base + q * 16 + lane;
        else i2 = base + q * 16 + (lane >> 2) * 37;
        const double2 x = s2[i2 & 2047];
        acc = fma(acc, 0.999999, x.x);
        acc = fma(acc, 0.999999, x.y);
      }
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
  const char* names[6] = {"64 LDS.64 pairs", "32 LDS.128 pairs", "32 LDS.128 quads", "32 LDS.128 distinct",
                          "64 LDS.64 quads", "32 LDS.128 quads scattered"};
  for (int m = 0; m < 6; ++m) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      if (m == 0) k<0><<<grid, 256>>>(iters, out);
      if (m == 1) k<1><<<grid, 256>>>(iters, out);
      if (m == 2) k<2><<<grid, 256>>>(iters, out);
      if (m == 3) k<3><<<grid, 256>>>(iters, out);
      if (m == 4) k<4><<<grid, 256>>>(iters, out);
      if (m == 5) k<5><<<grid, 256>>>(iters, out);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double warp_iters = (double)grid * 8 * iters;
      if (rep == 1)
        printf("%-28s %.3f ms  -> %.2f clk per 64-double warp-iteration per SM (at 1.965 GHz)\n", names[m], ms,
               ms * 1e-3 * 1.965e9 / (warp_iters / sms));
    }
  }
  return 0;
}
