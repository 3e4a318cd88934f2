// Microbenchmark: the cost of a warp's LDS.64 when its 32 lanes read 32 distinct
// doubles, by how the bank pairs (address / 8 mod 16, "residues") are spread:
//   0: lane l reads double l (consecutive: each residue twice, lanes l and l+16)
//   1: each half-warp 16 distinct residues, scattered rows (addr = 16*row + residue)
//   2: residue l/2: lanes 2i, 2i+1 same residue, different rows (each residue twice)
//   3: 16 distinct doubles, lanes 2i, 2i+1 share (one wavefront reference)
//   4: each half-warp 16 distinct residues, the two halves the same residues in
//      the same order (lane l and l+16 same residue, different rows)
//   5: 3 lanes per residue in one half (conflicts)
// Cycles per LDS.64 from clock64 around 64 dependent-free loads, 8 warps per SM.
#include <cstdio>
#include <cuda_runtime.h>

__device__ int addr_of(int mode, int lane, int q) {
  const int row = (lane * 7 + q * 5) & 31;  // scattered rows (any row: residue unchanged)
  switch (mode) {
    case 0: return ((q * 32) + lane) & 4095;
    case 1: {
      const int r = lane < 16 ? (lane * 5) & 15 : ((lane - 16) * 3 + 7) & 15;
      return (16 * (row + 32 * (lane >> 4)) + r) & 4095;
    }
    case 2: return (16 * (row + 32 * (lane & 1)) + (lane >> 1)) & 4095;
    case 3: return (16 * ((q * 3) & 31) + (lane >> 1) * 17) & 4095;
    case 4: return (16 * (row + 32 * (lane >> 4)) + (lane & 15)) & 4095;
    default: return (16 * row + (lane < 16 ? lane / 3 : lane & 15)) & 4095;
  }
}

template <int MODE>
__global__ void __launch_bounds__(256) k(int iters, double* out, long long* cyc) {
  __shared__ double sm[4096];
  const int tid = threadIdx.x, lane = tid & 31;
  for (int i = tid; i < 4096; i += 256) sm[i] = 1.0 + i * 1e-6;
  int ad[64];
#pragma unroll
  for (int q = 0; q < 64; ++q) ad[q] = addr_of(MODE, lane, q);
  __syncthreads();
  double acc = 0.0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const int sh = (it & 1) << 9;  // alternate two copies 512 doubles apart (same banks): no hoisting
#pragma unroll
    for (int q = 0; q < 64; ++q) acc += sm[(ad[q] + sh) & 4095];
  }
  long long t1 = clock64();
  if (acc == 12345.0) out[0] = acc;
  if (tid == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 8);
  cudaMalloc(&cyc, 8);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 2000;
  const char* names[6] = {"consecutive (residue twice, l and l+16)", "halves distinct, scattered rows",
                          "residue l/2 (pairs of lanes, different rows)", "16 distinct shared by lane pairs",
                          "halves distinct, same residue order", "3 lanes per residue in half 0"};
  void (*ks[6])(int, double*, long long*) = {k<0>, k<1>, k<2>, k<3>, k<4>, k<5>};
  for (int m = 0; m < 6; ++m) {
    ks[m]<<<sms, 256>>>(iters, out, cyc);  // 8 warps per SM
    cudaDeviceSynchronize();
    long long c = 0;
    ks[m]<<<sms, 256>>>(iters, out, cyc);
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    // 8 warps share the SM's shared-memory pipe: cycles per warp-instruction
    printf("%-48s %.2f cycles per warp LDS.64 (8 warps/SM)\n", names[m], (double)c / (iters * 64.0 * 8));
  }
  return 0;
}
