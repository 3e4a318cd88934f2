// internal.cuh — private definitions of the CPM CUDA library (not part of the ABI).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <utility>
#include <vector>

#include "../../include/cpm.h"

struct cpm_band;

namespace cpm {

constexpr int kBrick = 8;                 // brick edge (lattice cells)
constexpr int kBrickCells = 512;          // 8^3
constexpr int kMaxBoxEdge = 30;           // per-axis cap of a tile's stencil box
constexpr int kMaxBoxCells = 12288;       // 96 KiB of doubles per tile box
constexpr int kMortonBias = 1 << 16;      // brick coordinate bias (reading R8)

// ------------------------------------------------------------------ error state
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what, const char* file, int line);

#define CPM_CUDA(call)                                                   \
  do {                                                                   \
    cudaError_t _e = (call);                                             \
    if (_e != cudaSuccess) return ::cpm::cuda_fail(_e, #call, __FILE__, __LINE__); \
  } while (0)

#define CPM_TRY(call)             \
  do {                            \
    int _rc = (call);             \
    if (_rc != CPM_OK) return _rc; \
  } while (0)

// ------------------------------------------------------------------ profiling
// Kernel ids for cpm_profile_read.
enum KernelId { K_EXTEND = 0, K_LAPLACE, K_MDOT, K_CGS_UPDATE, K_CGS_FINAL, K_AXPY, K_OTHER, K_COUNT };
struct ProfScope {
  ProfScope(KernelId id, cudaStream_t s);
  ~ProfScope();
  KernelId id;
  cudaStream_t s;
  cudaEvent_t a = nullptr, b = nullptr;
};
void count_launch();

// Programmatic dependent launch for the per-step kernels (extend, laplace, the
// two Krylov passes): the next kernel's CTAs are launched while the previous
// grid drains and wait in pdl_wait() (griddepcontrol.wait: the predecessor has
// completed and its writes are visible) before touching any data.  Every kernel
// launched with launch_pdl calls pdl_wait() first.  CPM_PDL=0 disables it.
bool pdl_enabled();
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
// Early trigger, called right after pdl_wait() by the Krylov reduction passes only:
// the update pass that follows may launch once every CTA of the reduction pass has
// started, and loads its first tile (Q columns, u_j, z: written two or more kernels
// back) before its own pdl_wait(), while the reduction's completing block runs the
// GMRES step epilogue (config-1 solve 0.887 -> 0.883 s).  Its pdl_wait() still waits
// for this grid's completion and memory flush.  Triggering in every per-step kernel
// (extend, laplace, update too) was measured: solve 1.05 s — the waiting dependents'
// CTAs cost the draining grids more than their early start saves.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// L2 persistence window of a launch (the E u bricks between extend and laplace,
// apply.cu): {base, bytes}; bytes == 0: none.
struct L2Window {
  void* base = nullptr;
  size_t bytes = 0;
  float hit = 1.0f;
};
L2Window vb_window(const cpm_band* b);  // apply.cu
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl_l2(const L2Window& w, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                                 cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  int na = 0;
  if (pdl_enabled()) {
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if (w.bytes) {
    at[na].id = cudaLaunchAttributeAccessPolicyWindow;
    at[na].val.accessPolicyWindow.base_ptr = w.base;
    at[na].val.accessPolicyWindow.num_bytes = w.bytes;
    at[na].val.accessPolicyWindow.hitRatio = w.hit;
    at[na].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    at[na].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    ++na;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// ------------------------------------------------------------------ band data
// One tile = one occupied 8^3 brick.  176 bytes, 16-byte aligned: the fields every
// thread of the extend needs (e0..pad2, then the strides) come first, so it reads
// them with two 16-byte and one 8-byte load instead of eight 4-byte loads.
// E u of the tile's eval nodes lives in vb[slot * 512 + cell] (only the cells set
// in emask are written by the extend).
struct alignas(16) TileHdr {
  int32_t e0, e1;      // eval nodes (Sigma_A u Sigma_G in the brick) [e0, e1)
  int32_t a0, a1;      // output (active / owned) nodes [a0, a1)
  int32_t r0, r1;      // stencil-box fill runs [r0, r1)
  int32_t np;          // pair order: eval nodes e0 + 2p, e0 + 2p + 1 (p < np) share a stencil base;
                       // item order: index of the tile's first round word in cpm_band::rnd
  int32_t pad2;        // pair order: nd, unpaired nodes 2np .. 2np+nd-1 run on lane pairs (the
                       // rest one per lane); item order: number of rounds
  int32_t pad[3];      // row stride, plane stride of the box; segment id (RAS)
  int32_t ox, oy, oz;  // stencil box origin (lattice)
  int32_t sx, sy, sz;  // stencil box extent (cells)
  int32_t nbr[6];      // face neighbour tile slots (+x,-x,+y,-y,+z,-z), -1 = none
  int32_t bx, by, bz;  // brick coordinates (lattice origin = 8*b)
  uint32_t emask[16];  // eval-node cells of the brick (Sigma_A u Sigma_G), bit = cell
  int32_t spare[2];
};
static_assert(sizeof(TileHdr) == 176 && alignof(TileHdr) == 16, "TileHdr layout");

__host__ __device__ inline int popc32(uint32_t v) {
#ifdef __CUDA_ARCH__
  return __popc(v);
#else
  return __builtin_popcount(v);
#endif
}

// A fill run copies len consecutive source doubles u[src..src+len) to
// box[dst..dst+len).  Packed: src (bits 0-31), dst (32-47), len (48-55).
__host__ __device__ inline uint64_t pack_run(uint32_t src, uint32_t dst, uint32_t len) {
  return (uint64_t)src | ((uint64_t)dst << 32) | ((uint64_t)len << 48);
}

struct Surface {
  int kind;
  double p[4];
};

struct Workspace;  // krylov.cuh

}  // namespace cpm

// The band handle.  All pointers are device memory unless noted.
struct cpm_band {
  cpm::Surface surf;
  double h = 0, lam = 0, L = 0;
  int M = 0;
  int64_t nA = 0, nG = 0, nE = 0;  // active, ghost, eval (= nA + nG for a full band)
  int nT = 0;                      // tiles
  int nTint = 0;                   // partitioned sub-bands: tiles [0, nTint) read no halo source
  int64_t nRuns = 0;
  int maxBox = 0;
  bool zeroFill = false;
  int ilo[3] = {0, 0, 0}, ihi[3] = {0, 0, 0};
  int rank = 0, nranks = 1;
  int64_t nOwned = 0, nHalo = 0;   // partitioned bands

  cpm::TileHdr* tiles = nullptr;
  double* tx = nullptr;            // nE fractional offsets (SoA)
  double* ty = nullptr;
  double* tz = nullptr;
  uint32_t* eoff = nullptr;        // nE: box offset (low 16) | brick cell of the node (high 16)
  uint16_t* acell = nullptr;       // nA: brick cell of each output node
  int32_t* aijk = nullptr;         // 3*nA lattice coords (band order)
  int32_t* gijk = nullptr;         // 3*nG lattice coords
  uint64_t* runs = nullptr;        // nRuns fill runs
  double* vb = nullptr;            // nT*512 scratch: E u per brick cell
  uint32_t* amask = nullptr;       // nT*16: Sigma_A occupancy bits of each tile's brick
  int* bmap = nullptr;             // dense brick map over the brick box -> tile slot or -1
  int blo[3] = {0, 0, 0}, bdim[3] = {0, 0, 0};
  bool owns = true;                // false for sub-bands sharing the eval arrays
  uint32_t srcSplit = 0xffffffffu; // fill-run sources >= srcSplit read the halo buffer
  // node order of the extend: items (k_extend_it, rounds in rnd; TileHdr np = first
  // round, pad2 = rounds) or pairs (k_extend_nt; np = pairs, pad2 = unpaired on lane pairs)
  bool itemOrder = false;
  uint64_t* rnd = nullptr;
  // TMA laplace (apply.cu k_laplace_tma): CUtensorMaps over vb, encoded on first use
  alignas(64) unsigned char tmX[128] = {}, tmY[128] = {};
  bool tmReady = false;

  // host staging for host-pointer calls
  double* dstage0 = nullptr;       // nA
  double* dstage1 = nullptr;       // nA
  // cpm_apply_async (pinned host buffers): two staging slots, copy-in / copy-out streams
  struct AsyncStage {
    double* u[2] = {nullptr, nullptr};
    double* y[2] = {nullptr, nullptr};
    cudaStream_t in = nullptr, out = nullptr;
    cudaEvent_t ein[2] = {nullptr, nullptr}, ek[2] = {nullptr, nullptr}, eout[2] = {nullptr, nullptr};
    unsigned calls = 0;
  };
  AsyncStage* as = nullptr;
  int64_t bytes = 0;
  cpm::Workspace* ws = nullptr;    // cached GMRES workspace (host-owned object)

  // single-kernel (fused) apply, an experiment built when CPM_FUSED=1 at band build
  // (build.cu build_fused, apply.cu k_apply_fused)
  cpm::TileHdr* fzT = nullptr;     // per tile: the fused box (origin, extents, strides, runs)
  int* fzH = nullptr;              // nT + 1: halo node ranges
  uint64_t* fzHalo = nullptr;      // halo nodes: eval index | box offset << 32 | halo cell << 48
  uint32_t* fzEoff = nullptr;      // own eval nodes: fused box offset | cell << 16
  uint64_t* fzRuns = nullptr;
  int fzMaxBox = 0;
  int64_t fzNHalo = 0, fzNRuns = 0;
};

namespace cpm {
// apply.cu
// y = scale_seg * (c - Delta_S^h) u ; scale (device, may be null) is read at
// scale[seg * lds] with seg = the tile's segment id (0 for a plain band).
// skip (device, may be null): when *skip != 0 at kernel start the kernels return
// without work (GMRES steps queued past convergence).
int apply_device(const cpm_band* b, double c, const double* u, double* y, const double* scale,
                 int lds, cudaStream_t s, const int* skip = nullptr);
// as apply_device, with fill-run sources >= b->srcSplit read from uh[src - srcSplit]
int apply_device_split(const cpm_band* b, double c, const double* u, const double* uh, double* y,
                       const double* scale, int lds, cudaStream_t s, const int* skip = nullptr);
// The two halves of apply_device_split, for the overlapped partitioned apply
// (part.cu): the extend of tiles [t0, t1) (E u into vb), and the laplace of all tiles.
int extend_tiles(const cpm_band* b, const double* u, const double* uh, cudaStream_t s, const int* skip,
                 int t0, int t1);
int laplace_tiles(const cpm_band* b, double c, const double* u, double* y, const double* scale, int lds,
                  cudaStream_t s, const int* skip);
// build.cu
int build_band(const cpm_surface* surf, double h, int p, double L, cudaStream_t s, cpm_band** out);
void free_band(cpm_band* b);
// problems.cu
int eval_sph_device(const cpm_band* b, int l, int m, double scale, double* out, cudaStream_t s);
int eval_torus_device(const cpm_band* b, const double* coeffs, int nq, double* out,
                      cudaStream_t s);
// pointer helpers (capi.cpp)
bool is_device_ptr(const void* p);
}  // namespace cpm
