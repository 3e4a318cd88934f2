// capi.cu — the extern "C" boundary (include/cpm.h): argument checks, host-pointer
// staging, error state, profiling.  Every compute step runs in the kernels of
// build.cu / apply.cu / krylov.cu / ras.cu / problems.cu.
#include <cuda_runtime.h>

#include <atomic>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "internal.cuh"
#include "krylov.cuh"

namespace cpm {

// ------------------------------------------------------------------ errors
static thread_local std::string g_err;

void set_error(const std::string& msg) { g_err = msg; }
int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}
int cuda_fail(cudaError_t e, const char* what, const char* file, int line) {
  g_err = std::string("CUDA error ") + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) +
          ") in " + what + " at " + file + ":" + std::to_string(line);
  return CPM_ERR_CUDA;
}

// ------------------------------------------------------------------ profiling
namespace {
std::atomic<int64_t> g_launches{0};
std::mutex g_prof_mu;
bool g_prof_on = false;
struct Pending {
  int id;
  cudaEvent_t a, b;
};
std::vector<Pending> g_pending;
std::vector<cudaEvent_t> g_pool;
double g_ms[K_COUNT] = {0};
int64_t g_cnt[K_COUNT] = {0};
const char* g_names[K_COUNT] = {"extend", "laplace", "mdot", "cgs_update", "cgs_final", "axpy", "other"};

cudaEvent_t take_event() {
  if (!g_pool.empty()) {
    cudaEvent_t e = g_pool.back();
    g_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}
void drain_pending() {
  for (auto& p : g_pending) {
    cudaEventSynchronize(p.b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, p.a, p.b);
    g_ms[p.id] += ms;
    g_cnt[p.id] += 1;
    g_pool.push_back(p.a);
    g_pool.push_back(p.b);
  }
  g_pending.clear();
}
}  // namespace

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

bool pdl_enabled() {
  static const bool on = [] {
    const char* v = getenv("CPM_PDL");
    return !v || *v != '0';
  }();
  return on;
}

ProfScope::ProfScope(KernelId id_, cudaStream_t s_) : id(id_), s(s_) {
  if (!g_prof_on) return;
  std::lock_guard<std::mutex> lk(g_prof_mu);
  a = take_event();
  b = take_event();
  cudaEventRecord(a, s);
}
ProfScope::~ProfScope() {
  if (!a) return;
  std::lock_guard<std::mutex> lk(g_prof_mu);
  cudaEventRecord(b, s);
  g_pending.push_back({(int)id, a, b});
  if (g_pending.size() > 4096) drain_pending();
}

// ------------------------------------------------------------------ pointers
bool is_device_ptr(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

void free_workspace(Workspace* w) { delete w; }

Workspace& band_ws(const cpm_band* b) {
  cpm_band* mb = const_cast<cpm_band*>(b);
  if (!mb->ws) mb->ws = new Workspace();
  return *mb->ws;
}

static int ensure_stage(const cpm_band* b) {
  cpm_band* mb = const_cast<cpm_band*>(b);
  if (!mb->dstage0) {
    CPM_CUDA(cudaMalloc(&mb->dstage0, sizeof(double) * std::max<int64_t>(b->nA, 1)));
    CPM_CUDA(cudaMalloc(&mb->dstage1, sizeof(double) * std::max<int64_t>(b->nA, 1)));
  }
  return CPM_OK;
}

}  // namespace cpm

using namespace cpm;

extern "C" {

const char* cpm_version(void) { return "paper_2110_06322_b200 cpm 0.1 (sm_100a)"; }
const char* cpm_last_error(void) { return g_err.c_str(); }

int cpm_build_band(const cpm_surface* surface, double h, int p, double L, void* stream,
                   cpm_band** out) {
  return build_band(surface, h, p, L, (cudaStream_t)stream, out);
}

int cpm_band_get_info(const cpm_band* b, cpm_band_info* info) {
  if (!b || !info) return fail(CPM_ERR_ARG, "cpm_band_get_info: null argument");
  memset(info, 0, sizeof(*info));
  info->n_active = b->nA;
  info->n_ghost = b->nG;
  info->n_tiles = b->nT;
  info->n_runs = b->nRuns;
  info->max_box = b->maxBox;
  info->bytes_device = b->bytes;
  info->h = b->h;
  info->lambda = b->lam;
  info->L = b->L;
  for (int q = 0; q < 3; ++q) {
    info->lattice_lo[q] = b->ilo[q];
    info->lattice_hi[q] = b->ihi[q];
  }
  info->zero_fill = b->zeroFill ? 1 : 0;
  info->rank = b->rank;
  info->nranks = b->nranks;
  info->n_owned = b->nOwned;
  info->n_halo = b->nHalo;
  return CPM_OK;
}

int cpm_band_active_coords(const cpm_band* b, int32_t* ijk_host) {
  if (!b || !ijk_host) return fail(CPM_ERR_ARG, "cpm_band_active_coords: null argument");
  CPM_CUDA(cudaMemcpy(ijk_host, b->aijk, sizeof(int32_t) * 3 * b->nA, cudaMemcpyDeviceToHost));
  return CPM_OK;
}

int cpm_band_ghost_coords(const cpm_band* b, int32_t* ijk_host) {
  if (!b || !ijk_host) return fail(CPM_ERR_ARG, "cpm_band_ghost_coords: null argument");
  if (b->nG > 0)
    CPM_CUDA(cudaMemcpy(ijk_host, b->gijk, sizeof(int32_t) * 3 * b->nG, cudaMemcpyDeviceToHost));
  return CPM_OK;
}

int cpm_band_eval_order(const cpm_band* b, int32_t* tiles_host, uint32_t* eoff_host) {
  if (!b || !tiles_host) return fail(CPM_ERR_ARG, "cpm_band_eval_order: null argument");
  std::vector<TileHdr> T((size_t)b->nT);
  if (b->nT > 0)
    CPM_CUDA(cudaMemcpy(T.data(), b->tiles, sizeof(TileHdr) * b->nT, cudaMemcpyDeviceToHost));
  for (int64_t t = 0; t < b->nT; ++t) {
    int32_t* o = tiles_host + 6 * t;
    o[0] = T[t].e0;
    o[1] = T[t].e1;
    o[2] = b->itemOrder ? (int32_t)(0x40000000 | T[t].pad2) : (T[t].np | (T[t].pad2 << 16));
    o[3] = T[t].pad[0];
    o[4] = T[t].pad[1];
    o[5] = T[t].pad[1] * T[t].sz;
  }
  if (eoff_host && b->nT > 0) {
    const int64_t ne = T[b->nT - 1].e1;
    CPM_CUDA(cudaMemcpy(eoff_host, b->eoff, sizeof(uint32_t) * ne, cudaMemcpyDeviceToHost));
  }
  return CPM_OK;
}

int cpm_band_item_rounds(const cpm_band* b, uint64_t* rounds_host) {
  if (!b || !rounds_host) return fail(CPM_ERR_ARG, "cpm_band_item_rounds: null argument");
  if (!b->itemOrder || !b->rnd) return fail(CPM_ERR_ARG, "cpm_band_item_rounds: band is in pair order");
  if (b->nT > 0)
    CPM_CUDA(cudaMemcpy(rounds_host, b->rnd, sizeof(uint64_t) * 32 * (size_t)b->nT, cudaMemcpyDeviceToHost));
  return CPM_OK;
}

void cpm_band_free(cpm_band* b) { free_band(b); }

int cpm_apply(const cpm_band* b, double c, const double* u, double* y, void* stream) {
  if (!b || !u || !y) return fail(CPM_ERR_ARG, "cpm_apply: null argument");
  if ((const void*)u == (const void*)y) return fail(CPM_ERR_ARG, "cpm_apply: u and y must not alias");
  cudaStream_t s = (cudaStream_t)stream;
  const bool du = is_device_ptr(u), dy = is_device_ptr(y);
  if (du && dy) return apply_device(b, c, u, y, nullptr, 0, s);
  CPM_TRY(ensure_stage(b));
  const size_t bytes = sizeof(double) * b->nA;
  const double* uu = u;
  if (!du) {
    CPM_CUDA(cudaMemcpyAsync(b->dstage0, u, bytes, cudaMemcpyHostToDevice, s));
    uu = b->dstage0;
  }
  double* yy = dy ? y : b->dstage1;
  CPM_TRY(apply_device(b, c, uu, yy, nullptr, 0, s));
  if (!dy) CPM_CUDA(cudaMemcpyAsync(y, yy, bytes, cudaMemcpyDeviceToHost, s));
  CPM_CUDA(cudaStreamSynchronize(s));
  return CPM_OK;
}

static bool is_pinned_host(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

// Pipelined host-buffer apply: call i copies u in on the copy-in stream, applies on
// the caller's stream, copies y out on the copy-out stream, through staging slot
// i % 2, and returns.  The copy-in of call i+1 waits only for the kernels of call
// i-1 (its slot's previous reader), so it overlaps call i's apply and copy-out: the
// two directions of the PCIe link and the kernels run concurrently.
int cpm_apply_async(const cpm_band* b, double c, const double* u, double* y, void* stream) {
  if (!b || !u || !y) return fail(CPM_ERR_ARG, "cpm_apply_async: null argument");
  if ((const void*)u == (const void*)y) return fail(CPM_ERR_ARG, "cpm_apply_async: u and y must not alias");
  if (!is_pinned_host(u) || !is_pinned_host(y)) return cpm_apply(b, c, u, y, stream);
  cudaStream_t s = (cudaStream_t)stream;
  cpm_band* mb = const_cast<cpm_band*>(b);
  if (!mb->as) {  // staging slots, streams, events: all or nothing
    auto* a = new cpm_band::AsyncStage();
    bool ok = true;
    const size_t bytes = sizeof(double) * std::max<int64_t>(b->nA, 1);
    for (int q = 0; q < 2 && ok; ++q) {
      ok = cudaMalloc(&a->u[q], bytes) == cudaSuccess && cudaMalloc(&a->y[q], bytes) == cudaSuccess &&
           cudaEventCreateWithFlags(&a->ein[q], cudaEventDisableTiming) == cudaSuccess &&
           cudaEventCreateWithFlags(&a->ek[q], cudaEventDisableTiming) == cudaSuccess &&
           cudaEventCreateWithFlags(&a->eout[q], cudaEventDisableTiming) == cudaSuccess &&
           cudaEventRecord(a->ek[q], s) == cudaSuccess && cudaEventRecord(a->eout[q], s) == cudaSuccess;
    }
    ok = ok && cudaStreamCreateWithFlags(&a->in, cudaStreamNonBlocking) == cudaSuccess &&
         cudaStreamCreateWithFlags(&a->out, cudaStreamNonBlocking) == cudaSuccess;
    if (!ok) {
      cudaGetLastError();
      for (int q = 0; q < 2; ++q) {
        if (a->u[q]) cudaFree(a->u[q]);
        if (a->y[q]) cudaFree(a->y[q]);
        for (cudaEvent_t e : {a->ein[q], a->ek[q], a->eout[q]})
          if (e) cudaEventDestroy(e);
      }
      if (a->in) cudaStreamDestroy(a->in);
      delete a;
      return fail(CPM_ERR_NOMEM, "cpm_apply_async: staging allocation failed");
    }
    mb->as = a;
  }
  cpm_band::AsyncStage* a = mb->as;
  const int q = (int)(a->calls++ & 1u);
  const size_t bytes = sizeof(double) * b->nA;
  CPM_CUDA(cudaStreamWaitEvent(a->in, a->ek[q], 0));      // slot q's previous apply has read u
  CPM_CUDA(cudaMemcpyAsync(a->u[q], u, bytes, cudaMemcpyHostToDevice, a->in));
  CPM_CUDA(cudaEventRecord(a->ein[q], a->in));
  CPM_CUDA(cudaStreamWaitEvent(s, a->ein[q], 0));
  CPM_CUDA(cudaStreamWaitEvent(s, a->eout[q], 0));        // slot q's previous y has been copied out
  CPM_TRY(apply_device(b, c, a->u[q], a->y[q], nullptr, 0, s));
  CPM_CUDA(cudaEventRecord(a->ek[q], s));
  CPM_CUDA(cudaStreamWaitEvent(a->out, a->ek[q], 0));
  CPM_CUDA(cudaMemcpyAsync(y, a->y[q], bytes, cudaMemcpyDeviceToHost, a->out));
  CPM_CUDA(cudaEventRecord(a->eout[q], a->out));
  return CPM_OK;
}

int cpm_apply_sync(const cpm_band* b) {
  if (!b) return fail(CPM_ERR_ARG, "cpm_apply_sync: null band");
  if (b->as) {
    CPM_CUDA(cudaStreamSynchronize(b->as->in));
    CPM_CUDA(cudaStreamSynchronize(b->as->out));
  }
  return CPM_OK;
}

int cpm_solve(const cpm_band* b, double c, const double* f, double* u, double rtol, int restart,
              int maxit, const cpm_ras* ras, cpm_solve_stats* stats, void* stream);

int cpm_eval_sph(const cpm_band* b, int l, int m, double scale, double* out, void* stream) {
  if (!b || !out) return fail(CPM_ERR_ARG, "cpm_eval_sph: null argument");
  cudaStream_t s = (cudaStream_t)stream;
  if (is_device_ptr(out)) return eval_sph_device(b, l, m, scale, out, s);
  CPM_TRY(ensure_stage(b));
  CPM_TRY(eval_sph_device(b, l, m, scale, b->dstage1, s));
  CPM_CUDA(cudaMemcpyAsync(out, b->dstage1, sizeof(double) * b->nA, cudaMemcpyDeviceToHost, s));
  CPM_CUDA(cudaStreamSynchronize(s));
  return CPM_OK;
}

int cpm_eval_torus_rhs(const cpm_band* b, const double* coeffs, int nq, double* out,
                       void* stream) {
  if (!b || !out) return fail(CPM_ERR_ARG, "cpm_eval_torus_rhs: null argument");
  cudaStream_t s = (cudaStream_t)stream;
  if (is_device_ptr(out)) return eval_torus_device(b, coeffs, nq, out, s);
  CPM_TRY(ensure_stage(b));
  CPM_TRY(eval_torus_device(b, coeffs, nq, b->dstage1, s));
  CPM_CUDA(cudaMemcpyAsync(out, b->dstage1, sizeof(double) * b->nA, cudaMemcpyDeviceToHost, s));
  CPM_CUDA(cudaStreamSynchronize(s));
  return CPM_OK;
}

int cpm_profile_enable(int on) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  g_prof_on = on != 0;
  return CPM_OK;
}
int cpm_profile_reset(void) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  drain_pending();
  for (int q = 0; q < K_COUNT; ++q) {
    g_ms[q] = 0;
    g_cnt[q] = 0;
  }
  return CPM_OK;
}
int cpm_profile_read(const char* name, double* ms, int64_t* launches) {
  if (!name) return fail(CPM_ERR_ARG, "cpm_profile_read: null name");
  std::lock_guard<std::mutex> lk(g_prof_mu);
  drain_pending();
  for (int q = 0; q < K_COUNT; ++q)
    if (strcmp(name, g_names[q]) == 0) {
      if (ms) *ms = g_ms[q];
      if (launches) *launches = g_cnt[q];
      return CPM_OK;
    }
  return fail(CPM_ERR_ARG, std::string("cpm_profile_read: unknown kernel name ") + name);
}
int64_t cpm_kernel_launches(void) { return g_launches.load(); }

}  // extern "C"
