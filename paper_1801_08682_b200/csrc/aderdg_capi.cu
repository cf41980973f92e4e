// aderdg_capi.cu — C ABI (include/aderdg_b200.h) over the sm_100a kernels.
//
// The handle owns every device buffer: Q and D per local cell, two parities
// of face-trace records, the device-resident TimeControl (DevState) and the
// step-record ring.  A realisation step is three stream-ordered launches
// (rerun predict [device-conditional] -> fused sweep -> time control) with no
// host synchronisation; adg_step syncs once at the end, adg_run only after
// the last step.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <stdio.h>
#include <string.h>
#include <math.h>
#include <limits.h>
#include <stdlib.h>
#include <atomic>
#include <string>
#include <thread>
#include <vector>

#include "../../include/aderdg_b200.h"
#include "aderdg_kernels.cuh"
#include "aderdg_sweep_p3.cuh"
#include "aderdg_sweep_ho.cuh"
#include "aderdg_sweep_p5.cuh"
#include "aderdg_sweep_p7.cuh"
#include "aderdg_sweep_p9.cuh"
#include "aderdg_sweep_2d_p3.cuh"
#include "aderdg_limiter.cuh"

using namespace adg;

namespace {

typedef void (*launch_fn)(const SweepParams&, unsigned grid, cudaStream_t s);

// The dynamic shared-memory opt-in (cudaFuncAttributeMaxDynamicSharedMemorySize)
// is a property of the function *per device context*: a second handle on another
// GPU of the same process (Driver(device=1), the in-process multi-GPU group) must
// set it again.  One bit per device ordinal; setting it twice is harmless, so a
// relaxed atomic is enough when several host threads launch concurrently.
template <class K>
void ensure_smem_optin(K kernel, size_t bytes, std::atomic<unsigned long long>& done) {
  if (bytes <= 48 * 1024) return;
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_relaxed) & bit) return;
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  // the whole unified L1 / shared array as shared memory: a kernel node of a captured
  // graph otherwise keeps the default carveout, which holds fewer of these CTAs per SM
  cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, (int)cudaSharedmemCarveoutMaxShared);
  done.fetch_or(bit, std::memory_order_relaxed);
}

template <class PDE, int DIM, int NQ>
void launch_sweep(const SweepParams& P, unsigned grid, cudaStream_t s) {
  using S = Shape<DIM, NQ, PDE::M>;
  static std::atomic<unsigned long long> optin{0};
  ensure_smem_optin(sweep_kernel<PDE, DIM, NQ>, S::SMEM_BYTES, optin);
  sweep_kernel<PDE, DIM, NQ><<<grid, S::THREADS, S::SMEM_BYTES, s>>>(P);
}

typedef int (*occupancy_fn)();

// resident CTAs per SM of a kernel with the given block and dynamic shared memory
template <class K>
int occupancy_of(K kernel, int threads, size_t smem) {
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, threads, smem) != cudaSuccess) n = 1;
  return n > 0 ? n : 1;
}

template <class PDE, int DIM, int NQ>
int occ_generic() {
  using S = Shape<DIM, NQ, PDE::M>;
  return occupancy_of(sweep_kernel<PDE, DIM, NQ>, S::THREADS, S::SMEM_BYTES);
}

// sweep + time control in one launch (the last CTA runs finish_body); kernels without it: null
typedef void (*launch_fused_fn)(const SweepParams&, const FinishParams&, unsigned* arrive, unsigned grid,
                                cudaStream_t s);

// `steps` whole realisation steps in one cooperative launch (grid barrier between the steps);
// returns the launch's cudaError_t, grid = 0 asks for the largest co-resident grid
typedef cudaError_t (*launch_run_fn)(const SweepParams&, const FinishParams&, unsigned* sync, double* tr0,
                                     double* tr1, int steps, unsigned cells, cudaStream_t s);

struct Dispatch {
  launch_fn sweep;
  int rec;
  occupancy_fn occ = nullptr;   // resident sweep CTAs per SM (adg_step_host chunking)
  launch_fused_fn sweep_finish = nullptr;
  launch_run_fn run = nullptr;
};

template <int DIM, int NQ>
Dispatch make_dispatch() {
  return Dispatch{&launch_sweep<EulerPDE<DIM>, DIM, NQ>, Shape<DIM, NQ>::REC, &occ_generic<EulerPDE<DIM>, DIM, NQ>};
}

template <int DIM, int NQ>
Dispatch make_dispatch_adv() {
  return Dispatch{&launch_sweep<AdvectionPDE<DIM>, DIM, NQ>, Shape<DIM, NQ, 1>::REC,
                  &occ_generic<AdvectionPDE<DIM>, DIM, NQ>};
}

// AdvectionSystem: the generic kernel with the advection plug-in, every d and p
template <int DIM>
bool dispatch_adv(int n, Dispatch* out) {
  switch (n) {
    case 1: *out = make_dispatch_adv<DIM, 1>(); return true;
    case 2: *out = make_dispatch_adv<DIM, 2>(); return true;
    case 3: *out = make_dispatch_adv<DIM, 3>(); return true;
    case 4: *out = make_dispatch_adv<DIM, 4>(); return true;
    case 5: *out = make_dispatch_adv<DIM, 5>(); return true;
    case 6: *out = make_dispatch_adv<DIM, 6>(); return true;
    case 7: *out = make_dispatch_adv<DIM, 7>(); return true;
    case 8: *out = make_dispatch_adv<DIM, 8>(); return true;
    case 9: *out = make_dispatch_adv<DIM, 9>(); return true;
    case 10: *out = make_dispatch_adv<DIM, 10>(); return true;
  }
  return false;
}

// 3D p = 6 and p = 8 (aderdg_sweep_ho.cuh): DMMA tiles, time line in local memory (+ TMEM)
template <int NQ>
void launch_sweep_ho(const SweepParams& P, unsigned grid, cudaStream_t s) {
  using S = ShapeHO<NQ>;
  static std::atomic<unsigned long long> optin{0};
  ensure_smem_optin(sweep_kernel_ho<NQ>, S::SMEM_BYTES, optin);
  sweep_kernel_ho<NQ><<<grid, S::THREADS, S::SMEM_BYTES, s>>>(P);
}

template <int NQ>
int occ_ho() {
  return occupancy_of(sweep_kernel_ho<NQ>, ShapeHO<NQ>::THREADS, ShapeHO<NQ>::SMEM_BYTES);
}

template <int NQ>
Dispatch make_dispatch_ho() {
  static_assert(ShapeHO<NQ>::REC == Shape<3, NQ>::REC, "record layout must match");
  return Dispatch{&launch_sweep_ho<NQ>, ShapeHO<NQ>::REC, &occ_ho<NQ>};
}

// 3D p = 5: Picard derivatives on DMMA, two CTAs per SM (aderdg_sweep_p5.cuh)
void launch_sweep_p5(const SweepParams& P, unsigned grid, cudaStream_t s) {
  static std::atomic<unsigned long long> optin{0};
  ensure_smem_optin(sweep_kernel_p5, ShapeP5::SMEM_BYTES, optin);
  sweep_kernel_p5<<<grid, ShapeP5::THREADS, ShapeP5::SMEM_BYTES, s>>>(P);
}

int occ_p5() { return occupancy_of(sweep_kernel_p5, ShapeP5::THREADS, ShapeP5::SMEM_BYTES); }

Dispatch make_dispatch_p5() {
  static_assert(ShapeP5::REC == Shape<3, 6>::REC, "record layout must match");
  return Dispatch{&launch_sweep_p5, ShapeP5::REC, &occ_p5};
}

// 3D p = 7: Picard state in TMEM + shared memory, exact DMMA tiles (aderdg_sweep_p7.cuh)
void launch_sweep_p7(const SweepParams& P, unsigned grid, cudaStream_t s) {
  static std::atomic<unsigned long long> optin{0};
  ensure_smem_optin(sweep_kernel_p7, ShapeP7::SMEM_BYTES, optin);
  sweep_kernel_p7<<<grid, ShapeP7::THREADS, ShapeP7::SMEM_BYTES, s>>>(P);
}

int occ_p7() { return occupancy_of(sweep_kernel_p7, ShapeP7::THREADS, ShapeP7::SMEM_BYTES); }

Dispatch make_dispatch_p7() {
  static_assert(ShapeP7::REC == Shape<3, 8>::REC, "record layout must match");
  return Dispatch{&launch_sweep_p7, ShapeP7::REC, &occ_p7};
}

// 3D p = 9: the Picard state of the cell in TMEM + shared memory (aderdg_sweep_p9.cuh)
void launch_sweep_p9(const SweepParams& P, unsigned grid, cudaStream_t s) {
  static std::atomic<unsigned long long> optin{0};
  ensure_smem_optin(sweep_kernel_p9, ShapeP9::SMEM_BYTES, optin);
  sweep_kernel_p9<<<grid, ShapeP9::THREADS, ShapeP9::SMEM_BYTES, s>>>(P);
}

int occ_p9() { return occupancy_of(sweep_kernel_p9, ShapeP9::THREADS, ShapeP9::SMEM_BYTES); }

Dispatch make_dispatch_p9() {
  static_assert(ShapeP9::REC == Shape<3, 10>::REC, "record layout must match");
  return Dispatch{&launch_sweep_p9, ShapeP9::REC, &occ_p9};
}

// 3D p = 3: DMMA axes 1-2 from registers, pipelined slices (aderdg_sweep_p3.cuh)
void launch_sweep_p3(const SweepParams& P, unsigned grid, cudaStream_t s) {
  static std::atomic<unsigned long long> optin{0};
  ensure_smem_optin(sweep_kernel_p3, ShapeP3::SMEM_BYTES, optin);
  sweep_kernel_p3<<<grid, ShapeP3::THREADS, ShapeP3::SMEM_BYTES, s>>>(P);
}

int occ_p3() { return occupancy_of(sweep_kernel_p3, ShapeP3::THREADS, ShapeP3::SMEM_BYTES); }

Dispatch make_dispatch_p3() {
  static_assert(ShapeP3::REC == Shape<3, 4>::REC, "record layout must match");
  return Dispatch{&launch_sweep_p3, ShapeP3::REC, &occ_p3};
}

// 2D p = 3 (BASELINE cfg 1): 128 threads per cell, one barrier per Picard iteration, optional
// fused time control (aderdg_sweep_2d_p3.cuh)
void launch_sweep_2d_p3(const SweepParams& P, unsigned grid, cudaStream_t s) {
  FusedFinish X;
  memset(&X, 0, sizeof X);
  sweep_kernel_2d_p3<<<grid, Shape2P3::THREADS, Shape2P3::SMEM_BYTES, s>>>(P, X);
}

void launch_sweep_2d_p3_finish(const SweepParams& P, const FinishParams& F, unsigned* arrive, unsigned grid,
                               cudaStream_t s) {
  FusedFinish X;
  X.F = F;
  X.arrive = arrive;
  X.on = 1;
  sweep_kernel_2d_p3<<<grid, Shape2P3::THREADS, Shape2P3::SMEM_BYTES, s>>>(P, X);
}

int occ_2d_p3() { return occupancy_of(sweep_kernel_2d_p3, Shape2P3::THREADS, Shape2P3::SMEM_BYTES); }

cudaError_t launch_run_2d_p3(const SweepParams& P, const FinishParams& F, unsigned* sync, double* tr0, double* tr1,
                             int steps, unsigned cells, cudaStream_t s) {
  int dev = 0, sms = 0, per_sm = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e == cudaSuccess)
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, run_kernel_2d_p3, Shape2P3::THREADS,
                                                      Shape2P3::SMEM_BYTES);
  if (e != cudaSuccess) return e;
  const unsigned cap = (unsigned)(sms * per_sm);
  if (cap == 0) return cudaErrorCooperativeLaunchTooLarge;
  RunParams2P3 R;
  R.F = F;
  R.sync = sync;
  R.tr[0] = tr0;
  R.tr[1] = tr1;
  R.steps = steps;
  SweepParams Pc = P;
  void* args[] = {(void*)&Pc, (void*)&R};
  return cudaLaunchCooperativeKernel((const void*)run_kernel_2d_p3, dim3(cells < cap ? cells : cap),
                                     dim3(Shape2P3::THREADS), args, Shape2P3::SMEM_BYTES, s);
}

Dispatch make_dispatch_2d_p3() {
  static_assert(Shape2P3::REC == Shape<2, 4>::REC, "record layout must match");
  static_assert(Shape2P3::SMEM_BYTES <= 48 * 1024, "no dynamic shared-memory opt-in");
  return Dispatch{&launch_sweep_2d_p3, Shape2P3::REC, &occ_2d_p3, &launch_sweep_2d_p3_finish, &launch_run_2d_p3};
}

// subcell limiter kernels (aderdg_limiter.cuh), per PDE plug-in and dimension
struct LimDispatch {
  void (*detect)(const LimParams&, unsigned, size_t, cudaStream_t);
  void (*apply)(const LimParams&, unsigned, cudaStream_t);
};

template <class PDE, int DIM>
void launch_lim_detect(const LimParams& L, unsigned grid, size_t smem, cudaStream_t s) {
  // per device: the largest opt-in set so far (detection smem depends on p only)
  static std::atomic<size_t> optin[64];
  int dev = 0;
  cudaGetDevice(&dev);
  if (smem > optin[dev & 63].load(std::memory_order_relaxed)) {
    cudaFuncSetAttribute(lim_detect_kernel<PDE, DIM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    optin[dev & 63].store(smem, std::memory_order_relaxed);
  }
  lim_detect_kernel<PDE, DIM><<<grid, 256, smem, s>>>(L);
}

template <class PDE, int DIM>
void launch_lim_apply(const LimParams& L, unsigned grid, cudaStream_t s) {
  lim_apply_kernel<PDE, DIM><<<grid, 256, 0, s>>>(L);
}

template <class PDE, int DIM>
LimDispatch make_lim_dispatch() { return LimDispatch{&launch_lim_detect<PDE, DIM>, &launch_lim_apply<PDE, DIM>}; }

LimDispatch lim_dispatch_for(int d, int system) {
  if (system == 1) return d == 2 ? make_lim_dispatch<AdvectionPDE<2>, 2>() : make_lim_dispatch<AdvectionPDE<3>, 3>();
  return d == 2 ? make_lim_dispatch<EulerPDE<2>, 2>() : make_lim_dispatch<EulerPDE<3>, 3>();
}

// the generic kernel (the one with the limiter / outflow hooks) for every Euler (d, p)
bool dispatch_generic(int d, int p, Dispatch* out) {
  const int n = p + 1;
  if (d == 2) {
    switch (n) {
      case 1: *out = make_dispatch<2, 1>(); return true;
      case 2: *out = make_dispatch<2, 2>(); return true;
      case 3: *out = make_dispatch<2, 3>(); return true;
      case 4: *out = make_dispatch<2, 4>(); return true;
      case 5: *out = make_dispatch<2, 5>(); return true;
      case 6: *out = make_dispatch<2, 6>(); return true;
      case 7: *out = make_dispatch<2, 7>(); return true;
      case 8: *out = make_dispatch<2, 8>(); return true;
      case 9: *out = make_dispatch<2, 9>(); return true;
      case 10: *out = make_dispatch<2, 10>(); return true;
    }
  } else if (d == 3) {
    switch (n) {
      case 1: *out = make_dispatch<3, 1>(); return true;
      case 2: *out = make_dispatch<3, 2>(); return true;
      case 3: *out = make_dispatch<3, 3>(); return true;
      case 4: *out = make_dispatch<3, 4>(); return true;
      case 5: *out = make_dispatch<3, 5>(); return true;
      case 6: *out = make_dispatch<3, 6>(); return true;
      case 7: *out = make_dispatch<3, 7>(); return true;
      case 8: *out = make_dispatch<3, 8>(); return true;
      case 9: *out = make_dispatch<3, 9>(); return true;
      case 10: *out = make_dispatch<3, 10>(); return true;
    }
  }
  return false;
}

// The product kernel of every (system, d, p): one instantiation each, no run-time
// variant selection.  3D Euler: p = 3 sweep_kernel_p3 (DMMA axes 1-2, pipelined
// slices), p = 5 sweep_kernel_p5, p = 7 sweep_kernel_p7, p = 9 sweep_kernel_p9,
// p = 6, 8 sweep_kernel_ho; the rest
// (2D, 3D p <= 2, p = 4) run the generic kernel.
bool dispatch_for(int d, int p, int system, Dispatch* out) {
  const int n = p + 1;
  if (system == 1) return d == 2 ? dispatch_adv<2>(n, out) : d == 3 ? dispatch_adv<3>(n, out) : false;
  if (d == 3) {
    switch (n) {
      case 4: *out = make_dispatch_p3(); return true;
      case 6: *out = make_dispatch_p5(); return true;
      case 7: *out = make_dispatch_ho<7>(); return true;
      case 8: *out = make_dispatch_p7(); return true;
      case 9: *out = make_dispatch_ho<9>(); return true;
      case 10: *out = make_dispatch_p9(); return true;
    }
  }
  return dispatch_generic(d, p, out);
}

// 2D Euler p = 3 under the fused driver (periodic): the latency kernel of BASELINE cfg 1.  The
// straightforward driver's passes, outflow boundaries and the limiter stay in the generic kernel.
bool dispatch_small(const adg_config& c, Dispatch* out) {
  if (c.system == 0 && c.d == 2 && c.p == 3 && c.boundary == 0 && c.driver_mode == 0) {
    *out = make_dispatch_2d_p3();
    return true;
  }
  return false;
}

}  // namespace

// NCCL entry points resolved at run time (torch has already loaded libnccl.so.2
// in the bench / test processes; no link-time dependency of the library)
struct NcclApi {
  bool ok = false;
  decltype(&ncclGetUniqueId) getUniqueId = nullptr;
  decltype(&ncclCommInitRank) commInitRank = nullptr;
  decltype(&ncclCommInitAll) commInitAll = nullptr;
  decltype(&ncclCommDestroy) commDestroy = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclGroupStart) groupStart = nullptr;
  decltype(&ncclGroupEnd) groupEnd = nullptr;
  decltype(&ncclAllReduce) allReduce = nullptr;
  decltype(&ncclGetErrorString) errorString = nullptr;
};

static NcclApi& nccl_api() {
  static NcclApi a;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) lib = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (lib) {
      a.getUniqueId = (decltype(a.getUniqueId))dlsym(lib, "ncclGetUniqueId");
      a.commInitRank = (decltype(a.commInitRank))dlsym(lib, "ncclCommInitRank");
      a.commInitAll = (decltype(a.commInitAll))dlsym(lib, "ncclCommInitAll");
      a.commDestroy = (decltype(a.commDestroy))dlsym(lib, "ncclCommDestroy");
      a.send = (decltype(a.send))dlsym(lib, "ncclSend");
      a.recv = (decltype(a.recv))dlsym(lib, "ncclRecv");
      a.groupStart = (decltype(a.groupStart))dlsym(lib, "ncclGroupStart");
      a.groupEnd = (decltype(a.groupEnd))dlsym(lib, "ncclGroupEnd");
      a.allReduce = (decltype(a.allReduce))dlsym(lib, "ncclAllReduce");
      a.errorString = (decltype(a.errorString))dlsym(lib, "ncclGetErrorString");
      a.ok = a.getUniqueId && a.commInitRank && a.commInitAll && a.commDestroy && a.send && a.recv && a.groupStart &&
             a.groupEnd && a.allReduce && a.errorString;
    }
  }
  return a;
}

struct adg_handle {
  adg_config cfg;
  int n = 0, m = 0, NS = 0, NF = 0, REC = 0, K = 0;
  long long cells_global = 0, cells_local = 0;
  int planes_local = 0, plane_cells = 0, plane0 = 0;
  long long slots = 0;
  double h = 0;
  Ops ops;
  bool ops_set = false;
  Dispatch disp;
  double* Q = nullptr;
  double* D = nullptr;
  double* tr[2] = {nullptr, nullptr};
  DevState* st = nullptr;
  StepRecord* recs = nullptr;
  int rec_cap = 4096;
  void* flush = nullptr;
  size_t flush_bytes = 0;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  int sweep_index = 0;       // index of the next regular sweep (0 = priming)
  int disp_ctas_per_sm = 0;  // resident sweep CTAs per SM (adg_step_host chunking)
  bool seeded = false;
  bool loaded = false;
  int host_steps = 0;        // steps whose records were fetched
  DevState hst;              // host mirror after the last sync
  std::string err;
  // subcell limiter (adg_set_limiter; straightforward mode, one slab)
  bool lim = false;
  LimDispatch ldisp;
  int lim_ns = 0;
  double* lim_P = nullptr;
  double* lim_R = nullptr;
  int* lim_nearest = nullptr;
  int* lim_sample = nullptr;
  int* lim_rank = nullptr;
  double* lim_prev[2] = {nullptr, nullptr};
  unsigned char* lim_troubled = nullptr;
  int* lim_list = nullptr;
  double* lim_lam = nullptr;
  double* sm_scratch = nullptr;   // per-SM slots of the p = 9 kernel (previous Picard iterate)
  double* lim_scratch = nullptr;
  long long lim_scratch_cta = 0;
  unsigned lim_grid = 0;
  size_t lim_detect_smem = 0;
  double lim_cfl = 0.9;
  // adg_step_host: copy streams and per-chunk events
  cudaStream_t copy_in = nullptr, copy_out = nullptr;
  // library-owned NCCL communicator of the slab ranks (adg_nccl_init)
  ncclComm_t comm = nullptr;
  int comm_rank = 0, comm_world = 1;
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t comm_ev[2] = {nullptr, nullptr};
  std::vector<cudaEvent_t> chunk_ev;
  StepRecord* rec_host = nullptr;      // pinned landing slot of the step record
  bool hst_fresh = false;              // hst mirrors the device (no phase call since the last pull)
  bool has_next_cond = false;          // adg_run_timed_ex: the finish sets the next rerun node's condition
  unsigned long long next_cond = 0;
  // adg_set_option (explicit, per handle; no environment lookups in the library)
  int opt_graph = 1;                   // ADG_OPT_GRAPH: captured step graphs in adg_run / adg_run_timed*
  int opt_cond_rerun = 1;              // ADG_OPT_COND_RERUN: rerun pass as a conditional graph node
  int opt_fuse_finish = 1;             // ADG_OPT_FUSE_FINISH: time control inside the sweep launch (kernels that have it)
  int opt_persistent = 1;              // ADG_OPT_PERSISTENT: whole step sequences in one cooperative launch
  unsigned* arrive = nullptr;          // [0] CTA arrival counter (fused time control, grid barrier), [1] generation
  bool finish_fused = false;           // the sweep in flight carries the time control of its step
  int opt_host_chunks = 16;            // ADG_OPT_HOST_CHUNKS: wave-aligned chunks of adg_step_host
                                       // (cfg 2: 16 -> 1.526 ms, 9 -> 1.557, 23 -> 1.784)
};

constexpr int ADG_HOST_CHUNKS_MAX = 81;
constexpr int ADG_TIMED_NO_PULL = 1 << 16;   // internal adg_run_timed_ex flag: adg_run's graph chunks

static adg_status fail(adg_handle* h, adg_status code, const std::string& msg) {
  if (h) h->err = msg;
  return code;
}

static adg_status cuda_check(adg_handle* h, cudaError_t e, const char* what) {
  if (e == cudaSuccess) return ADG_OK;
  char buf[512];
  snprintf(buf, sizeof buf, "CUDA error in %s: %s", what, cudaGetErrorString(e));
  return fail(h, ADG_ERR_RUNTIME, buf);
}

#define CUDA_TRY(h, expr)                                   \
  do {                                                      \
    adg_status _s = cuda_check((h), (expr), #expr);         \
    if (_s != ADG_OK) return _s;                            \
  } while (0)

static SweepParams sweep_params(adg_handle* h, int mode) {
  SweepParams P;
  P.ops = h->ops;
  P.Q = h->Q;
  P.D = h->D;
  const int par = h->sweep_index & 1;
  // the sweep (and the rerun before it) read parity `par`; the sweep's own
  // predictions go to the other parity, the rerun pass overwrites `par`.
  if (mode == MODE_RERUN) {
    P.tr_in = h->tr[par];
    P.tr_out = h->tr[par];
  } else {
    P.tr_in = h->tr[par];
    P.tr_out = h->tr[par ^ 1];
  }
  if (mode == MODE_PRIMING) P.tr_out = h->tr[1];
  if (mode == MODE_SF_PREDICT || mode == MODE_SF_CORRECT) {   // straightforward: one record parity
    P.tr_in = h->tr[0];
    P.tr_out = h->tr[0];
  }
  P.st = h->st;
  P.slots = h->slots;
  P.mode = mode;
  P.K = h->K;
  P.planes_local = h->planes_local;
  P.plane_cells = h->plane_cells;
  P.cell_offset = (int)(h->plane0 * (long long)h->plane_cells);
  P.halo = (h->cfg.world > 1 || h->cfg.halo_mode == 1) ? 1 : 0;
  P.cell_a = 0;
  P.blk_split = INT_MAX;
  P.cell_jump = 0;
  P.sweep = h->sweep_index;
  P.outflow = h->cfg.boundary == 1 ? 1 : 0;
  // limiter hooks: the corrector of step s snapshots prev_Q into lim_prev[s & 1]
  P.lim_troubled = h->lim ? h->lim_troubled : nullptr;
  P.lim_cur = h->lim ? h->lim_prev[h->sweep_index & 1] : nullptr;
  P.lim_lam = h->lim ? h->lim_lam : nullptr;
  P.sm_scratch = h->sm_scratch;
  P.spike_step = h->cfg.spike_step;
  P.p = h->cfg.p;
  P.h = h->h;
  P.cfl = h->cfg.cfl;
  P.spike_factor = h->cfg.spike_factor;
  for (int a = 0; a < 3; ++a) P.vel[a] = h->cfg.velocity[a];
  return P;
}

static FinishParams finish_params(adg_handle* h, int priming, int seed) {
  FinishParams F;
  F.st = h->st;
  F.recs = h->recs;
  F.rec_cap = h->rec_cap;
  F.priming = priming;
  F.seed = seed;
  F.d = h->cfg.d;
  F.p = h->cfg.p;
  F.h = h->h;
  F.cfl = h->cfg.cfl;
  F.c_dt = h->cfg.c_dt;
  F.forced_dt = h->cfg.forced_dt;
  F.creeping = h->cfg.creeping;
  F.inject_rerun = h->cfg.inject_rerun;
  F.straightforward = (h->cfg.driver_mode == 1 && !seed) ? 1 : 0;
  F.has_cond = h->has_next_cond ? 1 : 0;
  F.cond = h->next_cond;
  return F;
}

// part: ADG_PART_ALL = every local cell; ADG_PART_INTERIOR = slab planes
// 1..P-2 (read no halo slot, write no record a neighbour needs);
// ADG_PART_BOUNDARY = planes 0 and P-1 (the halo readers / record producers).
static adg_status launch(adg_handle* h, int mode, int part = ADG_PART_ALL) {
  SweepParams P = sweep_params(h, mode);
  const int Pl = h->planes_local, pc = h->plane_cells;
  unsigned blocks = (unsigned)h->cells_local;
  if (part == ADG_PART_INTERIOR) {
    if (Pl <= 2) return ADG_OK;                       // no interior plane
    P.cell_a = pc;
    blocks = (unsigned)((Pl - 2) * (long long)pc);
  } else if (part == ADG_PART_BOUNDARY) {
    if (Pl >= 2) {
      P.blk_split = pc;
      P.cell_jump = (Pl - 2) * pc;                    // block pc -> first cell of plane P-1
      blocks = (unsigned)(2 * pc);
    } else {
      blocks = (unsigned)pc;
    }
  } else if (part != ADG_PART_ALL) {
    return fail(h, ADG_ERR_CONFIG, "unknown sweep part");
  }
  h->disp.sweep(P, blocks, h->stream);
  return cuda_check(h, cudaGetLastError(), "sweep launch");
}

// subcell limiter pass after the straightforward corrector (scheduler.py:282-309):
// detect (one CTA per cell) -> apply (persistent CTAs over the troubled list)
// -> max lambda.  prev_Q of this step is lim_prev[sweep_index & 1].
static adg_status launch_limiter(adg_handle* h) {
  LimParams L;
  L.sp = sweep_params(h, MODE_SF_CORRECT);
  L.P = h->lim_P;
  L.R = h->lim_R;
  L.nearest = h->lim_nearest;
  L.sample = h->lim_sample;
  L.rank = h->lim_rank;
  L.Q = h->Q;
  L.cur = h->lim_prev[h->sweep_index & 1];
  L.old = h->lim_prev[(h->sweep_index & 1) ^ 1];
  L.troubled = h->lim_troubled;
  L.list = h->lim_list;
  L.lam = h->lim_lam;
  L.scratch = h->lim_scratch;
  L.scratch_cta = h->lim_scratch_cta;
  L.st = h->st;
  L.n = h->n;
  L.ns = h->lim_ns;
  L.K = h->K;
  L.n_cells = (int)h->cells_local;
  L.outflow = h->cfg.boundary == 1 ? 1 : 0;
  L.h_sub = h->h / (double)h->lim_ns;          // limiter.py:96  grid.h / ns
  L.cfl = h->lim_cfl;
  h->ldisp.detect(L, (unsigned)h->cells_local, h->lim_detect_smem, h->stream);
  adg_status s = cuda_check(h, cudaGetLastError(), "limiter detect launch");
  if (s != ADG_OK) return s;
  h->ldisp.apply(L, h->lim_grid, h->stream);
  if ((s = cuda_check(h, cudaGetLastError(), "limiter apply launch")) != ADG_OK) return s;
  lim_lambda_kernel<<<148, 256, 0, h->stream>>>(h->lim_lam, (int)h->cells_local, h->st);
  return cuda_check(h, cudaGetLastError(), "limiter lambda launch");
}

static adg_status launch_finish(adg_handle* h, int priming, int seed) {
  FinishParams F = finish_params(h, priming, seed);
  finish_kernel<<<1, 1, 0, h->stream>>>(F);
  return cuda_check(h, cudaGetLastError(), "finish launch");
}

static adg_status pull_state(adg_handle* h) {
  CUDA_TRY(h, cudaMemcpyAsync(&h->hst, h->st, sizeof(DevState), cudaMemcpyDeviceToHost, h->stream));
  CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  h->hst_fresh = true;
  return ADG_OK;
}

static adg_status status_from_state(adg_handle* h) {
  const DevState& s = h->hst;
  char buf[512];
  switch (s.status) {
    case 0: return ADG_OK;
    case ADG_EK_INIT_INADMISSIBLE:
      snprintf(buf, sizeof buf, "initial data inadmissible in cell %lld", s.err_cell);
      return fail(h, ADG_ERR_NUMERICAL, buf);
    case ADG_EK_NO_INITIAL_STEP:
      snprintf(buf, sizeof buf, "no admissible initial step (got %.17g)", s.err_value);
      return fail(h, ADG_ERR_NUMERICAL, buf);
    case ADG_EK_INADMISSIBLE:
      snprintf(buf, sizeof buf, "inadmissible state in cell %lld at step %d", s.err_cell, s.err_step);
      return fail(h, ADG_ERR_NUMERICAL, buf);
    case ADG_EK_PREDICTOR:
      snprintf(buf, sizeof buf, "predictor produced non-finite values (cell %lld)", s.err_cell);
      return fail(h, ADG_ERR_PREDICTOR, buf);
    case ADG_EK_DEGENERATE:
      snprintf(buf, sizeof buf, "admissible step degenerated to %.17g", s.err_value);
      return fail(h, ADG_ERR_NUMERICAL, buf);
    case ADG_EK_SUBCELL:
      snprintf(buf, sizeof buf, "subcell update left cell %lld inadmissible", s.err_cell);
      return fail(h, ADG_ERR_NUMERICAL, buf);
    case ADG_EK_STALE:
      snprintf(buf, sizeof buf, "stale face record read by cell %lld at step %d (debug check)", s.err_cell,
               s.err_step);
      return fail(h, ADG_ERR_RUNTIME, buf);
    case ADG_EK_BOUNDS:
      snprintf(buf, sizeof buf, "cell / record slot out of bounds in cell %lld at step %d (debug check)",
               s.err_cell, s.err_step);
      return fail(h, ADG_ERR_RUNTIME, buf);
  }
  return fail(h, ADG_ERR_RUNTIME, "unknown device status");
}

extern "C" {

adg_status adg_create(const adg_config* cfg, adg_handle** out) {
  if (!cfg || !out) return ADG_ERR_CONFIG;
  *out = nullptr;
  adg_handle* h = new adg_handle();
  h->cfg = *cfg;
  const adg_config& c = *cfg;
  char buf[256];
  if (c.d != 2 && c.d != 3) { snprintf(buf, sizeof buf, "dimension must be 2 or 3, got %d", c.d); h->err = buf; *out = h; return ADG_ERR_CONFIG; }
  if (c.L < 1 || c.L > 4) { snprintf(buf, sizeof buf, "depth L must be in [1, 4], got %d", c.L); h->err = buf; *out = h; return ADG_ERR_CONFIG; }
  if (c.p < 0 || c.p > 9) { snprintf(buf, sizeof buf, "order p must be in [0, 9], got %d", c.p); h->err = buf; *out = h; return ADG_ERR_CONFIG; }
  if (!(c.c_dt > 0.0 && c.c_dt <= 1.0)) { snprintf(buf, sizeof buf, "c_dt must be in (0, 1], got %g", c.c_dt); h->err = buf; *out = h; return ADG_ERR_CONFIG; }
  if (c.driver_mode != 0 && c.driver_mode != 1) { h->err = "driver_mode must be 0 (fused) or 1 (straightforward)"; *out = h; return ADG_ERR_CONFIG; }
  if (c.system != 0 && c.system != 1) { h->err = "system must be 0 (euler) or 1 (advection)"; *out = h; return ADG_ERR_CONFIG; }
  if (c.system == 1 && c.spike_step >= 0) {                      // scheduler.py:170-171
    h->err = "the speed spike is defined for Euler runs"; *out = h; return ADG_ERR_CONFIG;
  }
  if (c.boundary != 0 && c.boundary != 1) { h->err = "boundary must be 0 (periodic) or 1 (outflow)"; *out = h; return ADG_ERR_CONFIG; }
  if (c.boundary == 1 && (c.world > 1 || c.halo_mode != 0)) {
    h->err = "outflow boundaries run on a single slab (world = 1)"; *out = h; return ADG_ERR_CONFIG;
  }
  if (c.boundary == 1 && c.system == 0) {        // ghost faces live in the generic kernel
    if (!dispatch_generic(c.d, c.p, &h->disp)) { h->err = "no generic kernel for this order"; *out = h; return ADG_ERR_CONFIG; }
  } else if (!dispatch_small(c, &h->disp) && !dispatch_for(c.d, c.p, c.system, &h->disp)) {
    snprintf(buf, sizeof buf, "no sm_100a kernel instantiated for d=%d p=%d", c.d, c.p);
    h->err = buf; *out = h; return ADG_ERR_CONFIG;
  }
  h->n = c.p + 1;
  h->m = c.system == 1 ? 1 : c.d + 2;
  h->NS = 1; for (int a = 0; a < c.d; ++a) h->NS *= h->n;
  h->NF = h->NS / h->n;
  h->REC = h->disp.rec;
  h->K = 1; for (int l = 0; l < c.L; ++l) h->K *= 3;
  h->h = pow(3.0, -(double)c.L);   // mesh.py:71  3.0 ** (-L)
  h->plane_cells = 1; for (int a = 1; a < c.d; ++a) h->plane_cells *= h->K;
  h->cells_global = (long long)h->K * h->plane_cells;
  const int world = c.world < 1 ? 1 : c.world;
  h->cfg.world = world;
  if (c.rank < 0 || c.rank >= world || world > h->K) { h->err = "bad rank/world for the slab decomposition"; *out = h; return ADG_ERR_CONFIG; }
  // x-slabs of whole cell planes: the first K % world slabs get one extra plane
  const int base = h->K / world, extra = h->K % world;
  h->planes_local = base + (c.rank < extra ? 1 : 0);
  h->plane0 = c.rank * base + (c.rank < extra ? c.rank : extra);
  h->cells_local = (long long)h->planes_local * h->plane_cells;
  h->slots = (long long)(h->planes_local + 2) * h->plane_cells;
  *out = h;

  CUDA_TRY(h, cudaSetDevice(c.device));
  CUDA_TRY(h, cudaStreamCreateWithFlags(&h->own_stream, cudaStreamNonBlocking));
  h->stream = h->own_stream;
  const size_t state_bytes = sizeof(double) * (size_t)h->cells_local * h->NS * h->m;
  const size_t tr_bytes = sizeof(double) * (size_t)(2 * c.d) * h->slots * h->REC;
  CUDA_TRY(h, cudaMalloc(&h->Q, state_bytes));
  CUDA_TRY(h, cudaMalloc(&h->D, state_bytes));
  CUDA_TRY(h, cudaMalloc(&h->tr[0], tr_bytes));
  CUDA_TRY(h, cudaMalloc(&h->tr[1], tr_bytes));
  CUDA_TRY(h, cudaMalloc(&h->st, sizeof(DevState)));
  if (h->rec_cap & (h->rec_cap - 1)) return fail(h, ADG_ERR_CONFIG, "the step-record ring is a power of two");
  CUDA_TRY(h, cudaMalloc(&h->recs, sizeof(StepRecord) * h->rec_cap));
  CUDA_TRY(h, cudaMalloc(&h->arrive, 2 * sizeof(unsigned)));
  CUDA_TRY(h, cudaMemsetAsync(h->arrive, 0, 2 * sizeof(unsigned), h->stream));
  if (c.d == 3 && c.p == 9 && c.system == 0) {     // sweep_kernel_p9: one slot per %smid value (one CTA per SM)
    unsigned* d_n = nullptr;
    unsigned nsm = 0;
    CUDA_TRY(h, cudaMalloc(&d_n, sizeof(unsigned)));
    nsmid_kernel<<<1, 1, 0, h->stream>>>(d_n);
    CUDA_TRY(h, cudaMemcpyAsync(&nsm, d_n, sizeof(unsigned), cudaMemcpyDeviceToHost, h->stream));
    CUDA_TRY(h, cudaStreamSynchronize(h->stream));
    cudaFree(d_n);
    if (nsm == 0 || nsm > 4096) return fail(h, ADG_ERR_RUNTIME, "cannot size the per-SM scratch slots");
    CUDA_TRY(h, cudaMalloc(&h->sm_scratch, sizeof(double) * (size_t)nsm * ShapeP9::SCRATCH));
  }
#ifdef ADG_P5_TIMING
  if (c.d == 3 && c.p == 5) {                      // tools/p5_timeline.py: 8 stamps per CTA
    CUDA_TRY(h, cudaMalloc(&h->sm_scratch, sizeof(double) * 8 * (size_t)h->cells_local));
    CUDA_TRY(h, cudaMemsetAsync(h->sm_scratch, 0, sizeof(double) * 8 * (size_t)h->cells_local, h->stream));
  }
#endif
#ifdef ADG_2P3_TIMING
  if (c.d == 2 && c.p == 3) {                      // tools/cta_timeline.py: 32 stamps per CTA
    CUDA_TRY(h, cudaMalloc(&h->sm_scratch, sizeof(double) * 32 * (size_t)h->cells_local));
    CUDA_TRY(h, cudaMemsetAsync(h->sm_scratch, 0, sizeof(double) * 32 * (size_t)h->cells_local, h->stream));
  }
#endif
  CUDA_TRY(h, cudaMemsetAsync(h->D, 0, state_bytes, h->stream));        // mesh.py:238-239
  CUDA_TRY(h, cudaMemsetAsync(h->tr[0], 0, tr_bytes, h->stream));
  CUDA_TRY(h, cudaMemsetAsync(h->tr[1], 0, tr_bytes, h->stream));
  DevState s0;
  memset(&s0, 0, sizeof s0);
  s0.dt_adm = INFINITY;                                                // TimeControl.__init__
  CUDA_TRY(h, cudaMemcpyAsync(h->st, &s0, sizeof s0, cudaMemcpyHostToDevice, h->stream));
  if (h->disp.run) {
    // a zero-step launch now: lazy module loading would otherwise bill the cooperative
    // kernel's first use (~0.4 ms) to a step; a device that refuses it uses the step graph
    const cudaError_t we = h->disp.run(sweep_params(h, MODE_NORMAL), finish_params(h, 0, 0), h->arrive, h->tr[0],
                                       h->tr[1], 0, (unsigned)h->cells_local, h->stream);
    if (we != cudaSuccess) {
      cudaGetLastError();
      h->disp.run = nullptr;
    }
  }
  CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  h->hst = s0;
  return ADG_OK;
}

void adg_destroy(adg_handle* h) {
  if (!h) return;
  if (h->Q) cudaFree(h->Q);
  if (h->D) cudaFree(h->D);
  if (h->tr[0]) cudaFree(h->tr[0]);
  if (h->tr[1]) cudaFree(h->tr[1]);
  if (h->st) cudaFree(h->st);
  if (h->recs) cudaFree(h->recs);
  if (h->arrive) cudaFree(h->arrive);
  if (h->sm_scratch) cudaFree(h->sm_scratch);
  if (h->flush) cudaFree(h->flush);
  void* lim_bufs[] = {h->lim_P, h->lim_R, h->lim_nearest, h->lim_sample, h->lim_rank, h->lim_prev[0],
                      h->lim_prev[1], h->lim_troubled, h->lim_list, h->lim_lam, h->lim_scratch};
  for (void* b : lim_bufs)
    if (b) cudaFree(b);
  for (cudaEvent_t e : h->chunk_ev) cudaEventDestroy(e);
  if (h->copy_in) cudaStreamDestroy(h->copy_in);
  if (h->comm) nccl_api().commDestroy(h->comm);
  if (h->comm_stream) cudaStreamDestroy(h->comm_stream);
  for (cudaEvent_t e : h->comm_ev)
    if (e) cudaEventDestroy(e);
  if (h->rec_host) cudaFreeHost(h->rec_host);
  if (h->copy_out) cudaStreamDestroy(h->copy_out);
  if (h->own_stream) cudaStreamDestroy(h->own_stream);
  delete h;
}

adg_status adg_set_operators(adg_handle* h, const double* nodes, const double* weights,
                             const double* diff, const double* integ,
                             const double* left, const double* right) {
  if (!h || !weights || !diff || !integ || !left || !right) return ADG_ERR_CONFIG;
  (void)nodes;
  const int n = h->n;
  memset(&h->ops, 0, sizeof h->ops);
  for (int i = 0; i < n; ++i) {
    h->ops.w[i] = weights[i];
    h->ops.left[i] = left[i];
    h->ops.right[i] = right[i];
    h->ops.lift_lo[i] = left[i] / weights[i];     // kernels.py:58
    h->ops.lift_hi[i] = right[i] / weights[i];    // kernels.py:59
    for (int j = 0; j < n; ++j) {
      h->ops.diff[i][j] = diff[i * n + j];
      h->ops.integ[i][j] = integ[i * n + j];
      // kvol[i, j] = diff[j, i] * w[j] / w[i]     kernels.py:56
      h->ops.kvol[i][j] = (diff[j * n + i] * weights[j]) / weights[i];
    }
  }
  if (n % 2 == 0) {
    // even / odd blocks of diff (exact for a centro-antisymmetric matrix,
    // diff[n-1-i][n-1-j] = -diff[i][j]; the reference's operators satisfy it to
    // rounding): averaged over the two mirror rows
    const int hn = n / 2;
    for (int i = 0; i < hn; ++i)
      for (int j = 0; j < hn; ++j) {
        const double a = diff[i * n + j], b = diff[i * n + (n - 1 - j)];
        const double am = -diff[(n - 1 - i) * n + (n - 1 - j)], bm = -diff[(n - 1 - i) * n + j];
        h->ops.eo_e[i][j] = 0.25 * ((a + b) + (am + bm));
        h->ops.eo_o[i][j] = 0.25 * ((a - b) + (am - bm));
      }
  }
  h->ops_set = true;
  return ADG_OK;
}

adg_status adg_set_stream(adg_handle* h, void* s) {
  if (!h) return ADG_ERR_CONFIG;
  h->stream = (cudaStream_t)s;
  return ADG_OK;
}

adg_status adg_reset(adg_handle* h) {
  if (!h) return ADG_ERR_CONFIG;
  CUDA_TRY(h, cudaSetDevice(h->cfg.device));
  const size_t state_bytes = sizeof(double) * (size_t)h->cells_local * h->NS * h->m;
  const size_t tr_bytes = sizeof(double) * (size_t)(2 * h->cfg.d) * h->slots * h->REC;
  CUDA_TRY(h, cudaMemsetAsync(h->D, 0, state_bytes, h->stream));
  CUDA_TRY(h, cudaMemsetAsync(h->tr[0], 0, tr_bytes, h->stream));
  CUDA_TRY(h, cudaMemsetAsync(h->tr[1], 0, tr_bytes, h->stream));
  if (h->lim) {
    CUDA_TRY(h, cudaMemsetAsync(h->lim_prev[0], 0, state_bytes, h->stream));   // mesh.py:90-96
    CUDA_TRY(h, cudaMemsetAsync(h->lim_prev[1], 0, state_bytes, h->stream));
    CUDA_TRY(h, cudaMemsetAsync(h->lim_troubled, 0, (size_t)h->cells_local, h->stream));
  }
  DevState s0;
  memset(&s0, 0, sizeof s0);
  s0.dt_adm = INFINITY;
  CUDA_TRY(h, cudaMemcpyAsync(h->st, &s0, sizeof s0, cudaMemcpyHostToDevice, h->stream));
  CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  h->hst = s0;
  h->sweep_index = 0;
  h->seeded = false;
  h->finish_fused = false;
  CUDA_TRY(h, cudaMemsetAsync(h->arrive, 0, 2 * sizeof(unsigned), h->stream));
  h->err.clear();
  return ADG_OK;
}

adg_status adg_load_state(adg_handle* h, const double* Q, size_t n) {
  if (!h || !Q) return ADG_ERR_CONFIG;
  const size_t want = (size_t)h->cells_local * h->NS * h->m;
  if (n != want) return fail(h, ADG_ERR_CONFIG, "state size mismatch");
  CUDA_TRY(h, cudaSetDevice(h->cfg.device));
  CUDA_TRY(h, cudaMemcpyAsync(h->Q, Q, n * sizeof(double), cudaMemcpyHostToDevice, h->stream));
  CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  h->loaded = true;
  return ADG_OK;
}

adg_status adg_store_state(adg_handle* h, double* Q, size_t n) {
  if (!h || !Q) return ADG_ERR_CONFIG;
  const size_t want = (size_t)h->cells_local * h->NS * h->m;
  if (n != want) return fail(h, ADG_ERR_CONFIG, "state size mismatch");
  CUDA_TRY(h, cudaSetDevice(h->cfg.device));
  CUDA_TRY(h, cudaMemcpyAsync(Q, h->Q, n * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
  CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  return ADG_OK;
}

adg_status adg_phase_seed(adg_handle* h) {
  if (!h) return ADG_ERR_CONFIG;
  h->hst_fresh = false;
  if (!h->ops_set) return fail(h, ADG_ERR_CONFIG, "operators not set");
  if (!h->loaded) return fail(h, ADG_ERR_CONFIG, "state not loaded");
  CUDA_TRY(h, cudaSetDevice(h->cfg.device));
  return launch(h, MODE_SEED);
}

adg_status adg_phase_seed_finish(adg_handle* h) {
  if (!h) return ADG_ERR_CONFIG;
  adg_status s = launch_finish(h, 0, 1);
  if (s == ADG_OK) h->seeded = true;
  return s;
}

adg_status adg_seed(adg_handle* h) {
  adg_status s = adg_phase_seed(h);
  if (s != ADG_OK) return s;
  s = adg_phase_seed_finish(h);
  if (s != ADG_OK) return s;
  s = pull_state(h);
  if (s != ADG_OK) return s;
  return status_from_state(h);
}

static bool straightforward(const adg_handle* h) { return h->cfg.driver_mode == 1; }

adg_status adg_phase_rerun(adg_handle* h) {
  if (!h) return ADG_ERR_CONFIG;
  h->hst_fresh = false;
  if (straightforward(h)) {                     // the prediction sweep of the step
    if (!h->seeded) return fail(h, ADG_ERR_CONFIG, "time control not seeded");
    return launch(h, MODE_SF_PREDICT);
  }
  if (h->sweep_index == 0) return ADG_OK;       // nothing predicted yet
  return launch(h, MODE_RERUN);
}

adg_status adg_phase_sweep_part(adg_handle* h, int part) {
  if (!h) return ADG_ERR_CONFIG;
  h->hst_fresh = false;
  if (!h->seeded) return fail(h, ADG_ERR_CONFIG, "time control not seeded");
  if (straightforward(h)) {
    adg_status s = launch(h, MODE_SF_CORRECT, part);
    if (s != ADG_OK || !h->lim) return s;
    return launch_limiter(h);
  }
  if (h->sweep_index == 0 && part != ADG_PART_ALL)
    return fail(h, ADG_ERR_CONFIG, "the priming sweep is not split");
  const int mode = h->sweep_index == 0 ? MODE_PRIMING : MODE_NORMAL;
  // one slab, whole sweep: the kernel's last CTA is the step's time control (adg_phase_finish
  // then only advances the sweep index)
  if (part == ADG_PART_ALL && h->disp.sweep_finish && h->opt_fuse_finish && h->cfg.world == 1 &&
      h->cfg.halo_mode == 0 && !h->lim) {
    const SweepParams P = sweep_params(h, mode);
    h->disp.sweep_finish(P, finish_params(h, h->sweep_index == 0 ? 1 : 0, 0), h->arrive, (unsigned)h->cells_local,
                         h->stream);
    h->finish_fused = true;
    return cuda_check(h, cudaGetLastError(), "sweep launch");
  }
  return launch(h, mode, part);
}

adg_status adg_phase_sweep(adg_handle* h) { return adg_phase_sweep_part(h, ADG_PART_ALL); }

adg_status adg_phase_finish(adg_handle* h) {
  if (!h) return ADG_ERR_CONFIG;
  h->hst_fresh = false;
  adg_status s = ADG_OK;
  if (h->finish_fused) h->finish_fused = false;    // done by the sweep launch
  else s = launch_finish(h, (!straightforward(h) && h->sweep_index == 0) ? 1 : 0, 0);
  h->sweep_index += 1;
  return s;
}

int adg_trace_parity(const adg_handle* h) {
  if (!h) return 0;
  return straightforward(h) ? 0 : (h->sweep_index & 1);   // SF passes share parity 0
}

static adg_status enqueue_step(adg_handle* h) {
  adg_status s;
  if (!straightforward(h) && h->sweep_index == 0) {   // Driver.step: priming sweep first
    if ((s = adg_phase_sweep(h)) != ADG_OK) return s;
    if ((s = adg_phase_finish(h)) != ADG_OK) return s;
  }
  if ((s = adg_phase_rerun(h)) != ADG_OK) return s;
  if ((s = adg_phase_sweep(h)) != ADG_OK) return s;
  return adg_phase_finish(h);
}

static adg_status fetch_records(adg_handle* h, int from_step, int to_step, adg_step_record* out) {
  // records of steps (from_step, to_step] into out[0..]
  for (int s = from_step + 1; s <= to_step; ++s) {
    StepRecord r;
    CUDA_TRY(h, cudaMemcpyAsync(&r, h->recs + ((s - 1) % h->rec_cap), sizeof r,
                                cudaMemcpyDeviceToHost, h->stream));
    CUDA_TRY(h, cudaStreamSynchronize(h->stream));
    adg_step_record& o = out[s - from_step - 1];
    o.step = r.step; o.reruns = r.reruns; o.T = r.T; o.dt_old = r.dt_old;
    o.dt_new = r.dt_new; o.dt_adm = r.dt_adm; o.picard_iters = r.picard_iters; o.predicts = r.predicts;
    o.troubled = r.troubled;
  }
  return ADG_OK;
}

adg_status adg_step(adg_handle* h, adg_step_record* out) {
  if (!h) return ADG_ERR_CONFIG;
  if (h->hst.status) return status_from_state(h);
  CUDA_TRY(h, cudaSetDevice(h->cfg.device));
  const int before = h->hst.step;
  adg_status s = enqueue_step(h);
  if (s != ADG_OK) return s;
  if ((s = pull_state(h)) != ADG_OK) return s;
  if ((s = status_from_state(h)) != ADG_OK) return s;
  if (out && h->hst.step > before) return fetch_records(h, before, h->hst.step, out);
  return ADG_OK;
}

adg_status adg_run(adg_handle* h, int steps, adg_step_record* out) {
  if (!h) return ADG_ERR_CONFIG;
  if (h->hst.status) return status_from_state(h);
  CUDA_TRY(h, cudaSetDevice(h->cfg.device));
  int done = 0;
  while (done < steps) {
    const int chunk = (steps - done) < h->rec_cap ? (steps - done) : h->rec_cap;
    const int before = h->hst.step;
    int i = 0;
    if (!straightforward(h) && h->sweep_index == 0) {   // priming sweep + first step on the stream
      adg_status s = enqueue_step(h);
      if (s != ADG_OK) return s;
      i = 1;
    }
    // single GPU, fused driver, no limiter: the remaining steps as one CUDA graph with the
    // rerun pass as a conditional node (adg_run_timed_ex; bitwise the stream launches,
    // tests/test_gpu_parity.py::test_run_timed_graph_equals_device_run).  ADG_OPT_GRAPH 0:
    // stream launches.
    const bool graph = !straightforward(h) && h->cfg.world == 1 && h->cfg.halo_mode == 0 && !h->lim &&
                       chunk - i >= 2 && h->opt_graph;
    if (graph) {
      double tout[2];
      adg_status s = adg_run_timed_ex(h, chunk - i, ADG_TIMED_NO_PULL, tout);
      if (s != ADG_OK) return s;
    } else {
      for (; i < chunk; ++i) {
        adg_status s = enqueue_step(h);
        if (s != ADG_OK) return s;
      }
    }
    adg_status s = pull_state(h);
    if (s != ADG_OK) return s;
    if (out && h->hst.step > before) {
      s = fetch_records(h, before, h->hst.step, out + done);
      if (s != ADG_OK) return s;
    }
    if ((s = status_from_state(h)) != ADG_OK) return s;
    done += chunk;
  }
  return ADG_OK;
}

adg_status adg_step_records(adg_handle* h, int first, int count, adg_step_record* out) {
  if (!h || !out || first < 1 || count < 0) return ADG_ERR_CONFIG;
  if (first + count - 1 > h->hst.step || h->hst.step - first >= h->rec_cap)
    return fail(h, ADG_ERR_CONFIG, "requested step records are not available");
  return fetch_records(h, first - 1, first - 1 + count, out);
}

namespace {
__global__ void set_dt_new_kernel(DevState* st, double v, double h) {
  st->dt_new = v;
  st->scale_new = __ddiv_rn(v, h);
}
}  // namespace

adg_status adg_set_dt_new(adg_handle* h, double value) {
  if (!h) return ADG_ERR_CONFIG;
  CUDA_TRY(h, cudaSetDevice(h->cfg.device));
  set_dt_new_kernel<<<1, 1, 0, h->stream>>>(h->st, value, h->h);
  CUDA_TRY(h, cudaGetLastError());
  return pull_state(h);
}

adg_status adg_sync(adg_handle* h) {
  if (!h) return ADG_ERR_CONFIG;
  adg_status s = pull_state(h);
  if (s != ADG_OK) return s;
  return status_from_state(h);
}

int adg_step_count(const adg_handle* h) { return h ? h->hst.step : 0; }
int adg_rerun_count(const adg_handle* h) {
  // reruns already executed (a rerun decided for the coming step is not booked yet)
  return h ? h->hst.reruns_total - h->hst.rerun_next : 0;
}
int adg_sweep_count(const adg_handle* h) {
  // priming + one regular sweep per step + rerun passes (Driver.sweep_count);
  // straightforward: three sweeps per step (scheduler.py:236,255,267)
  if (!h || h->hst.step == 0) return 0;
  if (h->cfg.driver_mode == 1) return 3 * h->hst.step;
  return 1 + h->hst.step + h->hst.reruns_total - (h->hst.rerun_next ? 1 : 0);
}

adg_status adg_time_control(const adg_handle* h, double* T, double* dt_old, double* dt_new, double* dt_adm) {
  if (!h) return ADG_ERR_CONFIG;
  if (T) *T = h->hst.T;
  if (dt_old) *dt_old = h->hst.dt_old;
  if (dt_new) *dt_new = h->hst.dt_new;
  if (dt_adm) *dt_adm = h->hst.dt_adm;
  return ADG_OK;
}

adg_status adg_picard_histogram(const adg_handle* h, long long* hist, int n_bins) {
  if (!h || !hist) return ADG_ERR_CONFIG;
  for (int i = 0; i < n_bins && i < HIST_BINS; ++i) hist[i] = h->hst.hist[i];
  return ADG_OK;
}

adg_status adg_error_info(const adg_handle* h, int* kind, long long* cell, int* step, double* value) {
  if (!h) return ADG_ERR_CONFIG;
  if (kind) *kind = h->hst.status;
  if (cell) *cell = h->hst.err_cell;
  if (step) *step = h->hst.err_step;
  if (value) *value = h->hst.err_value;
  return ADG_OK;
}

const char* adg_last_error(const adg_handle* h) { return h ? h->err.c_str() : "null handle"; }

adg_status adg_set_limiter(adg_handle* h, const double* P, const double* R, const int* nearest,
                           const int* sample, const long long* traversal, double cfl) {
  if (!h || !P || !R || !nearest || !sample) return ADG_ERR_CONFIG;
  if (h->cfg.driver_mode != 1)                     // scheduler.py:100-102
    return fail(h, ADG_ERR_CONFIG, "subcell limiting is supported in straightforward mode only");
  if (h->cfg.world != 1 || h->cfg.halo_mode != 0)
    return fail(h, ADG_ERR_CONFIG, "the subcell limiter runs on a single slab (world = 1)");
  if (h->lim) return fail(h, ADG_ERR_CONFIG, "limiter already attached");
  if (h->sweep_index != 0) return fail(h, ADG_ERR_CONFIG, "attach the limiter before the first step");
  CUDA_TRY(h, cudaSetDevice(h->cfg.device));
  const int d = h->cfg.d, n = h->n, m = h->m, ns = 2 * h->cfg.p + 1;
  long long nsub = 1;
  for (int a = 0; a < d; ++a) nsub *= ns;
  const long long nlay = nsub / ns;
  if (h->cfg.system == 0 && !dispatch_generic(d, h->cfg.p, &h->disp))
    return fail(h, ADG_ERR_CONFIG, "no generic kernel for this order");
  h->ldisp = lim_dispatch_for(d, h->cfg.system);
  h->lim_ns = ns;
  h->lim_cfl = cfl;
  const long long cells = h->cells_local;
  const size_t state_bytes = sizeof(double) * (size_t)cells * h->NS * m;
  CUDA_TRY(h, cudaMalloc(&h->lim_P, sizeof(double) * ns * n));
  CUDA_TRY(h, cudaMalloc(&h->lim_R, sizeof(double) * n * ns));
  CUDA_TRY(h, cudaMalloc(&h->lim_nearest, sizeof(int) * ns));
  CUDA_TRY(h, cudaMalloc(&h->lim_sample, sizeof(int) * n));
  CUDA_TRY(h, cudaMalloc(&h->lim_rank, sizeof(int) * cells));
  CUDA_TRY(h, cudaMalloc(&h->lim_prev[0], state_bytes));
  CUDA_TRY(h, cudaMalloc(&h->lim_prev[1], state_bytes));
  CUDA_TRY(h, cudaMalloc(&h->lim_troubled, (size_t)cells));
  CUDA_TRY(h, cudaMalloc(&h->lim_list, sizeof(int) * cells));
  CUDA_TRY(h, cudaMalloc(&h->lim_lam, sizeof(double) * cells));
  // apply scratch: 5 patches + the frozen halo per CTA; up to 2 CTAs per SM
  h->lim_scratch_cta = LIM_SCRATCH_PATCHES * nsub * m + 2LL * d * nlay * m;
  h->lim_grid = (unsigned)(cells < 296 ? cells : 296);
  CUDA_TRY(h, cudaMalloc(&h->lim_scratch, sizeof(double) * (size_t)h->lim_scratch_cta * h->lim_grid));
  // detection shared memory (aderdg_limiter.cuh lim_detect_kernel)
  long long szA = ns, szB = (d == 3) ? (long long)ns * ns * n : (long long)n * n;
  for (int a = 1; a < d; ++a) szA *= n;
  szA *= m;
  szB *= m;
  const long long NM = (long long)h->NS * m;
  h->lim_detect_smem = sizeof(double) * (size_t)(szA + (NM > szB ? NM : szB) + 2 * m * 8 + 4 * m);
  if (h->lim_detect_smem > 227 * 1024) return fail(h, ADG_ERR_CONFIG, "limiter detection does not fit shared memory");
  std::vector<int> rank(cells);
  if (traversal) {
    std::vector<char> seen(cells, 0);
    for (long long i = 0; i < cells; ++i) {
      const long long c = traversal[i];
      if (c < 0 || c >= cells || seen[c]) return fail(h, ADG_ERR_CONFIG, "traversal must be a permutation of the cells");
      seen[c] = 1;
      rank[c] = (int)i;
    }
  } else {
    for (long long i = 0; i < cells; ++i) rank[i] = (int)i;     // lexicographic (mesh.py:279-282)
  }
  CUDA_TRY(h, cudaMemcpyAsync(h->lim_P, P, sizeof(double) * ns * n, cudaMemcpyHostToDevice, h->stream));
  CUDA_TRY(h, cudaMemcpyAsync(h->lim_R, R, sizeof(double) * n * ns, cudaMemcpyHostToDevice, h->stream));
  CUDA_TRY(h, cudaMemcpyAsync(h->lim_nearest, nearest, sizeof(int) * ns, cudaMemcpyHostToDevice, h->stream));
  CUDA_TRY(h, cudaMemcpyAsync(h->lim_sample, sample, sizeof(int) * n, cudaMemcpyHostToDevice, h->stream));
  CUDA_TRY(h, cudaMemcpyAsync(h->lim_rank, rank.data(), sizeof(int) * cells, cudaMemcpyHostToDevice, h->stream));
  CUDA_TRY(h, cudaMemsetAsync(h->lim_prev[0], 0, state_bytes, h->stream));     // mesh.py:90-96
  CUDA_TRY(h, cudaMemsetAsync(h->lim_prev[1], 0, state_bytes, h->stream));
  CUDA_TRY(h, cudaMemsetAsync(h->lim_troubled, 0, (size_t)cells, h->stream));
  CUDA_TRY(h, cudaMemsetAsync(h->lim_lam, 0, sizeof(double) * cells, h->stream));
  CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  h->lim = true;
  return ADG_OK;
}

adg_status adg_troubled_flags(adg_handle* h, unsigned char* out, size_t n) {
  if (!h || !out) return ADG_ERR_CONFIG;
  if (n != (size_t)h->cells_local) return fail(h, ADG_ERR_CONFIG, "troubled flag count mismatch");
  CUDA_TRY(h, cudaSetDevice(h->cfg.device));
  if (!h->lim) {
    memset(out, 0, n);
    return ADG_OK;
  }
  CUDA_TRY(h, cudaMemcpyAsync(out, h->lim_troubled, n, cudaMemcpyDeviceToHost, h->stream));
  CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  return ADG_OK;
}

adg_status adg_layout_info(const adg_handle* h, adg_layout* o) {
  if (!h || !o) return ADG_ERR_CONFIG;
  o->n_cells_global = (int)h->cells_global;
  o->n_cells_local = (int)h->cells_local;
  o->cell_offset = (int)(h->plane0 * (long long)h->plane_cells);
  o->planes_local = h->planes_local;
  o->plane_cells = h->plane_cells;
  o->record_doubles = h->REC;
  o->faces_per_cell = 2 * h->cfg.d;
  o->state_doubles = (size_t)h->cells_local * h->NS * h->m;
  return ADG_OK;
}

adg_status adg_buffer(adg_handle* h, int which, void** ptr, size_t* bytes) {
  if (!h || !ptr || !bytes) return ADG_ERR_CONFIG;
  const size_t state_bytes = sizeof(double) * (size_t)h->cells_local * h->NS * h->m;
  const size_t tr_bytes = sizeof(double) * (size_t)(2 * h->cfg.d) * h->slots * h->REC;
  switch (which) {
    case ADG_BUF_Q: *ptr = h->Q; *bytes = state_bytes; return ADG_OK;
    case ADG_BUF_D: *ptr = h->D; *bytes = state_bytes; return ADG_OK;
    case ADG_BUF_TRACE0: *ptr = h->tr[0]; *bytes = tr_bytes; return ADG_OK;
    case ADG_BUF_TRACE1: *ptr = h->tr[1]; *bytes = tr_bytes; return ADG_OK;
    case ADG_BUF_REDUCE: *ptr = h->st; *bytes = 2 * sizeof(long long); return ADG_OK;
#ifdef ADG_P5_TIMING
    case 98: *ptr = h->sm_scratch; *bytes = sizeof(double) * 8 * (size_t)h->cells_local; return ADG_OK;
#endif
#ifdef ADG_2P3_TIMING
    case 99: *ptr = h->sm_scratch; *bytes = sizeof(double) * 32 * (size_t)h->cells_local; return ADG_OK;
#endif
  }
  return ADG_ERR_CONFIG;
}

// The rerun pass of one step as an IF node of the capture on h->stream (condition
// handle hc, set by the previous step's finish kernel); the pass itself is captured
// into the node's body through `side`.
static adg_status capture_rerun_if(adg_handle* h, cudaGraphConditionalHandle hc, cudaStream_t side) {
  cudaStreamCaptureStatus cs;
  cudaGraph_t cg = nullptr;
  const cudaGraphNode_t* deps = nullptr;
  size_t nd = 0;
  CUDA_TRY(h, cudaStreamGetCaptureInfo(h->stream, &cs, nullptr, &cg, &deps, &nd));
  cudaGraphNodeParams np = {};
  np.type = cudaGraphNodeTypeConditional;
  np.conditional.handle = hc;
  np.conditional.type = cudaGraphCondTypeIf;
  np.conditional.size = 1;
  cudaGraphNode_t cn;
  CUDA_TRY(h, cudaGraphAddNode(&cn, cg, deps, nd, &np));
  CUDA_TRY(h, cudaStreamUpdateCaptureDependencies(h->stream, &cn, 1, cudaStreamSetCaptureDependencies));
  CUDA_TRY(h, cudaStreamBeginCaptureToGraph(side, np.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                            cudaStreamCaptureModeRelaxed));
  cudaStream_t keep = h->stream;
  h->stream = side;
  adg_status r = adg_phase_rerun(h);
  h->stream = keep;
  cudaGraph_t body = nullptr;
  CUDA_TRY(h, cudaStreamEndCapture(side, &body));
  return r;
}

adg_status adg_run_timed(adg_handle* h, int steps, double* out) {
  return adg_run_timed_ex(h, steps, ADG_TIMED_KERNEL_EVENTS, out);
}

static adg_status enqueue_halo(adg_handle* h, int par);

// `steps` realisation steps (rerun pass -> sweep -> [all-reduce] -> time control)
// enqueued back to back on h->stream.  By default they are captured into one CUDA
// graph and launched once (graph-node gaps instead of launch gaps), the rerun pass of
// every step an IF node whose condition the previous step's finish kernel sets (no
// rerun launch at all on the common no-rerun step: cfg 2 0.564 -> 0.555 ms/step).
// The launches, and the host-side counters they advance, are exactly those of the
// stream path (ADG_OPT_GRAPH 0).  mgpu: the handle's NCCL communicator exchanges the
// boundary records on the comm stream (forked from and joined to the capture through
// comm_ev) while the interior planes run, and all-reduces the step reduction.
// Events: ev[0] / ev[1] bracket the segment; with ADG_TIMED_KERNEL_EVENTS also every
// rerun / sweep launch (graph nodes that cost gaps: cfg 1 26.6 -> 35.4 us/step, so the
// throughput run leaves them out and an instrumented replay measures the kernels).
// `steps` fused steps of a primed single-slab driver in one cooperative launch
// (Dispatch::run).  *launched = false (and ADG_OK) when the device refuses the cooperative
// launch: the caller falls back to the step graph.
static adg_status run_persistent(adg_handle* h, int steps, int flags, double* out, bool* launched) {
  *launched = false;
  cudaEvent_t ev[2] = {nullptr, nullptr};
  CUDA_TRY(h, cudaEventCreate(&ev[0]));
  if (cudaEventCreate(&ev[1]) != cudaSuccess) {
    cudaEventDestroy(ev[0]);
    return fail(h, ADG_ERR_RUNTIME, "cudaEventCreate failed");
  }
  h->hst_fresh = false;
  h->has_next_cond = false;
  const SweepParams P = sweep_params(h, MODE_NORMAL);
  const FinishParams F = finish_params(h, 0, 0);
  cudaEventRecord(ev[0], h->stream);
  const cudaError_t le = h->disp.run(P, F, h->arrive, h->tr[0], h->tr[1], steps, (unsigned)h->cells_local, h->stream);
  if (le != cudaSuccess) {
    cudaGetLastError();                     // not sticky: nothing was enqueued
    cudaEventDestroy(ev[0]);
    cudaEventDestroy(ev[1]);
    return ADG_OK;
  }
  *launched = true;
  h->sweep_index += steps;
  cudaEventRecord(ev[1], h->stream);
  adg_status t = cuda_check(h, cudaEventSynchronize(ev[1]), "cudaEventSynchronize");
  float ms = 0.f;
  if (t == ADG_OK) t = cuda_check(h, cudaEventElapsedTime(&ms, ev[0], ev[1]), "cudaEventElapsedTime");
  out[0] = ms;
  out[1] = 0.0;
  cudaEventDestroy(ev[0]);
  cudaEventDestroy(ev[1]);
  if (t != ADG_OK) return t;
  if (flags & ADG_TIMED_NO_PULL) return ADG_OK;
  if ((t = pull_state(h)) != ADG_OK) return t;
  return status_from_state(h);
}

static adg_status run_steps(adg_handle* h, int steps, int flags, double* out, bool mgpu) {
  if (!h || !out || steps < 1) return ADG_ERR_CONFIG;
  if (mgpu && !h->comm) return fail(h, ADG_ERR_CONFIG, "adg_run_timed_mgpu needs adg_nccl_init");
  if (h->hst.status) return status_from_state(h);
  CUDA_TRY(h, cudaSetDevice(h->cfg.device));
  if (!straightforward(h) && h->sweep_index == 0)
    return fail(h, ADG_ERR_CONFIG, "adg_run_timed needs a primed driver (run one step first)");
  const bool exchange = mgpu && (h->comm_world > 1 || h->cfg.halo_mode == 1);
  const bool step_ev = (flags & ADG_TIMED_KERNEL_EVENTS) != 0;
  if (!mgpu && !step_ev && h->disp.run && h->opt_graph && h->opt_persistent && !straightforward(h) &&
      h->cfg.world == 1 && h->cfg.halo_mode == 0 && !h->lim) {
    // kernels that have it: the steps as ONE cooperative launch (no graph, no per-step launches)
    bool launched = false;
    const adg_status ps = run_persistent(h, steps, flags, out, &launched);
    if (launched || ps != ADG_OK) return ps;
  }
  std::vector<cudaEvent_t> ev(step_ev ? 4 * (size_t)steps + 2 : 2, nullptr);
  auto destroy_events = [&] {
    for (cudaEvent_t e : ev)
      if (e) cudaEventDestroy(e);
  };
  for (auto& e : ev) {
    const cudaError_t ce = cudaEventCreate(&e);
    if (ce != cudaSuccess) {
      destroy_events();
      return cuda_check(h, ce, "cudaEventCreate");
    }
  }
  const cudaStream_t run = h->stream;
  cudaStream_t cap = nullptr, side = nullptr;
  bool graph = h->opt_graph && cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking) == cudaSuccess;
  if (graph)
    graph = cudaStreamBeginCapture(cap, mgpu ? cudaStreamCaptureModeRelaxed : cudaStreamCaptureModeThreadLocal) ==
            cudaSuccess;
  if (!graph && cap) {
    cudaStreamDestroy(cap);
    cap = nullptr;
  }
  if (graph) h->stream = cap;
  // in a capture, timing events become event-record nodes only with the external flag
  const unsigned rec_flags = graph ? cudaEventRecordExternal : cudaEventRecordDefault;
  auto record0 = [&](cudaEvent_t e) { return cudaEventRecordWithFlags(e, h->stream, rec_flags); };
  auto record = [&](size_t i) { return step_ev ? record0(ev[i]) : cudaSuccess; };
  bool cond = graph && !straightforward(h) && h->opt_cond_rerun;
  std::vector<cudaGraphConditionalHandle> hc;
  // everything that can fail runs inside the capture, so the capture always ends
  // below and h->stream is restored whatever happens
  auto enqueue = [&]() -> adg_status {
    if (cond) {
      cudaStreamCaptureStatus cs;
      cudaGraph_t cg = nullptr;
      bool ok = cudaStreamGetCaptureInfo(cap, &cs, nullptr, &cg, nullptr, nullptr) == cudaSuccess &&
                cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking) == cudaSuccess;
      hc.resize(steps);
      // default 1: the first step's pass checks rerun_next itself
      for (int i = 0; i < steps && ok; ++i)
        ok = cudaGraphConditionalHandleCreate(&hc[i], cg, 1, cudaGraphCondAssignDefault) == cudaSuccess;
      if (!ok) {                 // no conditional nodes on this driver: plain rerun launches
        cudaGetLastError();
        cond = false;
      }
    }
    CUDA_TRY(h, record0(ev[0]));
    adg_status r = ADG_OK;
    for (int i = 0; i < steps && r == ADG_OK; ++i) {
      CUDA_TRY(h, record(2 + 4 * (size_t)i));
      r = cond ? capture_rerun_if(h, hc[i], side) : adg_phase_rerun(h);
      CUDA_TRY(h, record(3 + 4 * (size_t)i));
      if (r != ADG_OK) break;
      CUDA_TRY(h, record(4 + 4 * (size_t)i));
      // the time control of this step (finish_kernel, or the sweep's last CTA) sets the
      // condition of the next step's rerun node
      h->has_next_cond = cond && i + 1 < steps;
      if (h->has_next_cond) h->next_cond = hc[i + 1];
      if (exchange) {
        r = enqueue_halo(h, adg_trace_parity(h));
        if (r == ADG_OK) r = adg_phase_sweep_part(h, ADG_PART_INTERIOR);
        if (r == ADG_OK) {
          CUDA_TRY(h, cudaStreamWaitEvent(h->stream, h->comm_ev[1], 0));
          r = adg_phase_sweep_part(h, ADG_PART_BOUNDARY);
        }
      } else {
        r = adg_phase_sweep(h);
      }
      CUDA_TRY(h, record(5 + 4 * (size_t)i));
      if (r != ADG_OK) break;
      if (mgpu && h->comm_world > 1) {
        const ncclResult_t nr = nccl_api().allReduce(h->st, h->st, 2, ncclInt64, ncclMax, h->comm, h->stream);
        if (nr != ncclSuccess) return fail(h, ADG_ERR_RUNTIME, nccl_api().errorString(nr));
      }
      r = adg_phase_finish(h);
      h->has_next_cond = false;
    }
    CUDA_TRY(h, record0(ev[1]));
    return r;
  };
  adg_status s = enqueue();
  h->has_next_cond = false;
  h->stream = run;
  if (graph) {
    cudaGraph_t g = nullptr;
    cudaGraphExec_t ge = nullptr;
    const cudaError_t e1 = cudaStreamEndCapture(cap, &g);
    cudaError_t e2 = cudaErrorUnknown;
    if (e1 == cudaSuccess && s == ADG_OK) {
      e2 = cudaGraphInstantiate(&ge, g, 0);
      if (e2 == cudaSuccess) e2 = cudaGraphLaunch(ge, run);
    }
    if (ge) cudaGraphExecDestroy(ge);   // safe: the launch keeps its own reference
    if (g) cudaGraphDestroy(g);
    cudaStreamDestroy(cap);
    if (s == ADG_OK && (e1 != cudaSuccess || e2 != cudaSuccess))
      s = fail(h, ADG_ERR_RUNTIME, std::string("adg_run_timed graph: ") +
                                       cudaGetErrorString(e1 != cudaSuccess ? e1 : e2));
  }
  if (side) cudaStreamDestroy(side);
  if (s != ADG_OK) {
    cudaStreamSynchronize(run);
    destroy_events();
    return s;
  }
  adg_status t = cuda_check(h, cudaEventSynchronize(ev[1]), "cudaEventSynchronize");
  float ms = 0.f;
  if (t == ADG_OK) t = cuda_check(h, cudaEventElapsedTime(&ms, ev[0], ev[1]), "cudaEventElapsedTime");
  out[0] = ms;
  double kern = 0.0;
  for (int i = 0; i < steps && step_ev && t == ADG_OK; ++i) {
    float a = 0.f, b = 0.f;
    cudaEventElapsedTime(&a, ev[2 + 4 * (size_t)i], ev[3 + 4 * (size_t)i]);
    cudaEventElapsedTime(&b, ev[4 + 4 * (size_t)i], ev[5 + 4 * (size_t)i]);
    kern += a + b;
  }
  out[1] = kern;
  destroy_events();
  if (t != ADG_OK) return t;
  if (flags & ADG_TIMED_NO_PULL) return ADG_OK;     // adg_run pulls state and records itself
  if ((t = pull_state(h)) != ADG_OK) return t;
  return status_from_state(h);
}

adg_status adg_run_timed_ex(adg_handle* h, int steps, int flags, double* out) {
  return run_steps(h, steps, flags, out, false);
}

// ---------------------------------------------------------------------------
// Multi-GPU slab steps enqueued from C with the library's own NCCL communicator.
#define NCCL_TRY(h, call)                                                           \
  do {                                                                              \
    ncclResult_t r_ = (call);                                                       \
    if (r_ != ncclSuccess) return fail(h, ADG_ERR_RUNTIME, nccl_api().errorString(r_)); \
  } while (0)

adg_status adg_nccl_unique_id(unsigned char* out128) {
  if (!out128) return ADG_ERR_CONFIG;
  NcclApi& n = nccl_api();
  if (!n.ok) return ADG_ERR_RUNTIME;
  ncclUniqueId id;
  if (n.getUniqueId(&id) != ncclSuccess) return ADG_ERR_RUNTIME;
  static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
  memcpy(out128, &id, sizeof id);
  return ADG_OK;
}

adg_status adg_nccl_init(adg_handle* h, const unsigned char* id128, int rank, int world) {
  if (!h || !id128) return ADG_ERR_CONFIG;
  if (world != h->cfg.world || rank != h->cfg.rank)
    return fail(h, ADG_ERR_CONFIG, "adg_nccl_init: rank/world differ from the slab configuration");
  NcclApi& n = nccl_api();
  if (!n.ok) return fail(h, ADG_ERR_RUNTIME, "libnccl.so.2 not found");
  CUDA_TRY(h, cudaSetDevice(h->cfg.device));
  if (h->comm) { n.commDestroy(h->comm); h->comm = nullptr; }
  ncclUniqueId id;
  memcpy(&id, id128, sizeof id);
  NCCL_TRY(h, n.commInitRank(&h->comm, world, id, rank));
  h->comm_rank = rank;
  h->comm_world = world;
  if (!h->comm_stream) CUDA_TRY(h, cudaStreamCreateWithFlags(&h->comm_stream, cudaStreamNonBlocking));
  for (auto& e : h->comm_ev)
    if (!e) CUDA_TRY(h, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  return ADG_OK;
}

// the ring exchange of the boundary face records of parity `par` on the comm stream
// (the same four slices as parallel.HaloExchange.views; every rank sends to next first,
// so with world 2 / 1 the messages of one peer pair match in issue order)
static adg_status enqueue_halo(adg_handle* h, int par) {
  NcclApi& n = nccl_api();
  double* tr = h->tr[par];
  const size_t nrec = (size_t)h->plane_cells * h->REC;
  const long long P = h->planes_local, pc = h->plane_cells;
  double* send_prev = tr + (0 * h->slots + pc) * h->REC;             // low-x records, first plane
  double* recv_next = tr + (0 * h->slots + (P + 1) * pc) * h->REC;   // halo-hi
  double* send_next = tr + (1 * h->slots + P * pc) * h->REC;         // high-x records, last plane
  double* recv_prev = tr + (1 * h->slots + 0) * h->REC;              // halo-lo
  const int next = (h->comm_rank + 1) % h->comm_world, prev = (h->comm_rank + h->comm_world - 1) % h->comm_world;
  CUDA_TRY(h, cudaEventRecord(h->comm_ev[0], h->stream));            // after the rerun pass
  CUDA_TRY(h, cudaStreamWaitEvent(h->comm_stream, h->comm_ev[0], 0));
  NCCL_TRY(h, n.groupStart());
  NCCL_TRY(h, n.send(send_next, nrec, ncclFloat64, next, h->comm, h->comm_stream));
  NCCL_TRY(h, n.recv(recv_prev, nrec, ncclFloat64, prev, h->comm, h->comm_stream));
  NCCL_TRY(h, n.send(send_prev, nrec, ncclFloat64, prev, h->comm, h->comm_stream));
  NCCL_TRY(h, n.recv(recv_next, nrec, ncclFloat64, next, h->comm, h->comm_stream));
  NCCL_TRY(h, n.groupEnd());
  CUDA_TRY(h, cudaEventRecord(h->comm_ev[1], h->comm_stream));
  return ADG_OK;
}

adg_status adg_run_timed_mgpu(adg_handle* h, int steps, double* out) {
  return adg_run_timed_mgpu_ex(h, steps, ADG_TIMED_KERNEL_EVENTS, out);
}

adg_status adg_run_timed_mgpu_ex(adg_handle* h, int steps, int flags, double* out) {
  return run_steps(h, steps, flags, out, true);
}

// ---------------------------------------------------------------------------
// In-process multi-GPU group: the reference's Driver(..., parallel=True,
// n_workers=N) seam (scheduler.py:92-95,126-130) on N GPUs of one process.  The
// caller creates one slab handle per device (cfg.rank = i, cfg.world = N); one NCCL
// clique (ncclCommInitAll) connects them and every group call drives each handle
// from its own host thread with exactly the per-rank step sequence of the
// one-process-per-GPU path (run_steps with the communicator), so the results are
// those of adg_run_timed_mgpu and, max being exact, of one GPU bitwise.

static adg_status group_check(adg_handle** hs, int n) {
  if (!hs || n < 1) return ADG_ERR_CONFIG;
  for (int i = 0; i < n; ++i) {
    if (!hs[i]) return ADG_ERR_CONFIG;
    if (hs[i]->cfg.world != n || hs[i]->cfg.rank != i)
      return fail(hs[0], ADG_ERR_CONFIG, "group handles must be slabs rank 0..n-1 of one world");
  }
  return ADG_OK;
}

// run f(rank) on one host thread per handle; the first failing rank's status wins
}  // extern "C"
template <class F>
static adg_status group_for_each(adg_handle** hs, int n, F f) {
  std::vector<adg_status> st(n, ADG_OK);
  std::vector<std::thread> th;
  th.reserve(n);
  for (int i = 0; i < n; ++i)
    th.emplace_back([&, i] {
      if (cudaSetDevice(hs[i]->cfg.device) != cudaSuccess) {
        st[i] = fail(hs[i], ADG_ERR_RUNTIME, "cudaSetDevice failed");
        return;
      }
      st[i] = f(i);
    });
  for (auto& t : th) t.join();
  for (int i = 0; i < n; ++i)
    if (st[i] != ADG_OK) {
      if (i != 0) hs[0]->err = hs[i]->err;
      return st[i];
    }
  return ADG_OK;
}
extern "C" {

adg_status adg_group_init(adg_handle** hs, int n) {
  adg_status s = group_check(hs, n);
  if (s != ADG_OK) return s;
  NcclApi& api = nccl_api();
  if (!api.ok) return fail(hs[0], ADG_ERR_RUNTIME, "libnccl.so.2 not found");
  std::vector<int> devs(n);
  for (int i = 0; i < n; ++i) {
    devs[i] = hs[i]->cfg.device;
    for (int j = 0; j < i; ++j)
      if (devs[j] == devs[i]) return fail(hs[0], ADG_ERR_CONFIG, "group handles need distinct devices");
    if (hs[i]->comm) { api.commDestroy(hs[i]->comm); hs[i]->comm = nullptr; }
  }
  std::vector<ncclComm_t> comms(n, nullptr);
  const ncclResult_t r = api.commInitAll(comms.data(), n, devs.data());
  if (r != ncclSuccess) return fail(hs[0], ADG_ERR_RUNTIME, api.errorString(r));
  for (int i = 0; i < n; ++i) {
    adg_handle* h = hs[i];
    h->comm = comms[i];
    h->comm_rank = i;
    h->comm_world = n;
    CUDA_TRY(h, cudaSetDevice(h->cfg.device));
    if (!h->comm_stream) CUDA_TRY(h, cudaStreamCreateWithFlags(&h->comm_stream, cudaStreamNonBlocking));
    for (auto& e : h->comm_ev)
      if (!e) CUDA_TRY(h, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  return ADG_OK;
}

static adg_status comm_reduce(adg_handle* h) {
  if (h->comm_world <= 1) return ADG_OK;
  const ncclResult_t r = nccl_api().allReduce(h->st, h->st, 2, ncclInt64, ncclMax, h->comm, h->stream);
  return r == ncclSuccess ? ADG_OK : fail(h, ADG_ERR_RUNTIME, nccl_api().errorString(r));
}

adg_status adg_group_seed(adg_handle** hs, int n) {
  adg_status s = group_check(hs, n);
  if (s != ADG_OK) return s;
  if (!hs[0]->comm) return fail(hs[0], ADG_ERR_CONFIG, "adg_group_seed needs adg_group_init");
  return group_for_each(hs, n, [&](int i) -> adg_status {
    adg_handle* h = hs[i];
    adg_status r = adg_phase_seed(h);          // Driver._seed_time_control, global max
    if (r == ADG_OK) r = comm_reduce(h);
    if (r == ADG_OK) r = adg_phase_seed_finish(h);
    if (r == ADG_OK) r = pull_state(h);
    return r == ADG_OK ? status_from_state(h) : r;
  });
}

adg_status adg_group_run(adg_handle** hs, int n, int steps, adg_step_record* out) {
  adg_status s = group_check(hs, n);
  if (s != ADG_OK) return s;
  if (!hs[0]->comm) return fail(hs[0], ADG_ERR_CONFIG, "adg_group_run needs adg_group_init");
  if (steps < 1) return ADG_OK;
  const int before = hs[0]->hst.step;
  s = group_for_each(hs, n, [&](int i) -> adg_status {
    adg_handle* h = hs[i];
    if (h->hst.status) return status_from_state(h);
    int left = steps;
    adg_status r = ADG_OK;
    if (!straightforward(h) && h->sweep_index == 0) {     // priming sweep + the first step
      r = adg_phase_sweep(h);
      if (r == ADG_OK) r = comm_reduce(h);
      if (r == ADG_OK) r = adg_phase_finish(h);
      if (r == ADG_OK) r = adg_phase_rerun(h);
      if (r == ADG_OK) r = enqueue_halo(h, adg_trace_parity(h));
      if (r == ADG_OK) r = adg_phase_sweep_part(h, ADG_PART_INTERIOR);
      if (r == ADG_OK) r = cuda_check(h, cudaStreamWaitEvent(h->stream, h->comm_ev[1], 0), "wait halo");
      if (r == ADG_OK) r = adg_phase_sweep_part(h, ADG_PART_BOUNDARY);
      if (r == ADG_OK) r = comm_reduce(h);
      if (r == ADG_OK) r = adg_phase_finish(h);
      --left;
    }
    while (r == ADG_OK && left > 0) {      // the record ring bounds one chunk
      const int chunk = left < h->rec_cap ? left : h->rec_cap;
      double tout[2];
      r = run_steps(h, chunk, ADG_TIMED_NO_PULL, tout, true);
      if (r == ADG_OK) r = pull_state(h);
      if (r == ADG_OK && h->hst.status) break;
      left -= chunk;
    }
    if (r == ADG_OK) r = pull_state(h);
    return r;
  });
  if (s != ADG_OK) return s;
  // the time control is replicated (every rank finishes on the reduced lambda):
  // rank 0's records, with the per-rank Picard counts summed
  adg_handle* h0 = hs[0];
  const int done = h0->hst.step - before;
  if (out && done > 0) {
    if ((s = fetch_records(h0, before, h0->hst.step, out)) != ADG_OK) return s;
    std::vector<adg_step_record> tmp(done);
    for (int i = 1; i < n; ++i) {
      if ((s = fetch_records(hs[i], before, before + done, tmp.data())) != ADG_OK) return s;
      for (int k = 0; k < done; ++k) {
        out[k].picard_iters += tmp[k].picard_iters;
        out[k].predicts += tmp[k].predicts;
      }
    }
  }
  for (int i = 0; i < n; ++i)
    if (hs[i]->hst.status) return status_from_state(hs[i]);
  return ADG_OK;
}

int adg_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

adg_status adg_set_option(adg_handle* h, int option, int value) {
  if (!h) return ADG_ERR_CONFIG;
  switch (option) {
    case ADG_OPT_GRAPH: h->opt_graph = value ? 1 : 0; return ADG_OK;
    case ADG_OPT_COND_RERUN: h->opt_cond_rerun = value ? 1 : 0; return ADG_OK;
    case ADG_OPT_FUSE_FINISH: h->opt_fuse_finish = value ? 1 : 0; return ADG_OK;
    case ADG_OPT_PERSISTENT: h->opt_persistent = value ? 1 : 0; return ADG_OK;
    case ADG_OPT_HOST_CHUNKS:
      if (value < 1 || value > ADG_HOST_CHUNKS_MAX) return fail(h, ADG_ERR_CONFIG, "host chunks must be in [1, 81]");
      h->opt_host_chunks = value;
      return ADG_OK;
  }
  return fail(h, ADG_ERR_CONFIG, "unknown option");
}

// ---------------------------------------------------------------------------
// One realisation step from host buffers with the transfers pipelined against
// the sweep (single slab, fused driver).  The cell planes are cut into chunks;
// per chunk: H2D of its Q (copy-in stream) -> sweep of its cells (compute
// stream) -> D2H of its Q (copy-out stream).  Without a rerun a cell's sweep
// reads only its own Q plus device-resident D and face records, so chunk i
// computes while chunk i+1 lands and chunk i-1 drains.  When the step needs
// the priming sweep or a rerun (both read every cell's Q; the rerun decision
// of the previous step is known on the host after its final sync), all of Q
// is uploaded first and only the D2H is pipelined.
static adg_status ensure_copy_streams(adg_handle* h) {
  if (!h->copy_in) CUDA_TRY(h, cudaStreamCreateWithFlags(&h->copy_in, cudaStreamNonBlocking));
  if (!h->copy_out) CUDA_TRY(h, cudaStreamCreateWithFlags(&h->copy_out, cudaStreamNonBlocking));
  if (!h->rec_host) CUDA_TRY(h, cudaMallocHost(&h->rec_host, sizeof(StepRecord)));
  if (h->chunk_ev.empty()) {
    h->chunk_ev.resize(3 * ADG_HOST_CHUNKS_MAX + 1);
    for (auto& e : h->chunk_ev) CUDA_TRY(h, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  return ADG_OK;
}

static adg_status launch_range(adg_handle* h, int mode, long long first, long long count,
                               cudaStream_t st) {
  if (count <= 0) return ADG_OK;
  SweepParams P = sweep_params(h, mode);
  P.cell_a = (int)first;
  h->disp.sweep(P, (unsigned)count, st);
  return cuda_check(h, cudaGetLastError(), "sweep launch");
}

adg_status adg_step_host(adg_handle* h, const double* Q_in, double* Q_out, adg_step_record* out) {
  if (!h || !Q_in || !Q_out) return ADG_ERR_CONFIG;
  if (h->hst.status) return status_from_state(h);
  if (!h->seeded) return fail(h, ADG_ERR_CONFIG, "time control not seeded");
  if (straightforward(h) || h->cfg.world != 1 || h->cfg.halo_mode != 0 || h->lim)
    return fail(h, ADG_ERR_CONFIG, "adg_step_host pipelines the fused single-slab driver");
  CUDA_TRY(h, cudaSetDevice(h->cfg.device));
  adg_status s = ensure_copy_streams(h);
  if (s != ADG_OK) return s;
  if (!h->hst_fresh && (s = pull_state(h)) != ADG_OK) return s;   // rerun decision after phase calls
  if (h->hst.status) return status_from_state(h);
  const size_t cell_doubles = (size_t)h->NS * h->m;
  const int want = h->opt_host_chunks;
  // chunk i = cells [cell_of(i), cell_of(i+1)): boundaries on whole waves of
  // resident CTAs so the chunked sweep keeps the single launch's wave count
  const long long C = h->cells_local;
  long long wave = 0;
  {
    int dev_sms = 148;
    cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, h->cfg.device);
    if (h->disp_ctas_per_sm == 0) h->disp_ctas_per_sm = h->disp.occ ? h->disp.occ() : 1;
    wave = (long long)dev_sms * h->disp_ctas_per_sm;
  }
  const long long waves = (C + wave - 1) / wave;
  const int nch = (int)(waves < want ? waves : want);
  auto cell_of = [&](int i) {
    const long long w = waves * i / nch;   // whole waves per chunk
    return w * wave < C ? w * wave : C;
  };
  cudaEvent_t* ev_in = h->chunk_ev.data();
  cudaEvent_t* ev_sw = ev_in + ADG_HOST_CHUNKS_MAX;
  cudaEvent_t ev_start = h->chunk_ev[3 * ADG_HOST_CHUNKS_MAX];
  const int before = h->hst.step;
  // the previous call left the compute stream idle; order the copies after it
  CUDA_TRY(h, cudaEventRecord(ev_start, h->stream));
  CUDA_TRY(h, cudaStreamWaitEvent(h->copy_in, ev_start, 0));
  CUDA_TRY(h, cudaStreamWaitEvent(h->copy_out, ev_start, 0));
  const bool priming = h->sweep_index == 0;
  const bool rerun = !priming && h->hst.rerun_next;
  auto chunk_off = [&](int i) { return (size_t)cell_of(i) * cell_doubles; };
  auto chunk_len = [&](int i) { return (size_t)(cell_of(i + 1) - cell_of(i)) * cell_doubles; };
  if (priming) {
    // the priming sweep predicts every cell before any cell is corrected: upload all of Q first
    CUDA_TRY(h, cudaMemcpyAsync(h->Q, Q_in, sizeof(double) * cell_doubles * h->cells_local,
                                cudaMemcpyHostToDevice, h->stream));
    if ((s = adg_phase_sweep(h)) != ADG_OK) return s;
    if ((s = adg_phase_finish(h)) != ADG_OK) return s;
    if ((s = adg_phase_rerun(h)) != ADG_OK) return s;
  } else {
    for (int i = 0; i < nch; ++i) {
      CUDA_TRY(h, cudaMemcpyAsync(h->Q + chunk_off(i), Q_in + chunk_off(i), sizeof(double) * chunk_len(i),
                                  cudaMemcpyHostToDevice, h->copy_in));
      CUDA_TRY(h, cudaEventRecord(ev_in[i], h->copy_in));
    }
    if (rerun) {
      // the rerun pass re-predicts a cell from its own Q only: chunk i runs as soon as its
      // part of Q has landed, so the upload hides behind it; the corrector chunks below
      // follow in stream order (they read the re-predicted records of every neighbour)
      h->hst_fresh = false;
      for (int i = 0; i < nch; ++i) {
        CUDA_TRY(h, cudaStreamWaitEvent(h->stream, ev_in[i], 0));
        if ((s = launch_range(h, MODE_RERUN, cell_of(i), cell_of(i + 1) - cell_of(i), h->stream)) != ADG_OK)
          return s;
      }
    }
  }
  const int mode = MODE_NORMAL;
  for (int i = 0; i < nch; ++i) {
    const long long c0 = cell_of(i), c1 = cell_of(i + 1);
    cudaStream_t st = h->stream;
    if (!priming && !rerun) CUDA_TRY(h, cudaStreamWaitEvent(st, ev_in[i], 0));
    if ((s = launch_range(h, mode, c0, c1 - c0, st)) != ADG_OK) return s;
    CUDA_TRY(h, cudaEventRecord(ev_sw[i], st));
    CUDA_TRY(h, cudaStreamWaitEvent(h->copy_out, ev_sw[i], 0));
    CUDA_TRY(h, cudaMemcpyAsync(Q_out + c0 * cell_doubles, h->Q + c0 * cell_doubles,
                                sizeof(double) * (size_t)(c1 - c0) * cell_doubles, cudaMemcpyDeviceToHost,
                                h->copy_out));
  }
  if ((s = adg_phase_finish(h)) != ADG_OK) return s;
  // one sync for the state, the step record and the last chunk
  CUDA_TRY(h, cudaMemcpyAsync(&h->hst, h->st, sizeof(DevState), cudaMemcpyDeviceToHost, h->stream));
  CUDA_TRY(h, cudaMemcpyAsync(h->rec_host, h->recs + (before % h->rec_cap), sizeof(StepRecord),
                              cudaMemcpyDeviceToHost, h->stream));
  CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  CUDA_TRY(h, cudaStreamSynchronize(h->copy_out));
  h->hst_fresh = true;
  if ((s = status_from_state(h)) != ADG_OK) return s;
  if (out && h->hst.step == before + 1) {
    const StepRecord& r = *h->rec_host;
    out->step = r.step; out->reruns = r.reruns; out->T = r.T; out->dt_old = r.dt_old;
    out->dt_new = r.dt_new; out->dt_adm = r.dt_adm; out->picard_iters = r.picard_iters;
    out->predicts = r.predicts; out->troubled = r.troubled;
  }
  return ADG_OK;
}

adg_status adg_flush_l2(adg_handle* h) {
  if (!h) return ADG_ERR_CONFIG;
  if (!h->flush) {
    h->flush_bytes = (size_t)256 << 20;
    CUDA_TRY(h, cudaMalloc(&h->flush, h->flush_bytes));
  }
  CUDA_TRY(h, cudaMemsetAsync(h->flush, h->sweep_index & 0xff, h->flush_bytes, h->stream));
  return ADG_OK;
}

}  // extern "C"
