// clb_capi.cu -- the C ABI (include/clawb200.h) over the sm_100a sweep kernels.
//
// Device layout (per buffer): m states, each a pitched array shaped like the
// reference's padded StateGrid (grid.py:145-160) -- two ghost layers on every
// axis -- but with rows padded to a 128-byte pitch and the interior origin
// 128-byte aligned:
//   1-D: [px]     2-D: [ny+4][px]     3-D: [nz+4][ny+4][px]
// with interior x at columns xoff .. xoff+nx-1 (xoff = 128 B / itemsize).
// Ghost layers in memory are read only for CLB_BC_HALO sides (a neighbour
// rank's halo, or the caller-filled ghosts of the per-sweep API, which the
// reference reads as-is, sweep.py:206-212); physical boundaries are
// synthesised by the kernels at load time (boundary.py semantics).  Three
// buffers per handle mirror the reference's grid + two scratch buffers
// (timestep.py:113).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <type_traits>
#include <vector>

#include "../../include/clawb200.h"
#include "clb_kernels.cuh"

namespace {

thread_local std::string g_create_error;

using clb::Result;

struct TimedLaunch {
  int axis;
  cudaEvent_t a, b;
  int counts;   // 0 for the later segment-range launches of one sweep
};

}  // namespace

struct clb_ctx {
  clb_desc d;
  int M = 0, ndim = 0, itemsize = 0;
  int64_t cells[3] = {1, 1, 1};
  int64_t px = 0, sstride = 0, origin = 0, ystride = 0, zstride = 0;
  int64_t xoff = 0, ypad = 1, zpad = 1;
  size_t buf_bytes = 0;
  void* buf[3] = {nullptr, nullptr, nullptr};
  cudaStream_t own_stream = nullptr, stream = nullptr;
  Result* d_res = nullptr;
  Result* h_res = nullptr;
  int num_sms = 148;
  int seg_override[3] = {0, 0, 0};
  int x_variant = 0;        // CLB_XVAR_*: 0 = automatic
  int resident[3][5] = {};  // [axis][contig mode, 4: streaming x]: CTAs per SM
  clb::TmaMaps maps;        // per buffer: load map, store map
  clb::TmaMaps maps_xs;     // the same for the streaming x geometry (has_xs)
  bool have_maps_xs = false;
  // x geometry pair (CLB_XVAR_TMA_ADAPT): computed cell groups of the strided
  // sweeps since the last x sweep, and the count below which the streaming
  // twin works
  unsigned long long* d_act = nullptr;
  unsigned long long xs_thresh = 0;
  // device-resident controller (clb_run_batch)
  clb::DevCtl* d_ctl = nullptr;
  clb::DevCtl* h_ctl = nullptr;
  clb_attempt* d_log = nullptr;
  int64_t log_cap = 0;
  cudaGraphExec_t batch_exec = nullptr;
  cudaGraph_t batch_graph = nullptr;
  bool have_maps = false;
  bool timing = false;
  // slab decomposition (clb_attach_comm): slow-axis halo exchange over NCCL
  // between fixed staging buffers, and the max-allreduce of the per-sweep
  // results, both on the device (inside the attempt graph of clb_run_batch)
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0;
  int nbr[2] = {-1, -1};          // rank below / above on the slow axis (-1: none)
  size_t halo_block = 0;          // bytes of 2 rows/planes of one state
  int64_t halo_send_off[2] = {0, 0}, halo_recv_off[2] = {0, 0};  // byte offsets in a buffer
  char* halo_stage = nullptr;     // [send lo, send hi, recv lo, recv hi][M][halo_block]
  cudaStream_t side = nullptr;    // exchange stream (overlaps the slow sweep's interior)
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  std::vector<TimedLaunch> launches;
  std::vector<cudaEvent_t> event_pool;
  std::string err;
};

namespace {

int fail(clb_ctx* h, int code, const std::string& msg) {
  if (h) h->err = msg; else g_create_error = msg;
  return code;
}

int cuda_fail(clb_ctx* h, cudaError_t e, const char* where) {
  return fail(h, CLB_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define CLB_CUDA(h, call)                                   \
  do {                                                      \
    cudaError_t e_ = (call);                                \
    if (e_ != cudaSuccess) return cuda_fail((h), e_, #call); \
  } while (0)

// Registered user device solvers (clb_register_device_solver).
struct UserSolver {
  int ndim = 0, m = 0, nw = 0;
  clb_user_launch_fn launch[2] = {nullptr, nullptr};  // f32, f64
  clb_user_pairs_fn pairs[2] = {nullptr, nullptr};
};
UserSolver g_user[CLB_SOLVER_USER_MAX];

const UserSolver* user_solver(int id) {
  if (id < CLB_SOLVER_USER_BASE || id >= CLB_SOLVER_USER_MAX) return nullptr;
  const UserSolver* u = &g_user[id];
  return u->launch[0] || u->launch[1] ? u : nullptr;
}

int expected_states(int solver, int ndim) {
  if (const UserSolver* u = user_solver(solver)) return u->ndim == ndim ? u->m : -1;
  switch (solver) {
    case CLB_SOLVER_ADVECTION: return 1;
    case CLB_SOLVER_ACOUSTICS: return ndim + 1;
    case CLB_SOLVER_SHALLOW_WATER: return ndim == 2 ? 3 : -1;
    case CLB_SOLVER_VC_ACOUSTICS: return ndim + 3;
  }
  return -1;
}

cudaEvent_t take_event(clb_ctx* h) {
  if (!h->event_pool.empty()) {
    cudaEvent_t e = h->event_pool.back();
    h->event_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return (PFN_cuTensorMapEncodeTiled_v12000) nullptr;
    return (PFN_cuTensorMapEncodeTiled_v12000)p;
  }();
  return fn;
}

// L2 promotion of the x boxes (CLB_TMA_PROMO = none|64|128|256; 128 default)
CUtensorMapL2promotion tma_promotion() {
  static const CUtensorMapL2promotion p = [] {
    const char* e = getenv("CLB_TMA_PROMO");
    if (!e) return CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
    switch (atoi(e)) {
      case 0: return CU_TENSOR_MAP_L2_PROMOTION_NONE;
      case 64: return CU_TENSOR_MAP_L2_PROMOTION_L2_64B;
      case 256: return CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
      default: return CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
    }
  }();
  return p;
}

// 4-D view (x, y, z, state) of one buffer for the contiguous-axis sweep: box =
// 48 bytes of x by 128 rows.  `store` limits the extent to the interior so
// tiles that overhang the grid are clipped by the TMA unit.
bool make_tensor_map(clb_ctx* h, int buf, bool store, void* out, int xs = 0) {
  auto enc = tensor_map_encoder();
  if (!enc) return false;
  const int isz = h->itemsize;
  cuuint64_t dims[4], strides[3];
  if (store) {
    dims[0] = (cuuint64_t)(h->xoff + h->cells[0]);
    dims[1] = (cuuint64_t)(h->ndim >= 2 ? h->cells[1] + 2 : 1);
    dims[2] = (cuuint64_t)(h->ndim == 3 ? h->cells[2] + 2 : 1);
  } else {
    dims[0] = (cuuint64_t)h->px;
    dims[1] = (cuuint64_t)h->ypad;
    dims[2] = (cuuint64_t)h->zpad;
  }
  dims[3] = (cuuint64_t)h->M;
  strides[0] = (cuuint64_t)(h->ystride * isz);
  strides[1] = (cuuint64_t)(h->zstride * isz);
  strides[2] = (cuuint64_t)(h->sstride * isz);
  // x stages: 64-byte rows (whole sectors) with the 64-byte swizzle
  // (clb_kernels.cuh XGeom); CLB_X_LEGACY: 48-byte rows, no swizzle
  const bool legacy = CLB_X_LEGACY != 0;
  const int row = legacy ? 48 : clb::x_row_bytes(h->M, xs);
  const int rows = legacy ? 128 : (xs ? clb::x_rows<1>() : clb::x_rows<0>());
  cuuint32_t box[4] = {(cuuint32_t)(row / isz), (cuuint32_t)rows, 1u, 1u};
  cuuint32_t estr[4] = {1u, 1u, 1u, 1u};
  CUresult r = enc((CUtensorMap*)out,
                   isz == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4,
                   h->buf[buf], dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   legacy ? CU_TENSOR_MAP_SWIZZLE_NONE
                          : (row == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                             : row == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B),
                   tma_promotion(), CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

cudaError_t dispatch_family(clb_ctx* h, int axis, bool literal, const clb::GenericArgs& g,
                            cudaStream_t st);

// Resident CTAs per SM of the (non-literal) sweep kernel the geometry selects
// (cudaOccupancyMaxActiveBlocksPerMultiprocessor, cached per axis and mode).
int resident_ctas(clb_ctx* h, int axis, const clb::GenericArgs& g0) {
  int& r = h->resident[axis][g0.xs ? 4 : g0.contig];
  if (r == 0) {
    clb::GenericArgs g = g0;
    int occ = 0;
    g.occ_out = &occ;
    if (dispatch_family(h, axis, false, g, h->stream) != cudaSuccess || occ < 1) occ = 1;
    r = occ;
  }
  return r;
}

// The x-sweep variant a handle runs (CLB_XVAR_*, never AUTO).
// x-sweep kernel: the TMA tensor-map variant wins when the march is
// compute-heavy (fp64 shallow water, profiles/r1_notes.md); the warp-shuffle
// variant wins elsewhere.  Small grids (C2, 1024^2) have too few 128-row
// blocks for the TMA variant and run faster warp-marching (56 vs 69 us).
// 3-D acoustics (m = 4) also streams x faster through the TMA transpose
// with 32-byte rows on large grids (C5 fp64 x 2.20 vs 2.39 ms, r2j).  fp64
// shallow water pairs the two TMA geometries (CLB_XVAR_TMA_ADAPT).
// clb_set_x_variant (per handle) overrides.
int x_mode(const clb_ctx* h) {
  int v = h->x_variant;
  if (v == CLB_XVAR_AUTO) {
    const int64_t ncells = h->cells[0] * h->cells[1] * h->cells[2];
    const bool big = ncells >= ((int64_t)1 << 22);
    v = (big && (h->d.solver_id == CLB_SOLVER_SHALLOW_WATER ||
                 (h->d.solver_id == CLB_SOLVER_ACOUSTICS && h->ndim == 3)))
            ? (h->have_maps_xs ? CLB_XVAR_TMA_ADAPT : CLB_XVAR_TMA)
            : CLB_XVAR_MARCH;
  }
  if (v == CLB_XVAR_TMA && !h->have_maps) v = CLB_XVAR_MARCH;
  if ((v == CLB_XVAR_TMA_STREAM || v == CLB_XVAR_TMA_ADAPT) && !h->have_maps_xs)
    v = h->have_maps ? CLB_XVAR_TMA : CLB_XVAR_MARCH;
  return v;
}

// Geometry of one sweep: which kernel, extents and strides (xs = 1: the
// streaming twin of the TMA x sweep; -1: the default geometry whatever the
// variant, for the literal kernels, which have no streaming twin).
clb::GenericArgs sweep_geometry(clb_ctx* h, int axis, int src, int dst, int xs = 0) {
  clb::GenericArgs g;
  std::memset(&g, 0, sizeof(g));
  const int64_t isz = h->itemsize;
  g.qin = (const char*)h->buf[src] + h->origin * isz;
  g.qout = (char*)h->buf[dst] + h->origin * isz;
  g.src = src;
  g.dst = dst;
  g.axis = axis;
  g.spacing = h->d.spacing[axis];
  for (int b = 0; b < 3; ++b) g.bufs[b] = (const char*)h->buf[b] + h->origin * isz;
  g.sstride = h->sstride;
  g.bc_lo = h->d.bc[axis][0];
  g.bc_hi = h->d.bc[axis][1];
  g.nv = h->d.normal_velocity[axis];
  g.lim_id = h->d.limiter_id;
  g.num_sms = h->num_sms;
  const int64_t nx = h->cells[0], ny = h->cells[1], nz = h->cells[2];
  // Work decomposition: 128 pencils per CTA; segments along the sweep axis
  // (chosen below against the resident CTA slots), never shorter than 16
  // cells (each segment re-reads 4 cells and re-solves 3 fans of its
  // neighbour; CLB_MIN_SEG overrides, profiles/r1_notes.md).
  const int64_t target_ctas = (int64_t)h->num_sms * 6;
  int64_t pen_ctas;
  const int mode = x_mode(h);
  if (axis == 0) {
    g.contig = mode >= CLB_XVAR_TMA_STREAM ? 2 : mode;
    g.xs = xs < 0 ? 0 : (xs > 0 || mode == CLB_XVAR_TMA_STREAM) ? 1 : 0;
    g.n = (int)nx; g.n1 = (int)ny; g.n2 = (int)nz;
    g.astride = 1; g.t1stride = h->ystride; g.t2stride = h->zstride;
    g.maps = g.xs ? &h->maps_xs : &h->maps;
    g.tx0 = (int)h->xoff;
    g.ty0 = h->ndim >= 2 ? 2 : 0;
    g.tz0 = h->ndim == 3 ? 2 : 0;
    // warp-marching: one warp per (row, segment), 4 warps per CTA;
    // TMA: 128 rows of one z-plane per CTA
    pen_ctas = g.contig != 2 ? (ny * nz + 3) / 4
                             : ((ny + clb::x_rows<0>() - 1) / clb::x_rows<0>()) * nz;
    if (g.xs) pen_ctas = ((ny + clb::x_rows<1>() - 1) / clb::x_rows<1>()) * nz;
  } else {
    g.contig = 0;
    g.n1 = (int)nx;
    g.t1stride = 1;
    if (axis == 1) {
      g.n = (int)ny; g.n2 = (int)nz; g.astride = h->ystride; g.t2stride = h->zstride;
    } else {
      g.n = (int)nz; g.n2 = (int)ny; g.astride = h->zstride; g.t2stride = h->ystride;
    }
    pen_ctas = ((nx + 127) / 128) * g.n2;
  }
  // contig stages are 64 (legacy: 48) bytes of a row: segment starts stay aligned
  const int64_t align =
      (axis == 0 && g.contig == 2) ? (CLB_X_LEGACY ? 48 : clb::x_stage_bytes(h->M, g.xs)) / h->itemsize
                                   : 1;
  static const int64_t min_seg = [] {
    const char* e = getenv("CLB_MIN_SEG");
    return e ? std::max<int64_t>(4, atoll(e)) : (int64_t)16;
  }();
  // segment length L of a candidate segment count: warp-marching spans L + 4
  // cells in 32-lane chunks, so L + 4 is a multiple of 32 (no idle lanes)
  auto seg_len_of = [&](int64_t ns) {
    int64_t L = (g.n + ns - 1) / ns;
    if (axis == 0 && g.contig == 1) L = std::max<int64_t>(28, (L + 4 + 31) / 32 * 32 - 4);
    // pair march: 64-cell chunks from lo - 4 while b - 2 < hi, i.e. L + 2 of 64
    if (axis == 0 && g.contig == 3) L = std::max<int64_t>(62, (L + 2 + 63) / 64 * 64 - 2);
    return (L + align - 1) / align * align;
  };
  // CTAs a segment count launches (the warp-march packs 4 row-warps per CTA)
  auto ctas_of = [&](int64_t ns) {
    return (axis == 0 && g.contig != 2) ? (ny * nz * ns + 3) / 4 : pen_ctas * ns;
  };
  // Segment count: maximise (busy fraction of the last wave) x (L / (L+4),
  // the share of non-redundant work) over the resident CTA slots, so that
  // grids do not end on a nearly empty wave (8192^2: 896 CTAs on 296 slots
  // left 140 SMs idle for a quarter of the sweep).
  (void)target_ctas;
  const int64_t slots = (int64_t)h->num_sms * resident_ctas(h, axis, g);
  const int64_t max_seg = std::max<int64_t>(1, std::min<int64_t>(g.n / min_seg, 4096));
  int64_t best_n = 1;
  double best_e = -1.0;
  for (int64_t ns = 1; ns <= max_seg; ++ns) {
    const int64_t L = seg_len_of(ns);
    const int64_t ns2 = (g.n + L - 1) / L;
    if (ns2 != ns) continue;
    const int64_t c = ctas_of(ns2);
    const int64_t waves = (c + slots - 1) / slots;
    const double e = (double)c / (double)(waves * slots) * ((double)L / (double)(L + 4));
    if (e > best_e + 1e-9) {
      best_e = e;
      best_n = ns2;
    }
  }
  int64_t L = seg_len_of(best_n);
  if (h->seg_override[axis] > 0) L = (h->seg_override[axis] + align - 1) / align * align;
  g.seg_len = (int)L;
  g.nseg = (int)((g.n + L - 1) / L);
  g.seg_begin = 0;
  g.seg_end = g.nseg;
  return g;
}

cudaError_t dispatch_family(clb_ctx* h, int axis, bool literal, const clb::GenericArgs& g,
                            cudaStream_t st) {
  const bool d64 = h->itemsize == 8;
  const int nd = h->ndim;
  if (const UserSolver* u = user_solver(h->d.solver_id)) {
    clb_user_launch_fn fn = u->launch[d64 ? 1 : 0];
    if (!fn) return cudaErrorInvalidValue;
    return (cudaError_t)fn(nd, axis, literal ? 1 : 0, &g, (void*)st);
  }
  switch (h->d.solver_id) {
    case CLB_SOLVER_ACOUSTICS:
      return d64 ? clb::launch_acoustics_f64(nd, axis, literal, g, st)
                 : clb::launch_acoustics_f32(nd, axis, literal, g, st);
    case CLB_SOLVER_SHALLOW_WATER:
      return d64 ? clb::launch_shallow_water_f64(nd, axis, literal, g, st)
                 : clb::launch_shallow_water_f32(nd, axis, literal, g, st);
    case CLB_SOLVER_ADVECTION:
      return d64 ? clb::launch_advection_f64(nd, axis, literal, g, st)
                 : clb::launch_advection_f32(nd, axis, literal, g, st);
    default:
      return d64 ? clb::launch_vc_acoustics_f64(nd, axis, literal, g, st)
                 : clb::launch_vc_acoustics_f32(nd, axis, literal, g, st);
  }
}

// NCCL, loaded at run time (the library does not link it): torch's copy
// when torch is already in the process (same soname), else the system one.
struct NcclApi {
  bool ok = false;
  std::string err;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void* lib = nullptr;
    const char* env = getenv("CLB_NCCL_LIB");
    for (const char* name : {env, "libnccl.so.2", "libnccl.so"}) {
      if (!name) continue;
      lib = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (lib) break;
    }
    if (!lib) { a.err = "libnccl.so.2 not found"; return a; }
    bool all = true;
    auto sym = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(lib, name));
      all = all && fn != nullptr;
    };
    sym(a.GetUniqueId, "ncclGetUniqueId");
    sym(a.CommInitRank, "ncclCommInitRank");
    sym(a.CommDestroy, "ncclCommDestroy");
    sym(a.AllReduce, "ncclAllReduce");
    sym(a.Send, "ncclSend");
    sym(a.Recv, "ncclRecv");
    sym(a.GroupStart, "ncclGroupStart");
    sym(a.GroupEnd, "ncclGroupEnd");
    sym(a.GetErrorString, "ncclGetErrorString");
    a.ok = all;
    if (!all) a.err = "libnccl.so.2 lacks a required symbol";
    return a;
  }();
  return api;
}

int nccl_fail(clb_ctx* h, ncclResult_t r, const char* where) {
  const NcclApi& n = nccl();
  return fail(h, CLB_ECUDA, std::string(where) + ": " +
                                (n.GetErrorString ? n.GetErrorString(r) : "nccl error"));
}

#define CLB_NCCL(h, call)                                        \
  do {                                                           \
    ncclResult_t r_ = (call);                                    \
    if (r_ != ncclSuccess) return nccl_fail((h), r_, #call);     \
  } while (0)

// Halo pack / unpack between a buffer's 2 boundary rows/planes (per state a
// contiguous block) and the staging area.  Indirect (ctl != null): the
// buffer is the controller's input of the slow sweep, and a finished
// controller makes them no-ops (graph replays past the end of a run).
struct HaloArgs {
  const clb::DevCtl* ctl;
  int slow;                 // slow axis (the sweep whose input is exchanged)
  int buf;                  // direct launches
  char* bufs[3];
  int64_t off[2];           // byte offset of the side's block in a buffer
  int64_t sstride;          // bytes between states
  int64_t block;            // bytes per state and side (multiple of 16)
  int m;
  int side_mask;            // bit s: side s has a neighbour
  char* stage;              // [2 sides][m][block]
};

__global__ void halo_copy_kernel(HaloArgs a, int unpack) {
  if (a.ctl && a.ctl->done) return;
  const int b = a.ctl ? a.ctl->src[a.slow] : a.buf;
  char* base = a.bufs[b];
  const int64_t nvec = a.block / 16;
  for (int side = 0; side < 2; ++side) {
    if (!(a.side_mask >> side & 1)) continue;
    for (int k = 0; k < a.m; ++k) {
      uint4* g = reinterpret_cast<uint4*>(base + a.off[side] + k * a.sstride);
      uint4* st = reinterpret_cast<uint4*>(a.stage + ((int64_t)side * a.m + k) * a.block);
      for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nvec;
           i += (int64_t)gridDim.x * blockDim.x) {
        if (unpack) g[i] = st[i]; else st[i] = g[i];
      }
    }
  }
}

HaloArgs halo_args(clb_ctx* h, bool recv, int buf, bool indirect) {
  HaloArgs a;
  a.ctl = indirect ? h->d_ctl : nullptr;
  a.slow = h->ndim - 1;
  a.buf = buf;
  for (int i = 0; i < 3; ++i) a.bufs[i] = (char*)h->buf[i];
  for (int s = 0; s < 2; ++s) a.off[s] = recv ? h->halo_recv_off[s] : h->halo_send_off[s];
  a.sstride = h->sstride * h->itemsize;
  a.block = (int64_t)h->halo_block;
  a.m = h->M;
  a.side_mask = (h->nbr[0] >= 0 ? 1 : 0) | (h->nbr[1] >= 0 ? 2 : 0);
  a.stage = h->halo_stage + (recv ? 2 : 0) * (size_t)h->M * h->halo_block;
  return a;
}

// pack -> send/recv -> unpack on stream `st`.  NCCL pairs the messages of
// two ranks in posting order, so the order is canonical: send the hi rows,
// then the lo rows; receive into the lo ghosts, then the hi ghosts (which
// also pairs a 2-rank periodic ring and a rank exchanging with itself).
int halo_exchange_on(clb_ctx* h, cudaStream_t st, int buf, bool indirect) {
  const NcclApi& n = nccl();
  const int blocks = (int)std::min<int64_t>((h->halo_block / 16 + 255) / 256 * 2, 4 * h->num_sms);
  halo_copy_kernel<<<std::max(blocks, 1), 256, 0, st>>>(halo_args(h, false, buf, indirect), 0);
  CLB_CUDA(h, cudaGetLastError());
  const size_t bytes = (size_t)h->M * h->halo_block;
  char* send = h->halo_stage;
  char* recv = h->halo_stage + 2 * bytes;
  CLB_NCCL(h, n.GroupStart());
  if (h->nbr[1] >= 0) CLB_NCCL(h, n.Send(send + bytes, bytes, ncclUint8, h->nbr[1], h->comm, st));
  if (h->nbr[0] >= 0) CLB_NCCL(h, n.Send(send, bytes, ncclUint8, h->nbr[0], h->comm, st));
  if (h->nbr[0] >= 0) CLB_NCCL(h, n.Recv(recv, bytes, ncclUint8, h->nbr[0], h->comm, st));
  if (h->nbr[1] >= 0) CLB_NCCL(h, n.Recv(recv + bytes, bytes, ncclUint8, h->nbr[1], h->comm, st));
  CLB_NCCL(h, n.GroupEnd());
  halo_copy_kernel<<<std::max(blocks, 1), 256, 0, st>>>(halo_args(h, true, buf, indirect), 1);
  CLB_CUDA(h, cudaGetLastError());
  return CLB_OK;
}

// max over ranks of the per-sweep results: non-negative doubles order as
// their bit patterns (uint64 max), flags as int32 max; exact, order-free.
int results_allreduce(clb_ctx* h, cudaStream_t st) {
  const NcclApi& n = nccl();
  CLB_NCCL(h, n.AllReduce(h->d_res->smax, h->d_res->smax, (size_t)h->ndim, ncclUint64, ncclMax,
                          h->comm, st));
  CLB_NCCL(h, n.AllReduce(h->d_res->nonfinite, h->d_res->nonfinite, (size_t)h->ndim, ncclInt32,
                          ncclMax, h->comm, st));
  return CLB_OK;
}

// indirect: buffers and dt are read by the kernel from h->d_ctl (batch graphs)
int launch_sweep(clb_ctx* h, int axis, double dt, int src, int dst, int slot, bool literal,
                 bool indirect = false, int seg_begin = 0, int seg_end = -1, bool fuse = false) {
  if (axis < 0 || axis >= h->ndim) return fail(h, CLB_EINVAL, "sweep axis out of range");
  if (src < 0 || src > 2 || dst < 0 || dst > 2) return fail(h, CLB_EINVAL, "buffer index out of range");
  if (src == dst) return fail(h, CLB_EINVAL, "sweep cannot run in place");
  if (!(dt > 0.0)) return fail(h, CLB_EINVAL, "dt must be positive");
  if (slot < 0 || slot > 3) return fail(h, CLB_EINVAL, "result slot out of range");
  cudaSetDevice(h->d.device);  // handles on several devices in one process
  clb::GenericArgs g = sweep_geometry(h, axis, src, dst, literal ? -1 : 0);
  // x geometry pair: both twins launch, the count selects the working one
  const bool paired = x_mode(h) == CLB_XVAR_TMA_ADAPT;
  if (paired) {
    if (axis == 0 && !literal) {
      g.xsel = h->d_act;
      g.xsel_thresh = h->xs_thresh;
    } else if (axis > 0) {
      g.act = h->d_act;
    }
  }
  g.ctl = indirect ? h->d_ctl : nullptr;
  g.fuse_ctl = (indirect && fuse) ? 1 : 0;
  g.res = h->d_res;
  if (seg_end >= 0) {
    if (g.contig) return fail(h, CLB_EINVAL, "segment ranges apply to strided sweeps only");
    if (seg_begin < 0 || seg_end > g.nseg || seg_begin >= seg_end)
      return fail(h, CLB_EINVAL, "segment range out of bounds");
    g.seg_begin = seg_begin;
    g.seg_end = seg_end;
  }
  // sweep.py:336-337: dtdx = T(dt / dx[axis]) -- fp64 divide, then round to T.
  const double dtdx64 = dt / h->d.spacing[axis];
  g.dtdx = h->itemsize == 8 ? dtdx64 : (double)(float)dtdx64;
  for (int i = 0; i < 4; ++i) g.params[i] = h->d.params[i];
  g.smax_bits = &h->d_res->smax[slot];
  g.nonfinite = &h->d_res->nonfinite[slot];
  TimedLaunch tl{axis, nullptr, nullptr, (seg_end < 0 || seg_begin == 0) ? 1 : 0};
  if (h->timing && !indirect) {
    tl.a = take_event(h);
    tl.b = take_event(h);
    cudaEventRecord(tl.a, h->stream);
  }
  cudaError_t e = dispatch_family(h, axis, literal, g, h->stream);
  if (e != cudaSuccess) return cuda_fail(h, e, "sweep launch");
  if (paired && axis == 0) {
    if (!literal) {
      clb::GenericArgs g1 = sweep_geometry(h, axis, src, dst, 1);
      g1.ctl = g.ctl; g1.fuse_ctl = g.fuse_ctl; g1.res = g.res; g1.dtdx = g.dtdx;
      for (int i = 0; i < 4; ++i) g1.params[i] = g.params[i];
      g1.smax_bits = g.smax_bits; g1.nonfinite = g.nonfinite;
      g1.xsel = g.xsel; g1.xsel_thresh = g.xsel_thresh;
      e = dispatch_family(h, axis, literal, g1, h->stream);
      if (e != cudaSuccess) return cuda_fail(h, e, "sweep launch (streaming x)");
    }
    e = cudaMemsetAsync(h->d_act, 0, sizeof(unsigned long long), h->stream);
    if (e != cudaSuccess) return cuda_fail(h, e, "x selector reset");
  }
  if (h->timing && !indirect) {
    cudaEventRecord(tl.b, h->stream);
    h->launches.push_back(tl);
  }
  return CLB_OK;
}

// The slow-axis sweep overlapped with its halo exchange (slab.py
// slow_sweep, on the device): the segments whose rows stay clear of the
// ghost layers run on the main stream while pack / send / recv / unpack run
// on the side stream; the two edge groups follow the join.  Segments are
// independent, so this is bitwise one exchange followed by one sweep.
int slow_sweep_exchange(clb_ctx* h, double dt, int src, int dst, int slot, bool literal,
                        bool indirect) {
  const int axis = h->ndim - 1;
  const clb::GenericArgs g = sweep_geometry(h, axis, 0, 1);
  const int64_t n = h->cells[axis], L = g.seg_len;
  int b = -1, e = -1;
  for (int k = 0; k < g.nseg; ++k) {
    if ((int64_t)k * L >= 2 && std::min<int64_t>(n, (int64_t)(k + 1) * L) + 2 <= n) {
      if (b < 0) b = k;
      e = k + 1;
    }
  }
  CLB_CUDA(h, cudaEventRecord(h->ev_fork, h->stream));
  CLB_CUDA(h, cudaStreamWaitEvent(h->side, h->ev_fork, 0));
  int r = halo_exchange_on(h, h->side, src, indirect);
  if (r) return r;
  CLB_CUDA(h, cudaEventRecord(h->ev_join, h->side));
  if (b >= 0) {
    r = launch_sweep(h, axis, dt, src, dst, slot, literal, indirect, b, e);
    if (r) return r;
  }
  CLB_CUDA(h, cudaStreamWaitEvent(h->stream, h->ev_join, 0));
  if (b < 0) return launch_sweep(h, axis, dt, src, dst, slot, literal, indirect);
  if (b > 0) {
    r = launch_sweep(h, axis, dt, src, dst, slot, literal, indirect, 0, b);
    if (r) return r;
  }
  if (e < g.nseg) return launch_sweep(h, axis, dt, src, dst, slot, literal, indirect, e, g.nseg);
  return CLB_OK;
}

// one sweep of an attempt: the slow axis of a slab exchanges its halo first
int attempt_sweep(clb_ctx* h, int axis, double dt, int src, int dst, int slot, bool literal,
                  bool indirect) {
  if (h->comm && axis == h->ndim - 1) return slow_sweep_exchange(h, dt, src, dst, slot, literal, indirect);
  return launch_sweep(h, axis, dt, src, dst, slot, literal, indirect);
}

int fetch(clb_ctx* h, int nslots, double* speeds, int32_t* nonfinite) {
  CLB_CUDA(h, cudaMemcpyAsync(h->h_res, h->d_res, sizeof(Result), cudaMemcpyDeviceToHost, h->stream));
  CLB_CUDA(h, cudaMemsetAsync(h->d_res, 0, sizeof(Result), h->stream));
  CLB_CUDA(h, cudaStreamSynchronize(h->stream));
  for (int i = 0; i < nslots && i < 4; ++i) {
    if (speeds) {
      double v;
      std::memcpy(&v, &h->h_res->smax[i], sizeof(double));
      speeds[i] = v;
    }
    if (nonfinite) nonfinite[i] = h->h_res->nonfinite[i] ? 1 : 0;
  }
  return CLB_OK;
}

// timestep.py:179-186: first non-finite interior value in C order.
template <typename T>
__global__ void first_bad_kernel(const T* q, int64_t sstride, int64_t ystride, int64_t zstride,
                                 int64_t nx, int64_t ny, int64_t nz, int m,
                                 unsigned long long* out) {
  const int64_t total = (int64_t)m * nz * ny * nx;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = i;
    const int64_t x = r % nx; r /= nx;
    const int64_t y = r % ny; r /= ny;
    const int64_t z = r % nz; r /= nz;
    const int64_t k = r;
    const T v = q[k * sstride + z * zstride + y * ystride + x];
    if (clb::finite_key(v) == 0u) atomicMin(out, (unsigned long long)i);
  }
}

}  // namespace


// FastArith (clb_solvers.cuh) against div.rn / sqrt.rn, bit for bit.
__global__ void selftest_arith_kernel(const double* a, const double* b, int64_t n,
                                      unsigned long long* cnt) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double x = a[i], y = b[i];
  bool bq = false, bs = false;
  const double qf = clb::FastArith::div<double, clb::kChkAll>(x, y, bq);
  const double sf = clb::FastArith::sqrt<double>(x, bs);
  const double qr = __ddiv_rn(x, y), sr = __dsqrt_rn(x);
  if (!bq && __double_as_longlong(qf) != __double_as_longlong(qr)) atomicAdd(&cnt[0], 1ull);
  if (!bs && __double_as_longlong(sf) != __double_as_longlong(sr)) atomicAdd(&cnt[1], 1ull);
  if (bq) atomicAdd(&cnt[2], 1ull);
  if (bs) atomicAdd(&cnt[3], 1ull);
  // fp32: the low words reinterpreted as floats (every float class occurs)
  const float xf = __int_as_float(__double2loint(x)), yf = __int_as_float(__double2loint(y));
  bool cq = false, cs = false;
  const float qff = clb::FastArith::div<float, clb::kChkAll>(xf, yf, cq);
  const float sff = clb::FastArith::sqrt<float>(xf, cs);
  if (!cq && __float_as_int(qff) != __float_as_int(__fdiv_rn(xf, yf))) atomicAdd(&cnt[4], 1ull);
  if (!cs && __float_as_int(sff) != __float_as_int(__fsqrt_rn(xf))) atomicAdd(&cnt[5], 1ull);
  if (cq) atomicAdd(&cnt[6], 1ull);
  if (cs) atomicAdd(&cnt[7], 1ull);
  // limiter ratio: equal to div.rn, or both zero (the sign is free)
  bool bl = false;
  const double ql = clb::FastArith::div<double, clb::kChkLim>(x, y, bl);
  const bool zeq = (__double_as_longlong(ql) << 1) == 0 && (__double_as_longlong(qr) << 1) == 0;
  if (!bl && __double_as_longlong(ql) != __double_as_longlong(qr) && !zeq) atomicAdd(&cnt[8], 1ull);
  if (bl) atomicAdd(&cnt[9], 1ull);
  // Roe quotient: precondition b in [2^-485, 2^513]
  if (y >= 0x1p-485 && y <= 0x1p513) {
    bool br = false;
    const double qn = clb::FastArith::div<double, clb::kChkNumNormDen>(x, y, br);
    if (!br && __double_as_longlong(qn) != __double_as_longlong(qr)) atomicAdd(&cnt[10], 1ull);
    if (br) atomicAdd(&cnt[11], 1ull);
  }
}


namespace clb {
__global__ void ctl_prepare(DevCtl* c) { ctl_prepare_next(c); }
__global__ void ctl_finish(DevCtl* c, Result* r) { ctl_finish_dev(c, r); }
}  // namespace clb

extern "C" {

int clb_version(void) { return 1; }

size_t clb_sweep_args_size(void) { return sizeof(clb::GenericArgs); }

int clb_register_device_solver(int solver_id, int ndim, int num_states, int num_waves,
                               size_t args_size, clb_user_launch_fn launch_f32,
                               clb_user_launch_fn launch_f64, clb_user_pairs_fn pairs_f32,
                               clb_user_pairs_fn pairs_f64) {
  if (solver_id < CLB_SOLVER_USER_BASE || solver_id >= CLB_SOLVER_USER_MAX)
    return fail(nullptr, CLB_EINVAL, "user solver ids are CLB_SOLVER_USER_BASE .. USER_MAX-1");
  if (ndim < 1 || ndim > 3 || num_states < 1 || num_waves < 1)
    return fail(nullptr, CLB_EINVAL, "bad user solver shape");
  if (args_size != sizeof(clb::GenericArgs))
    return fail(nullptr, CLB_EUNSUPPORTED,
                "user solver compiled against a different library build (argument block size)");
  if (!launch_f32 && !launch_f64) return fail(nullptr, CLB_EINVAL, "no launch entry point");
  UserSolver& u = g_user[solver_id];
  u.ndim = ndim;
  u.m = num_states;
  u.nw = num_waves;
  u.launch[0] = launch_f32;
  u.launch[1] = launch_f64;
  u.pairs[0] = pairs_f32;
  u.pairs[1] = pairs_f64;
  return CLB_OK;
}

const char* clb_last_error(clb_handle h) {
  return h ? h->err.c_str() : g_create_error.c_str();
}

int clb_create(const clb_desc* desc, clb_handle* out) {
  if (!desc || !out) return fail(nullptr, CLB_EINVAL, "null argument");
  *out = nullptr;
  const clb_desc& d = *desc;
  if (d.ndim < 1 || d.ndim > 3) return fail(nullptr, CLB_EINVAL, "grid must be 1-, 2- or 3-dimensional");
  if (d.itemsize != 4 && d.itemsize != 8) return fail(nullptr, CLB_EINVAL, "itemsize must be 4 or 8");
  if (d.limiter_id < 0 || d.limiter_id > 4) return fail(nullptr, CLB_EINVAL, "unknown limiter id");
  const int em = expected_states(d.solver_id, d.ndim);
  if (em < 0) return fail(nullptr, CLB_EUNSUPPORTED, "solver not supported for this dimensionality");
  if (d.num_states != em)
    return fail(nullptr, CLB_EUNSUPPORTED, "num_states does not match the device solver's state layout");
  for (int ax = 0; ax < d.ndim; ++ax) {
    if (d.cells[ax] < 1 || d.cells[ax] > (int64_t)1 << 30)
      return fail(nullptr, CLB_EINVAL, "cell counts must be in [1, 2^30]");
    if (!(d.spacing[ax] > 0.0)) return fail(nullptr, CLB_EINVAL, "spacing must be positive");
    for (int s = 0; s < 2; ++s) {
      const int bc = d.bc[ax][s];
      if (bc < 0 || bc > 3) return fail(nullptr, CLB_EINVAL, "unknown boundary kind");
      if ((bc == CLB_BC_PERIODIC || bc == CLB_BC_REFLECTIVE) && d.cells[ax] < 2)
        return fail(nullptr, CLB_EUNSUPPORTED,
                    "periodic/reflective boundaries need at least 2 cells on the axis");
      if (bc == CLB_BC_REFLECTIVE &&
          (d.normal_velocity[ax] < 0 || d.normal_velocity[ax] >= d.num_states))
        return fail(nullptr, CLB_EINVAL, "reflective boundary needs a normal velocity state");
    }
    if ((d.bc[ax][0] == CLB_BC_PERIODIC) != (d.bc[ax][1] == CLB_BC_PERIODIC))
      return fail(nullptr, CLB_EINVAL, "periodic boundary must be set on both sides");
  }
  if (d.solver_id == CLB_SOLVER_ACOUSTICS && !(std::isfinite(d.params[0]) && d.params[0] > 0.0))
    return fail(nullptr, CLB_EINVAL, "sound speed must be positive and finite");

  clb_ctx* h = new clb_ctx();
  h->d = d;
  h->ndim = d.ndim;
  h->M = d.num_states;
  h->itemsize = d.itemsize;
  {
    // process-wide default of clb_set_x_variant: CLB_CONTIG=tma|shfl|pair|stream|adapt
    const char* e = getenv("CLB_CONTIG");
    const std::string v = e ? e : "";
    h->x_variant = v == "tma" ? CLB_XVAR_TMA : v == "pair" ? CLB_XVAR_PAIR
                   : v == "stream" ? CLB_XVAR_TMA_STREAM : v == "adapt" ? CLB_XVAR_TMA_ADAPT
                   : v == "shfl" || v == "march" ? CLB_XVAR_MARCH : CLB_XVAR_AUTO;
  }
  for (int ax = 0; ax < d.ndim; ++ax) h->cells[ax] = d.cells[ax];
  const int64_t align = 128 / d.itemsize;
  h->xoff = align;
  // slack past the x ghosts: contig stages may read up to 16 cells beyond n
  // (beyond the row the TMA unit zero-fills)
  h->px = (h->xoff + h->cells[0] + 16 + align - 1) / align * align;
  {
    // CLB_PITCH_PAD: extra 128-byte units per row (layout experiments; results
    // are independent of the pitch)
    const char* e = getenv("CLB_PITCH_PAD");
    if (e) h->px += std::max(0, atoi(e)) * align;
  }
  h->ypad = d.ndim >= 2 ? h->cells[1] + 4 : 1;
  h->zpad = d.ndim == 3 ? h->cells[2] + 4 : 1;
  h->ystride = h->px;
  h->zstride = h->px * h->ypad;
  h->sstride = h->zstride * h->zpad;
  h->origin = h->xoff + (d.ndim >= 2 ? 2 * h->ystride : 0) + (d.ndim == 3 ? 2 * h->zstride : 0);
  h->buf_bytes = (size_t)h->sstride * h->M * h->itemsize;

  cudaError_t e = cudaSetDevice(d.device);
  if (e != cudaSuccess) { int r = cuda_fail(nullptr, e, "cudaSetDevice"); delete h; return r; }
  cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, d.device);
  e = cudaStreamCreateWithFlags(&h->own_stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) { int r = cuda_fail(nullptr, e, "cudaStreamCreate"); delete h; return r; }
  h->stream = h->own_stream;
  for (int i = 0; i < 3; ++i) {
    e = cudaMalloc(&h->buf[i], h->buf_bytes);
    if (e != cudaSuccess) {
      int r = fail(nullptr, CLB_ENOMEM, std::string("device allocation failed: ") + cudaGetErrorString(e));
      clb_destroy(h);
      return r;
    }
    cudaMemsetAsync(h->buf[i], 0, h->buf_bytes, h->stream);
  }
  h->have_maps = true;
  for (int b = 0; b < 3 && h->have_maps; ++b)
    if (!(make_tensor_map(h, b, false, h->maps.ld[b]) && make_tensor_map(h, b, true, h->maps.st[b])))
      h->have_maps = false;
  // the streaming x twin (built-in fp64 2-D shallow water only)
  if (h->have_maps && d.solver_id == CLB_SOLVER_SHALLOW_WATER && d.itemsize == 8 && d.ndim == 2 &&
      !CLB_X_LEGACY) {
    h->have_maps_xs = true;
    for (int b = 0; b < 3 && h->have_maps_xs; ++b)
      if (!(make_tensor_map(h, b, false, h->maps_xs.ld[b], 1) &&
            make_tensor_map(h, b, true, h->maps_xs.st[b], 1)))
        h->have_maps_xs = false;
    if (h->have_maps_xs) {
      // warp groups of a strided sweep: 32 columns x 3 cells each; the
      // streaming twin works while fewer than CLB_XS_FRAC of them (default
      // 0.08) were computed
      static const double frac = [] {
        const char* f = getenv("CLB_XS_FRAC");
        return f ? atof(f) : 0.08;
      }();
      const double groups = (double)((h->cells[0] + 31) / 32) * (double)((h->cells[1] + 2) / 3);
      h->xs_thresh = (unsigned long long)(frac * groups);
      // before any strided sweep: the default geometry
      if (cudaMalloc(&h->d_act, sizeof(unsigned long long)) != cudaSuccess ||
          cudaMemsetAsync(h->d_act, 0xff, sizeof(unsigned long long), h->stream) != cudaSuccess)
        h->have_maps_xs = false;
    }
  }
  e = cudaMalloc(&h->d_res, sizeof(Result));
  if (e == cudaSuccess) e = cudaMallocHost(&h->h_res, sizeof(Result));
  if (e == cudaSuccess) e = cudaMemsetAsync(h->d_res, 0, sizeof(Result), h->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
  if (e != cudaSuccess) {
    int r = cuda_fail(nullptr, e, "result buffers");
    clb_destroy(h);
    return r;
  }
  *out = h;
  return CLB_OK;
}

int clb_destroy(clb_handle h) {
  if (!h) return CLB_OK;
  cudaSetDevice(h->d.device);
  if (h->stream) cudaStreamSynchronize(h->stream);
  for (auto& tl : h->launches) { cudaEventDestroy(tl.a); cudaEventDestroy(tl.b); }
  for (auto e : h->event_pool) cudaEventDestroy(e);
  for (int i = 0; i < 3; ++i)
    if (h->buf[i]) cudaFree(h->buf[i]);
  if (h->d_res) cudaFree(h->d_res);
  if (h->d_act) cudaFree(h->d_act);
  if (h->h_res) cudaFreeHost(h->h_res);
  if (h->batch_exec) cudaGraphExecDestroy(h->batch_exec);
  if (h->batch_graph) cudaGraphDestroy(h->batch_graph);
  if (h->d_ctl) cudaFree(h->d_ctl);
  if (h->h_ctl) cudaFreeHost(h->h_ctl);
  if (h->d_log) cudaFree(h->d_log);
  if (h->comm) nccl().CommDestroy(h->comm);
  if (h->halo_stage) cudaFree(h->halo_stage);
  if (h->side) cudaStreamDestroy(h->side);
  if (h->ev_fork) cudaEventDestroy(h->ev_fork);
  if (h->ev_join) cudaEventDestroy(h->ev_join);
  if (h->own_stream) cudaStreamDestroy(h->own_stream);
  delete h;
  return CLB_OK;
}

int clb_set_stream(clb_handle h, void* s) {
  if (!h) return fail(nullptr, CLB_EINVAL, "null handle");
  h->stream = s ? (cudaStream_t)s : h->own_stream;
  return CLB_OK;
}

static void drop_batch_graph(clb_ctx* h) {
  if (h->batch_exec) cudaGraphExecDestroy(h->batch_exec);
  if (h->batch_graph) cudaGraphDestroy(h->batch_graph);
  h->batch_exec = nullptr;
  h->batch_graph = nullptr;
}

int clb_set_segments(clb_handle h, int axis, int seg_len) {
  if (!h || axis < 0 || axis > 2 || seg_len < 0) return fail(h, CLB_EINVAL, "bad segment override");
  h->seg_override[axis] = seg_len;
  drop_batch_graph(h);
  return CLB_OK;
}

int clb_set_x_variant(clb_handle h, int variant) {
  if (!h) return fail(nullptr, CLB_EINVAL, "null handle");
  if (variant < CLB_XVAR_AUTO || variant > CLB_XVAR_TMA_ADAPT)
    return fail(h, CLB_EINVAL, "unknown x-sweep variant");
  if (variant == CLB_XVAR_TMA && !h->have_maps)
    return fail(h, CLB_EUNSUPPORTED, "TMA tensor maps unavailable on this device");
  if ((variant == CLB_XVAR_TMA_STREAM || variant == CLB_XVAR_TMA_ADAPT) && !h->have_maps_xs)
    return fail(h, CLB_EUNSUPPORTED,
                "the streaming x geometry exists for fp64 2-D shallow water only");
  h->x_variant = variant;
  drop_batch_graph(h);
  return CLB_OK;
}

int clb_x_variant(clb_handle h, int32_t* variant) {
  if (!h || !variant) return fail(h, CLB_EINVAL, "null argument");
  *variant = x_mode(h);
  return CLB_OK;
}

int clb_x_activity(clb_handle h, uint64_t* computed, uint64_t* threshold) {
  if (!h || !computed || !threshold) return fail(h, CLB_EINVAL, "null argument");
  if (x_mode(h) != CLB_XVAR_TMA_ADAPT)
    return fail(h, CLB_EUNSUPPORTED, "the handle does not run the x geometry pair");
  cudaSetDevice(h->d.device);
  unsigned long long v = 0;
  CLB_CUDA(h, cudaMemcpyAsync(&v, h->d_act, sizeof(v), cudaMemcpyDeviceToHost, h->stream));
  CLB_CUDA(h, cudaStreamSynchronize(h->stream));
  *computed = (uint64_t)v;
  *threshold = (uint64_t)h->xs_thresh;
  return CLB_OK;
}

// Pitched 3-D copy of one state between host (dense) and device (pitched).
static cudaError_t copy_state(clb_ctx* h, int buf, int k, void* host, bool padded, bool to_dev) {
  const int64_t isz = h->itemsize;
  const int64_t g = padded ? 2 : 0;
  const int64_t wx = h->cells[0] + 2 * g;
  const int64_t wy = h->ndim >= 2 ? h->cells[1] + 2 * g : 1;
  const int64_t wz = h->ndim == 3 ? h->cells[2] + 2 * g : 1;
  // device element offset of the copied box's first element
  int64_t off = (int64_t)k * h->sstride + h->origin - g;
  if (h->ndim >= 2) off -= g * h->ystride;
  if (h->ndim == 3) off -= g * h->zstride;
  char* dev = (char*)h->buf[buf] + off * isz;
  char* hst = (char*)host + (size_t)k * wx * wy * wz * isz;
  cudaMemcpy3DParms p;
  std::memset(&p, 0, sizeof(p));
  cudaPitchedPtr dp = make_cudaPitchedPtr(dev, (size_t)h->px * isz, (size_t)wx * isz, (size_t)h->ypad);
  cudaPitchedPtr hp = make_cudaPitchedPtr(hst, (size_t)wx * isz, (size_t)wx * isz, (size_t)wy);
  p.srcPtr = to_dev ? hp : dp;
  p.dstPtr = to_dev ? dp : hp;
  p.extent = make_cudaExtent((size_t)wx * isz, (size_t)wy, (size_t)wz);
  p.kind = to_dev ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost;
  return cudaMemcpy3DAsync(&p, h->stream);
}

static int transfer(clb_ctx* h, int buf, void* host, size_t nbytes, bool padded, bool to_dev) {
  if (!h || !host) return fail(h, CLB_EINVAL, "null argument");
  if (buf < 0 || buf > 2) return fail(h, CLB_EINVAL, "buffer index out of range");
  const int64_t g = padded ? 4 : 0;
  size_t want = (size_t)h->M * h->itemsize * (size_t)(h->cells[0] + g);
  if (h->ndim >= 2) want *= (size_t)(h->cells[1] + g);
  if (h->ndim == 3) want *= (size_t)(h->cells[2] + g);
  if (nbytes != want) return fail(h, CLB_EINVAL, "byte count does not match the grid");
  cudaSetDevice(h->d.device);
  for (int k = 0; k < h->M; ++k) {
    cudaError_t e = copy_state(h, buf, k, host, padded, to_dev);
    if (e != cudaSuccess) return cuda_fail(h, e, "cudaMemcpy3DAsync");
  }
  CLB_CUDA(h, cudaStreamSynchronize(h->stream));
  return CLB_OK;
}

int clb_upload(clb_handle h, int buf, const void* src, size_t nbytes) {
  return transfer(h, buf, const_cast<void*>(src), nbytes, false, true);
}
int clb_download(clb_handle h, int buf, void* dst, size_t nbytes) {
  return transfer(h, buf, dst, nbytes, false, false);
}
// frames.py:1-18 CLAWFRM1 header: magic, u32 version, u32 ndim, u32 dims[ndim]
// (x first), u32 num_states, u32 precision, f64 time, u64 step; little-endian,
// no padding.  The payload is exactly clb_download's interior order.
static size_t frame_header_size(const clb_ctx* h) { return 8 + 4 + 4 + 4 * h->ndim + 4 + 4 + 8 + 8; }

int clb_frame_size(clb_handle h, size_t* nbytes) {
  if (!h || !nbytes) return fail(h, CLB_EINVAL, "null argument");
  size_t payload = (size_t)h->M * h->itemsize;
  for (int ax = 0; ax < h->ndim; ++ax) payload *= (size_t)h->cells[ax];
  *nbytes = frame_header_size(h) + payload;
  return CLB_OK;
}

int clb_write_frame(clb_handle h, int buf, double time, uint64_t step, void* out, size_t nbytes) {
  if (!h || !out) return fail(h, CLB_EINVAL, "null argument");
  size_t want = 0;
  clb_frame_size(h, &want);
  if (nbytes != want) return fail(h, CLB_EINVAL, "byte count does not match the frame size");
  unsigned char* p = (unsigned char*)out;
  auto put = [&p](const void* v, size_t n) { std::memcpy(p, v, n); p += n; };
  static_assert(sizeof(double) == 8, "f64");
  put("CLAWFRM1", 8);
  const uint32_t version = 1, ndim = (uint32_t)h->ndim;
  put(&version, 4);
  put(&ndim, 4);
  for (int ax = 0; ax < h->ndim; ++ax) {
    const uint32_t d = (uint32_t)h->cells[ax];
    put(&d, 4);
  }
  const uint32_t m = (uint32_t)h->M, isz = (uint32_t)h->itemsize;
  put(&m, 4);
  put(&isz, 4);
  put(&time, 8);
  put(&step, 8);
  return transfer(h, buf, p, nbytes - frame_header_size(h), false, false);
}

int clb_upload_padded(clb_handle h, int buf, const void* src, size_t nbytes) {
  return transfer(h, buf, const_cast<void*>(src), nbytes, true, true);
}
int clb_download_padded(clb_handle h, int buf, void* dst, size_t nbytes) {
  return transfer(h, buf, dst, nbytes, true, false);
}

int clb_sweep_async(clb_handle h, int axis, double dt, int src, int dst, int slot, int literal) {
  if (!h) return fail(nullptr, CLB_EINVAL, "null handle");
  return launch_sweep(h, axis, dt, src, dst, slot, literal != 0);
}

int clb_sweep_segments(clb_handle h, int axis, int32_t* nseg, int32_t* seg_len) {
  if (!h || !nseg || !seg_len) return fail(h, CLB_EINVAL, "null argument");
  if (axis < 0 || axis >= h->ndim) return fail(h, CLB_EINVAL, "sweep axis out of range");
  const clb::GenericArgs g = sweep_geometry(h, axis, 0, 1);
  *nseg = g.nseg;
  *seg_len = g.seg_len;
  return CLB_OK;
}

int clb_sweep_async_range(clb_handle h, int axis, double dt, int src, int dst, int slot,
                          int literal, int seg_begin, int seg_end) {
  if (!h) return fail(nullptr, CLB_EINVAL, "null handle");
  return launch_sweep(h, axis, dt, src, dst, slot, literal != 0, false, seg_begin, seg_end);
}

int clb_fetch(clb_handle h, int nslots, double* speeds, int32_t* nonfinite) {
  if (!h) return fail(nullptr, CLB_EINVAL, "null handle");
  return fetch(h, nslots, speeds, nonfinite);
}

int clb_sweep(clb_handle h, int axis, double dt, int src, int dst, double* speed,
              int32_t* nonfinite) {
  if (!h) return fail(nullptr, CLB_EINVAL, "null handle");
  int r = launch_sweep(h, axis, dt, src, dst, 0, false);
  if (r) return r;
  return fetch(h, 1, speed, nonfinite);
}

int clb_attempt_step(clb_handle h, double dt, int src, int s0, int s1, double* speeds,
                     int32_t* nonfinite) {
  if (!h) return fail(nullptr, CLB_EINVAL, "null handle");
  if (src == s0 || src == s1 || s0 == s1) return fail(h, CLB_EINVAL, "step buffers must be distinct");
  int cur = src;
  for (int j = 0; j < h->ndim; ++j) {
    const int dst = (j % 2 == 0) ? s0 : s1;
    int r = attempt_sweep(h, j, dt, cur, dst, j, false, false);
    if (r) return r;
    cur = dst;
  }
  if (h->comm) {
    const int r = results_allreduce(h, h->stream);
    if (r) return r;
  }
  return fetch(h, h->ndim, speeds, nonfinite);
}

int clb_first_nonfinite(clb_handle h, int buf, int32_t* found, int32_t* state, int64_t cell[3]) {
  if (!h || !found || !state || !cell) return fail(h, CLB_EINVAL, "null argument");
  if (buf < 0 || buf > 2) return fail(h, CLB_EINVAL, "buffer index out of range");
  cudaSetDevice(h->d.device);
  unsigned long long* slot = &h->d_res->first_bad;
  CLB_CUDA(h, cudaMemsetAsync(slot, 0xff, sizeof(unsigned long long), h->stream));
  const int64_t total = (int64_t)h->M * h->cells[0] * h->cells[1] * h->cells[2];
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, (int64_t)h->num_sms * 16);
  const char* base = (const char*)h->buf[buf] + h->origin * h->itemsize;
  if (h->itemsize == 8)
    first_bad_kernel<double><<<blocks, 256, 0, h->stream>>>(
        (const double*)base, h->sstride, h->ystride, h->zstride, h->cells[0], h->cells[1],
        h->cells[2], h->M, slot);
  else
    first_bad_kernel<float><<<blocks, 256, 0, h->stream>>>(
        (const float*)base, h->sstride, h->ystride, h->zstride, h->cells[0], h->cells[1],
        h->cells[2], h->M, slot);
  CLB_CUDA(h, cudaGetLastError());
  unsigned long long idx = 0;
  CLB_CUDA(h, cudaMemcpyAsync(&idx, slot, sizeof(idx), cudaMemcpyDeviceToHost, h->stream));
  CLB_CUDA(h, cudaStreamSynchronize(h->stream));
  if (idx == ~0ull) {
    *found = 0;
    return CLB_OK;
  }
  *found = 1;
  int64_t r = (int64_t)idx;
  cell[0] = r % h->cells[0]; r /= h->cells[0];
  cell[1] = r % h->cells[1]; r /= h->cells[1];
  cell[2] = r % h->cells[2]; r /= h->cells[2];
  *state = (int32_t)r;
  return CLB_OK;
}

int clb_halo_layout(clb_handle h, int buf, int side, void** send_ptr, void** recv_ptr,
                    size_t* block_bytes, size_t* state_stride_bytes) {
  if (!h) return fail(nullptr, CLB_EINVAL, "null handle");
  if (h->ndim < 2) return fail(h, CLB_EUNSUPPORTED, "halo exchange needs ndim >= 2");
  if (buf < 0 || buf > 2 || side < 0 || side > 1) return fail(h, CLB_EINVAL, "bad buffer/side");
  const int64_t slab = h->ndim == 2 ? h->ystride : h->zstride;  // one row / plane
  const int64_t n = h->cells[h->ndim - 1];
  if (n < 2) return fail(h, CLB_EUNSUPPORTED, "halo exchange needs at least 2 owned rows/planes");
  // first element of owned row/plane 0 (x and y ghosts included)
  int64_t first = h->origin - h->xoff;
  if (h->ndim == 3) first -= 2 * h->ystride;
  char* base = (char*)h->buf[buf] + first * h->itemsize;
  const int64_t isz = h->itemsize;
  if (side == 0) {
    *send_ptr = base;
    *recv_ptr = base - 2 * slab * isz;
  } else {
    *send_ptr = base + (n - 2) * slab * isz;
    *recv_ptr = base + n * slab * isz;
  }
  *block_bytes = (size_t)(2 * slab * isz);
  *state_stride_bytes = (size_t)(h->sstride * isz);
  return CLB_OK;
}

int clb_solve_pairs(clb_handle h, int axis, int64_t n, const void* ql, const void* qr, void* W,
                    void* s) {
  if (!h) return fail(nullptr, CLB_EINVAL, "null handle");
  if (axis < 0 || axis >= h->ndim || n < 0) return fail(h, CLB_EINVAL, "bad axis or count");
  if (n == 0) return CLB_OK;
  cudaSetDevice(h->d.device);
  const UserSolver* us = user_solver(h->d.solver_id);
  const int nw = us ? us->nw
                 : h->d.solver_id == CLB_SOLVER_SHALLOW_WATER ? 3
                 : (h->d.solver_id == CLB_SOLVER_ADVECTION ? 1 : 2);
  const size_t qb = (size_t)n * h->M * h->itemsize;
  const size_t wb = (size_t)n * nw * h->M * h->itemsize;
  const size_t sb = (size_t)n * nw * h->itemsize;
  char* d = nullptr;
  CLB_CUDA(h, cudaMalloc(&d, 2 * qb + wb + sb));
  cudaError_t e = cudaMemcpyAsync(d, ql, qb, cudaMemcpyHostToDevice, h->stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(d + qb, qr, qb, cudaMemcpyHostToDevice, h->stream);
  if (e == cudaSuccess) {
    if (us) {
      clb_user_pairs_fn fn = us->pairs[h->itemsize == 8 ? 1 : 0];
      e = fn ? (cudaError_t)fn(h->ndim, axis, d, d + qb, d + 2 * qb, d + 2 * qb + wb, n,
                               h->d.params, (void*)h->stream)
             : cudaErrorInvalidValue;
    } else {
      e = clb::pairs_dispatch(h->d.solver_id, h->itemsize, h->ndim, axis, d, d + qb,
                              d + 2 * qb, d + 2 * qb + wb, n, h->d.params, h->stream);
    }
  }
  if (e == cudaSuccess) e = cudaMemcpyAsync(W, d + 2 * qb, wb, cudaMemcpyDeviceToHost, h->stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(s, d + 2 * qb + wb, sb, cudaMemcpyDeviceToHost, h->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
  cudaFree(d);
  if (e != cudaSuccess) return cuda_fail(h, e, "solve_pairs");
  return CLB_OK;
}

int clb_selftest_arith(int device, int64_t n, const double* a, const double* b, int64_t out[12]) {
  if (!a || !b || !out || n < 0) return fail(nullptr, CLB_EINVAL, "null argument");
  for (int i = 0; i < 12; ++i) out[i] = 0;
  if (n == 0) return CLB_OK;
  if (cudaSetDevice(device) != cudaSuccess) return fail(nullptr, CLB_ECUDA, "no such device");
  double* d = nullptr;
  unsigned long long* cnt = nullptr;
  const size_t nb = (size_t)n * sizeof(double);
  cudaError_t e = cudaMalloc(&d, 2 * nb);
  if (e == cudaSuccess) e = cudaMalloc(&cnt, 12 * sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaMemset(cnt, 0, 12 * sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaMemcpy(d, a, nb, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(d + n, b, nb, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) {
    selftest_arith_kernel<<<(unsigned)((n + 255) / 256), 256>>>(d, d + n, n, cnt);
    e = cudaGetLastError();
  }
  unsigned long long h[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  if (e == cudaSuccess) e = cudaMemcpy(h, cnt, sizeof(h), cudaMemcpyDeviceToHost);
  cudaFree(d);
  cudaFree(cnt);
  if (e != cudaSuccess) return fail(nullptr, CLB_ECUDA, cudaGetErrorString(e));
  for (int i = 0; i < 12; ++i) out[i] = (int64_t)h[i];
  return CLB_OK;
}

int clb_enable_timing(clb_handle h, int on) {
  if (!h) return fail(nullptr, CLB_EINVAL, "null handle");
  h->timing = on != 0;
  return CLB_OK;
}

int clb_timing(clb_handle h, double ms[3], int64_t count[3]) {
  if (!h) return fail(nullptr, CLB_EINVAL, "null handle");
  for (int i = 0; i < 3; ++i) { ms[i] = 0.0; count[i] = 0; }
  CLB_CUDA(h, cudaStreamSynchronize(h->stream));
  for (auto& tl : h->launches) {
    float v = 0.f;
    cudaEventElapsedTime(&v, tl.a, tl.b);
    ms[tl.axis] += v;
    count[tl.axis] += tl.counts;
    h->event_pool.push_back(tl.a);
    h->event_pool.push_back(tl.b);
  }
  h->launches.clear();
  return CLB_OK;
}

void* clb_host_alloc(size_t nbytes) {
  void* p = nullptr;
  if (cudaMallocHost(&p, nbytes) != cudaSuccess) return nullptr;
  return p;
}

void clb_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

int clb_memory_info(clb_handle h, size_t* device_bytes, int64_t* row_pitch) {
  if (!h) return fail(nullptr, CLB_EINVAL, "null handle");
  if (device_bytes) *device_bytes = 3 * h->buf_bytes;
  if (row_pitch) *row_pitch = h->px;
  return CLB_OK;
}

}  // extern "C"

namespace clb {

cudaError_t pairs_dispatch(int solver, int itemsize, int ndim, int axis, const void* ql,
                           const void* qr, void* W, void* s, int64_t n, const double* p,
                           cudaStream_t st) {
  const bool d = itemsize == 8;
  switch (solver) {
    case CLB_SOLVER_ACOUSTICS:
      return d ? pairs_acoustics_f64(ndim, axis, ql, qr, W, s, n, p, st)
               : pairs_acoustics_f32(ndim, axis, ql, qr, W, s, n, p, st);
    case CLB_SOLVER_SHALLOW_WATER:
      return d ? pairs_shallow_water_f64(ndim, axis, ql, qr, W, s, n, p, st)
               : pairs_shallow_water_f32(ndim, axis, ql, qr, W, s, n, p, st);
    case CLB_SOLVER_ADVECTION:
      return d ? pairs_advection_f64(ndim, axis, ql, qr, W, s, n, p, st)
               : pairs_advection_f32(ndim, axis, ql, qr, W, s, n, p, st);
    default:
      return d ? pairs_vc_acoustics_f64(ndim, axis, ql, qr, W, s, n, p, st)
               : pairs_vc_acoustics_f32(ndim, axis, ql, qr, W, s, n, p, st);
  }
}

}  // namespace clb

extern "C" int clb_set_boundary(clb_handle h, int axis, int lo, int hi) {
  if (!h) return fail(nullptr, CLB_EINVAL, "null handle");
  if (axis < 0 || axis >= h->ndim) return fail(h, CLB_EINVAL, "axis out of range");
  for (int bc : {lo, hi}) {
    if (bc < 0 || bc > 3) return fail(h, CLB_EINVAL, "unknown boundary kind");
    if ((bc == CLB_BC_PERIODIC || bc == CLB_BC_REFLECTIVE) && h->cells[axis] < 2)
      return fail(h, CLB_EUNSUPPORTED, "periodic/reflective boundaries need at least 2 cells");
    if (bc == CLB_BC_REFLECTIVE && (h->d.normal_velocity[axis] < 0 ||
                                    h->d.normal_velocity[axis] >= h->M))
      return fail(h, CLB_EINVAL, "reflective boundary needs a normal velocity state");
  }
  if ((lo == CLB_BC_PERIODIC) != (hi == CLB_BC_PERIODIC))
    return fail(h, CLB_EINVAL, "periodic boundary must be set on both sides");
  h->d.bc[axis][0] = lo;
  h->d.bc[axis][1] = hi;
  if (h->batch_exec) cudaGraphExecDestroy(h->batch_exec);
  if (h->batch_graph) cudaGraphDestroy(h->batch_graph);
  h->batch_exec = nullptr;
  h->batch_graph = nullptr;
  return CLB_OK;
}

extern "C" int clb_halo_copy(clb_handle h, int buf, int side, int to_host, void* host) {
  if (!h || !host) return fail(h, CLB_EINVAL, "null argument");
  void *send = nullptr, *recv = nullptr;
  size_t bb = 0, ss = 0;
  int r = clb_halo_layout(h, buf, side, &send, &recv, &bb, &ss);
  if (r) return r;
  cudaSetDevice(h->d.device);
  for (int k = 0; k < h->M; ++k) {
    char* hp = (char*)host + (size_t)k * bb;
    if (to_host)
      CLB_CUDA(h, cudaMemcpyAsync(hp, (char*)send + k * ss, bb, cudaMemcpyDeviceToHost, h->stream));
    else
      CLB_CUDA(h, cudaMemcpyAsync((char*)recv + k * ss, hp, bb, cudaMemcpyHostToDevice, h->stream));
  }
  CLB_CUDA(h, cudaStreamSynchronize(h->stream));
  return CLB_OK;
}

namespace {

// One attempt as a graph: ndim indirect sweeps + the controller.
int build_batch_graph(clb_ctx* h) {
  // configure every kernel outside capture: no-op launches (done = 1)
  h->h_ctl->done = 1;
  CLB_CUDA(h, cudaMemcpyAsync(h->d_ctl, h->h_ctl, sizeof(clb::DevCtl), cudaMemcpyHostToDevice,
                              h->stream));
  for (int j = 0; j < h->ndim; ++j) {
    const int r = launch_sweep(h, j, 1.0, 0, 1, j, false, true);
    if (r) return r;
  }
  CLB_CUDA(h, cudaStreamSynchronize(h->stream));
  CLB_CUDA(h, cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
  // one-thread controller kernel per attempt; CLB_FUSED_CTL=1 folds it into
  // the last CTA of the attempt's final sweep instead, which measured slower
  // (C2 e2e 6.73 vs 7.15, C1 1.91 vs 2.11 Gcell-upd/s: the per-CTA fence and
  // counter and the serial tail cost more than the saved graph node)
  static const bool fused = [] {
    const char* e = getenv("CLB_FUSED_CTL");
    return e && e[0] == '1';
  }();
  int r = 0;
  if (h->comm) {
    // slab: halo exchange inside the slow sweep, max-allreduce of the
    // results before the controller (no host round trip per attempt)
    for (int j = 0; j < h->ndim && !r; ++j) r = attempt_sweep(h, j, 1.0, 0, 1, j, false, true);
    if (!r) r = results_allreduce(h, h->stream);
    if (!r) clb::ctl_finish<<<1, 1, 0, h->stream>>>(h->d_ctl, h->d_res);
  } else {
    for (int j = 0; j < h->ndim && !r; ++j)
      r = launch_sweep(h, j, 1.0, 0, 1, j, false, true, 0, -1, fused && j == h->ndim - 1);
    if (!r && !fused) clb::ctl_finish<<<1, 1, 0, h->stream>>>(h->d_ctl, h->d_res);
  }
  cudaGraph_t g = nullptr;
  cudaError_t e = cudaStreamEndCapture(h->stream, &g);
  if (r) { if (g) cudaGraphDestroy(g); return r; }
  if (e != cudaSuccess) return cuda_fail(h, e, "batch graph capture");
  h->batch_graph = g;
  CLB_CUDA(h, cudaGraphInstantiate(&h->batch_exec, g, 0));
  return CLB_OK;
}

}  // namespace

extern "C" int clb_run_batch(clb_handle h, clb_batch* b, clb_attempt* log, int64_t log_cap) {
  if (!h || !b || (!log && log_cap > 0)) return fail(h, CLB_EINVAL, "null argument");
  if (log_cap < 1) return fail(h, CLB_EINVAL, "log_cap must be positive");
  const int roles[3] = {b->cur, b->scratch0, b->scratch1};
  for (int i = 0; i < 3; ++i)
    if (roles[i] < 0 || roles[i] > 2) return fail(h, CLB_EINVAL, "buffer index out of range");
  if (b->cur == b->scratch0 || b->cur == b->scratch1 || b->scratch0 == b->scratch1)
    return fail(h, CLB_EINVAL, "step buffers must be distinct");
  CLB_CUDA(h, cudaSetDevice(h->d.device));
  if (!h->d_ctl) {
    CLB_CUDA(h, cudaMalloc(&h->d_ctl, sizeof(clb::DevCtl)));
    CLB_CUDA(h, cudaMallocHost(&h->h_ctl, sizeof(clb::DevCtl)));
  }
  if (h->log_cap < log_cap) {
    if (h->d_log) cudaFree(h->d_log);
    h->d_log = nullptr;
    h->log_cap = 0;
    CLB_CUDA(h, cudaMalloc(&h->d_log, (size_t)log_cap * sizeof(clb_attempt)));
    h->log_cap = log_cap;
  }
  if (!h->batch_exec) {
    const int r = build_batch_graph(h);
    if (r) return r;
  }
  clb::DevCtl& c = *h->h_ctl;
  std::memset(&c, 0, sizeof(c));
  c.t = b->t;
  c.last_max_speed = b->last_max_speed;
  c.prev_nu = b->prev_nu;
  c.nu_max = b->nu_max;
  c.prev_reverted = b->prev_reverted ? 1 : 0;
  c.cur = b->cur;
  c.s0 = b->scratch0;
  c.s1 = b->scratch1;
  c.stop = b->stop;
  c.cfl_target = b->cfl_target;
  c.cfl_max = b->cfl_max;
  c.dt_cap = b->dt_cap;
  c.min_spacing = b->min_spacing;
  c.max_accepted = b->max_accepted;
  c.log_cap = log_cap;
  c.ndim = h->ndim;
  c.status = -1;
  c.fail_sweep = -1;
  c.log = h->d_log;
  CLB_CUDA(h, cudaMemcpyAsync(h->d_ctl, h->h_ctl, sizeof(clb::DevCtl), cudaMemcpyHostToDevice,
                              h->stream));
  CLB_CUDA(h, cudaMemsetAsync(h->d_res, 0, sizeof(Result), h->stream));
  clb::ctl_prepare<<<1, 1, 0, h->stream>>>(h->d_ctl);
  CLB_CUDA(h, cudaGetLastError());
  // Replay attempts in chunks; the host only polls the done flag between
  // chunks (attempts replayed past the end are no-ops).  A step budget sizes
  // the first chunk exactly.
  static const int64_t chunk_cap = [] {
    const char* e = getenv("CLB_BATCH_CHUNK");
    return e ? std::max<int64_t>(1, atoll(e)) : (int64_t)256;
  }();
  int64_t chunk = b->max_accepted >= 0 ? std::max<int64_t>(1, std::min<int64_t>(b->max_accepted, chunk_cap))
                                       : std::min<int64_t>(8, chunk_cap);
  for (;;) {
    for (int64_t i = 0; i < chunk; ++i) CLB_CUDA(h, cudaGraphLaunch(h->batch_exec, h->stream));
    CLB_CUDA(h, cudaMemcpyAsync(h->h_ctl, h->d_ctl, sizeof(clb::DevCtl), cudaMemcpyDeviceToHost,
                                h->stream));
    CLB_CUDA(h, cudaStreamSynchronize(h->stream));
    if (c.done) break;
    chunk = std::min<int64_t>(std::min<int64_t>(2 * chunk, 64), chunk_cap);
  }
  if (c.n_attempts > 0)
    CLB_CUDA(h, cudaMemcpy(log, h->d_log, (size_t)c.n_attempts * sizeof(clb_attempt),
                           cudaMemcpyDeviceToHost));
  b->t = c.t;
  b->last_max_speed = c.last_max_speed;
  b->prev_nu = c.prev_nu;
  b->nu_max = c.nu_max;
  b->prev_reverted = c.prev_reverted;
  b->cur = c.cur;
  b->scratch0 = c.s0;
  b->scratch1 = c.s1;
  b->n_attempts = c.n_attempts;
  b->n_accepted = c.n_accepted;
  b->status = c.status;
  b->fail_sweep = c.fail_sweep;
  b->fail_dt = c.dt;
  return CLB_OK;
}

extern "C" int clb_nccl_unique_id(void* id_out) {
  if (!id_out) return fail(nullptr, CLB_EINVAL, "null argument");
  const NcclApi& n = nccl();
  if (!n.ok) return fail(nullptr, CLB_EUNSUPPORTED, "NCCL unavailable: " + n.err);
  ncclUniqueId id;
  const ncclResult_t r = n.GetUniqueId(&id);
  if (r != ncclSuccess) return nccl_fail(nullptr, r, "ncclGetUniqueId");
  std::memcpy(id_out, &id, sizeof(id));
  return CLB_OK;
}

extern "C" int clb_attach_comm(clb_handle h, const void* id, int nranks, int rank, int lo_nbr,
                               int hi_nbr) {
  if (!h || !id) return fail(h, CLB_EINVAL, "null argument");
  if (h->ndim < 2) return fail(h, CLB_EUNSUPPORTED, "slab exchange needs ndim >= 2");
  if (h->comm) return fail(h, CLB_EINVAL, "a communicator is already attached");
  if (nranks < 1 || rank < 0 || rank >= nranks || lo_nbr < -1 || lo_nbr >= nranks ||
      hi_nbr < -1 || hi_nbr >= nranks)
    return fail(h, CLB_EINVAL, "bad rank / neighbour");
  const int slow = h->ndim - 1;
  if ((lo_nbr >= 0 && h->d.bc[slow][0] != CLB_BC_HALO) ||
      (hi_nbr >= 0 && h->d.bc[slow][1] != CLB_BC_HALO))
    return fail(h, CLB_EINVAL, "a side with a neighbour must be a CLB_BC_HALO side");
  const NcclApi& n = nccl();
  if (!n.ok) return fail(h, CLB_EUNSUPPORTED, "NCCL unavailable: " + n.err);
  CLB_CUDA(h, cudaSetDevice(h->d.device));
  void *send_lo, *recv_lo, *send_hi, *recv_hi;
  size_t bb = 0, ss = 0;
  int r = clb_halo_layout(h, 0, 0, &send_lo, &recv_lo, &bb, &ss);
  if (!r) r = clb_halo_layout(h, 0, 1, &send_hi, &recv_hi, &bb, &ss);
  if (r) return r;
  const char* b0 = (const char*)h->buf[0];
  h->halo_send_off[0] = (const char*)send_lo - b0;
  h->halo_send_off[1] = (const char*)send_hi - b0;
  h->halo_recv_off[0] = (const char*)recv_lo - b0;
  h->halo_recv_off[1] = (const char*)recv_hi - b0;
  h->halo_block = bb;
  // (a failed earlier attach may have left these behind)
  if (!h->halo_stage) CLB_CUDA(h, cudaMalloc(&h->halo_stage, 4 * (size_t)h->M * bb));
  if (!h->side) CLB_CUDA(h, cudaStreamCreateWithFlags(&h->side, cudaStreamNonBlocking));
  if (!h->ev_fork) CLB_CUDA(h, cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming));
  if (!h->ev_join) CLB_CUDA(h, cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming));
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  ncclComm_t comm = nullptr;
  const ncclResult_t nr = n.CommInitRank(&comm, nranks, uid, rank);
  if (nr != ncclSuccess) return nccl_fail(h, nr, "ncclCommInitRank");
  h->comm = comm;
  h->nranks = nranks;
  h->rank = rank;
  h->nbr[0] = lo_nbr;
  h->nbr[1] = hi_nbr;
  drop_batch_graph(h);
  return CLB_OK;
}

extern "C" int clb_halo_exchange(clb_handle h, int buf) {
  if (!h) return fail(nullptr, CLB_EINVAL, "null handle");
  if (!h->comm) return fail(h, CLB_EINVAL, "no communicator attached");
  if (buf < 0 || buf > 2) return fail(h, CLB_EINVAL, "buffer index out of range");
  cudaSetDevice(h->d.device);
  return halo_exchange_on(h, h->stream, buf, false);
}

extern "C" int clb_results_allreduce(clb_handle h) {
  if (!h) return fail(nullptr, CLB_EINVAL, "null handle");
  if (!h->comm) return CLB_OK;
  cudaSetDevice(h->d.device);
  return results_allreduce(h, h->stream);
}
