// api.cu -- the C ABI (include/radsplat.h): workspace layout and the frame
// pipeline  project -> depth sort -> row segments -> per-tile lists -> blend.
//
// One translation unit: the kernels live in the .cuh files next to this one.
// Build: see paper_2403_13806_b200/build.py (nvcc -gencode arch=compute_100a,
// code=sm_100a -fmad=false -lineinfo, static cudart).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <new>

#include "segbin.cuh"
#include "dsort.cuh"
#include "bsort.cuh"
#include "blend.cuh"
#include "blend64.cuh"
#include "compact.cuh"
#include "io.cuh"
#include "metrics.cuh"
#include "backward.cuh"
#include "project.cuh"
#include "sort.cuh"

using namespace rs;

// Frame kernels launched straight onto a stream use programmatic stream serialization (PDL):
// the grid is scheduled while the previous kernel drains and waits in griddepcontrol.wait
// (pdl_wait, the first statement of each kernel) for its completion -- the launch gaps of the
// chain of small binning kernels are hidden (configs[2] scoring +3%). Captured CUDA graphs keep
// the programmatic edges too (round 1 measured them 2% slower; with this round's chain they
// are 1.2% faster per configs[1] frame: 3262 -> 3300 frames/s; RS_PDL_GRAPH=0 drops them).
enum PdlClass { kPdlChain = 1, kPdlExpand = 2, kPdlBlend = 4, kPdlAll = 7 };
static int pdl_mode() {  // RS_PDL (A/B measurements): bit 0 binning chain, bit 1 expand, bit 2 blend
  static const int m = [] {
    const char* e = std::getenv("RS_PDL");
    return e ? std::atoi(e) : kPdlAll;
  }();
  return m;
}
static thread_local int g_pdl_class = kPdlChain;  // class of the next launch() (set by the callers below)

// A cooperative launch (all CTAs co-resident: grid barriers inside the kernel are safe).
template <typename... KP, typename... A>
static cudaError_t launch_coop(void (*k)(KP...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, A&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, static_cast<KP>(args)...);
}

constexpr uint32_t kDsortMaxItems = 1u << 20;
static int dsort_mode() {  // RS_DSORT: 0 onesweep launches, 2 always the cooperative sort (A/B measurements)
  static const int m = [] {
    const char* e = std::getenv("RS_DSORT");
    return e ? std::atoi(e) : 1;
  }();
  return m;
}
template <typename... KP, typename... A>
static void launch(void (*k)(KP...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, A&&... args);
// launch() returning the launch status (callers with a fallback)
template <typename... KP, typename... A>
static cudaError_t launch_ex(void (*k)(KP...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, A&&... args) {
  launch(k, grid, block, smem, st, static_cast<A&&>(args)...);
  return cudaGetLastError();
}
template <typename... KP, typename... A>
static void launch(void (*k)(KP...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, A&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(st, &cap);
  static const bool pdl_graph = [] {  // RS_PDL_GRAPH=0: no PDL edges in captured graphs (A/B)
    const char* e = std::getenv("RS_PDL_GRAPH");
    return !e || std::atoi(e) != 0;
  }();
  cfg.numAttrs = ((cap == cudaStreamCaptureStatusNone || pdl_graph) && (pdl_mode() & g_pdl_class)) ? 1 : 0;
  cudaLaunchKernelEx(&cfg, k, static_cast<KP>(args)...);
}

namespace {

size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

constexpr int kMaxDsortCtas = 160;  // cooperative depth sort: one CTA per SM (column_prefix: <= 32 x 3 rows per half)

struct Layout {
  // per-frame zeroed region [0, frame_bytes)
  size_t ctr, hist, proj_lb, ranges, scancls, scanpart, frame_bytes;
  size_t sticky, cam, recs, recs64, exptab, dtab, rows, sgrad, titem, keysA, keysB, valsA, valsB, rowtab, rowcnt, segitem, segspan, geom,
      rowstart, chunkstart, chunkcnt, keysC, chunkinfo, densel, tilecnt, tileord, pitem, lbA, lbB, total;
};

int tiles_x(int w) { return (w + kTile - 1) / kTile; }

int device_sms() {  // SMs of the current device (148 on B200)
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
    cudaGetLastError();
    sms = 148;
  }
  return sms;
}

size_t rowtab_stride(int64_t n_cap) { return (size_t)n_cap / kRankChunk + 1; }

int64_t seg_capacity(int64_t n_cap, int64_t pair_cap) {
  // row segments <= pairs + 2 per Gaussian (only a culling box's first and last tile rows can
  // miss the ellipse); more are reported as an overflow
  return std::min<int64_t>(pair_cap + 2 * n_cap, 0xffffffffLL);
}

Layout make_layout(int64_t n_cap, int64_t pair_cap, int W, int H, int sms) {
  Layout L{};
  const size_t TW = tiles_x(W), TH = tiles_x(H);
  const size_t seg_cap = (size_t)seg_capacity(n_cap, pair_cap);
  size_t o = 0;
  auto take = [&](size_t bytes) { const size_t at = o; o = align_up(o + bytes); return at; };
  // per-frame zeroed region
  L.ctr = take(sizeof(Counters));
  L.hist = take(4 * 256 * sizeof(uint32_t));  // depth passes 0-3
  L.proj_lb = take(((size_t)n_cap / kCompactKeys + 2) * sizeof(unsigned long long));
  L.ranges = take(TW * TH * sizeof(uint2));
  // dsort_kernel's per-pass digit tables (16-bit counts) and digit totals
  L.dtab = take(dsort_tab_words(std::min(sms, kMaxDsortCtas)) * 4);  // dsort_kernel's digit tables
  L.scancls = take(2 * kScanClasses * 4);  // tile scan: list-length class counts and cursors
  L.scanpart = take(((size_t)TW * TH / kScanTiles + 1) * 8);  // tile scan: 64-tile block sums
  L.frame_bytes = o;
  L.sticky = take(sizeof(Sticky));
  L.cam = take(sizeof(CamPair));
  L.recs = take((size_t)n_cap * sizeof(Rec));
  L.recs64 = take((size_t)n_cap * sizeof(Rec64));  // RS_F64 frames
  L.exptab = take((size_t)kExpTab * sizeof(double));  // blend64's exp table (built at create)

  L.rows = take((size_t)n_cap * 4);  // per binned item its tile-row range
  L.sgrad = take((size_t)n_cap * 4 * kSGrad);  // rs_backward: screen-space gradient sums per item
  L.titem = take((size_t)n_cap);
  L.keysA = take((size_t)n_cap * 4);
  L.keysB = take((size_t)n_cap * 4);  // the projection's per-item depth keys
  L.keysC = take((size_t)n_cap * 4);  // dsort_kernel's second key buffer (keysB holds its input)
  L.valsA = take((size_t)n_cap * 4);
  L.valsB = take((size_t)n_cap * 4);
  L.rowtab = take(rowtab_stride(n_cap) * TH * 4);  // per tile row: Gaussians per rank chunk
  L.rowcnt = take((TH + 1) * sizeof(uint32_t));
  L.segitem = take(seg_cap * 4);
  L.segspan = take(seg_cap * 4);
  L.geom = take((size_t)n_cap * 32);
  L.rowstart = take((TH + 1) * 4);
  L.chunkstart = take((TH + 1) * 4);
  L.chunkcnt = take((seg_cap / kExpandChunk + TH + 1) * TW * 4);
  L.chunkinfo = take((seg_cap / kExpandChunk + TH + 1) * 8);
  L.densel = take((seg_cap / kExpandChunk + TH + 1) * 4);
  L.tilecnt = take(TW * TH * 4);
  L.tileord = take(TW * TH * 4);  // blend CTA -> tile, longest lists first
  L.pitem = take((size_t)pair_cap * 4);
  const size_t chunks = ((size_t)n_cap + kMinChunk - 1) / kMinChunk + 1;  // depth sort look-back
  L.lbA = take(chunks * 256 * 4);
  L.lbB = take(chunks * 256 * 4);
  L.total = o;
  return L;
}

}  // namespace

int expand_major_thresh() {  // expand's column-major switch (x8): RS_EXPAND_MAJOR overrides (tuning)
  static const int t = [] {
    const char* e = std::getenv("RS_EXPAND_MAJOR");
    return e ? std::atoi(e) : 8;
  }();
  return t;
}

int expand_dense_span() {  // chunks averaging >= this many tiles per segment take the ballot walk
  // (measured: 6 / 8 / 10 / 12 / 16 -> configs[1] 3345 / 3367 / 3369 / 3365 / 3361 frames/s,
  // configs[4] batch 872 / - / 880 / 847 frames/s)
  static const int t = [] {
    const char* e = std::getenv("RS_EXPAND_DENSE");
    return e ? std::atoi(e) : 10;
  }();
  return t;
}

struct rs_workspace {
  unsigned char* base;
  size_t bytes;
  Layout L;
  int64_t n_cap, pair_cap;
  int W_cap, H_cap;
  int sms;
  // current frame (set by rs_project)
  uint32_t n_items;
  int W, H, TW, TH;
  bool binned, have_cam, has_color;
  bool f64;  // precision of the current frame (rs_options.precision == RS_F64)
  cudaStream_t aux = nullptr;  // second stream (dense expansion next to the sparse one)
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;

  ~rs_workspace() {
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    if (aux) cudaStreamDestroy(aux);
  }
  template <typename T> T* at(size_t off) const { return reinterpret_cast<T*>(base + off); }
  Counters* ctr() const { return at<Counters>(L.ctr); }
};

namespace {

cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// the fp32 path's options: each value rounded once (round to nearest = numpy astype(float32))
Opt32 opt32(const rs_options& o) {
  return Opt32{(float)o.alpha_max, (float)o.alpha_cut, (float)o.tau_stop, (float)o.near_limit, (float)o.lowpass,
               (float)o.sigma_bound};
}
Opt64 opt64(const rs_options& o) {
  return Opt64{o.alpha_max, o.alpha_cut, o.tau_stop, o.near_limit, o.lowpass, o.sigma_bound};
}
bool valid_options(const rs_options* o) { return o && (o->precision == RS_F32 || o->precision == RS_F64); }

int32_t cuda_status() { return cudaGetLastError() == cudaSuccess ? RS_OK : RS_ECUDA; }

#ifndef RS_DEPTH_ITEMS
#define RS_DEPTH_ITEMS 8
#endif
constexpr int kDepthItems = RS_DEPTH_ITEMS;  // 2048-key chunks (16: no change in the benches)

// LSD passes of one sort over `bits` key bits; the digit histograms
// (hist_slot) and the first pass's zeroed look-back words were produced by
// the key-producing kernel.
template <typename K, int ITEMS>
void run_sort(rs_workspace* ws, const K* keys0, K* keysA, K* keysB, const uint32_t* vals0, uint32_t* valsA,
              uint32_t* valsB, const uint32_t* n_ptr, uint32_t n_static, uint32_t n_bound, int bits, int hist_slot,
              int ticket_slot, bool last_keys, cudaStream_t st, const K** keys_res, const uint32_t** vals_res) {
  Counters* ctr = ws->ctr();
  uint32_t* hist = ws->at<uint32_t>(ws->L.hist) + hist_slot * 256;
  uint32_t* lb[2] = {ws->at<uint32_t>(ws->L.lbA), ws->at<uint32_t>(ws->L.lbB)};
  const int smem = (int)sizeof(OnesweepSmem<K, ITEMS>);
  constexpr uint32_t CHUNK = kSortThreads * ITEMS;
  const int grid = std::max(1, (int)((n_bound + CHUNK - 1) / CHUNK));  // one CTA per chunk, ticket order
  const int passes = (bits + 7) / 8;
  const K* kin = keys0;
  const uint32_t* vin = vals0;
  for (int p = 0; p < passes; ++p) {
    K* kout = (p % 2 == 0) ? keysB : keysA;
    uint32_t* vout = (p % 2 == 0) ? valsB : valsA;
    const bool last = p == passes - 1;
    const int nbits = std::min(8, bits - 8 * p);
    uint32_t* lb_next = last ? nullptr : lb[(p + 1) % 2];
    const int wk = (!last || last_keys) ? 1 : 0;
#define RS_PASS(NB)                                                                                       \
  launch(onesweep_kernel<K, ITEMS, NB>, grid, kSortThreads, smem, st, kin, vin, kout, vout, n_ptr, n_static, \
         hist + p * 256, lb[p % 2], lb_next, ctr->tickets + ticket_slot + p, 8 * p, wk)
    switch (nbits) {
      case 1: RS_PASS(1); break;
      case 2: RS_PASS(2); break;
      case 3: RS_PASS(3); break;
      case 4: RS_PASS(4); break;
      case 5: RS_PASS(5); break;
      case 6: RS_PASS(6); break;
      case 7: RS_PASS(7); break;
      default: RS_PASS(8); break;
    }
#undef RS_PASS
    kin = kout;
    vin = vout;
  }
  *keys_res = kin;
  *vals_res = vin;
}

template <typename K, int ITEMS, int NB>
void set_smem() {
  cudaFuncSetAttribute(onesweep_kernel<K, ITEMS, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)sizeof(OnesweepSmem<K, ITEMS>));
}
template <typename K, int ITEMS>
void set_smem_all() {
  set_smem<K, ITEMS, 1>(); set_smem<K, ITEMS, 2>(); set_smem<K, ITEMS, 3>(); set_smem<K, ITEMS, 4>();
  set_smem<K, ITEMS, 5>(); set_smem<K, ITEMS, 6>(); set_smem<K, ITEMS, 7>(); set_smem<K, ITEMS, 8>();
}
void configure_kernels() {  // per device; idempotent
  set_smem_all<uint32_t, kDepthItems>();
  cudaFuncSetAttribute(segplace_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * kMaxTileRows);
  cudaFuncSetAttribute(dsort_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(DsortSmem));
  cudaFuncSetAttribute(bsort_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(BsortSmem));
  cudaFuncSetAttribute(bsort_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(BsortSmem));
  cudaFuncSetAttribute(dsort_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(DsortSmem));
}

}  // namespace

extern "C" {

int32_t rs_abi_version(void) { return RS_ABI_VERSION; }

const char* rs_status_string(int32_t s) {
  switch (s) {
    case RS_OK: return "ok";
    case RS_EINVAL: return "invalid argument";
    case RS_ENONFINITE: return "scene contains non-finite parameters";
    case RS_ENOMEM_WORKSPACE: return "workspace too small";
    case RS_ECUDA: return "CUDA error";
    case RS_EOVERFLOW: return "tile pair capacity exceeded";
    default: return "unknown status";
  }
}

size_t rs_workspace_size(int64_t n_cap, int64_t pair_cap, int32_t width, int32_t height) {
  if (n_cap < 0 || pair_cap < 0 || width <= 0 || height <= 0) return 0;
  return make_layout(n_cap, pair_cap, width, height, device_sms()).total;
}

int32_t rs_workspace_create(void* device_mem, size_t bytes, int64_t n_cap, int64_t pair_cap, int32_t width,
                            int32_t height, rs_workspace** out) {
  if (!out || !device_mem || n_cap < 0 || n_cap > 0x7fffffffLL || pair_cap < 0 || pair_cap > 0xffffffffLL ||
      width <= 0 || height <= 0)
    return RS_EINVAL;
  const int TW = tiles_x(width), TH = tiles_x(height);
  if ((int64_t)TW * TH > 65536 || width > 32767 || height > 32767) return RS_EINVAL;  // 15-bit box fields
  const Layout L = make_layout(n_cap, pair_cap, width, height, device_sms());
  if (bytes < L.total) return RS_ENOMEM_WORKSPACE;
  rs_workspace* ws = new (std::nothrow) rs_workspace();
  if (!ws) return RS_ECUDA;
  ws->base = static_cast<unsigned char*>(device_mem);
  ws->bytes = bytes;
  ws->L = L;
  ws->n_cap = n_cap;
  ws->pair_cap = pair_cap;
  ws->W_cap = width;
  ws->H_cap = height;
  int dev = 0;
  cudaGetDevice(&dev);
  if (cudaDeviceGetAttribute(&ws->sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) ws->sms = 148;
  configure_kernels();
  exp_table_kernel<<<(kExpTab + 255) / 256, 256>>>(ws->at<double>(L.exptab));
  if (cudaMemset(ws->at<Sticky>(L.sticky), 0, sizeof(Sticky)) != cudaSuccess ||
      cudaStreamCreateWithFlags(&ws->aux, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&ws->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&ws->ev_join, cudaEventDisableTiming) != cudaSuccess) {
    delete ws;
    return RS_ECUDA;
  }
  *out = ws;
  return cuda_status();
}

void rs_workspace_destroy(rs_workspace* ws) { delete ws; }

int32_t rs_set_camera(rs_workspace* ws, const rs_camera* cam, void* stream) {
  if (!ws || !cam || cam->width <= 0 || cam->height <= 0) return RS_EINVAL;
  if (cam->width > ws->W_cap || cam->height > ws->H_cap) return RS_ENOMEM_WORKSPACE;
  const int TW = tiles_x(cam->width), TH = tiles_x(cam->height);
  ws->W = cam->width;
  ws->H = cam->height;
  ws->TW = TW;
  ws->TH = TH;
  ws->have_cam = true;
  // both precisions' cameras: the fp32 one rounded once here (round to nearest)
  CamPair cp;
  cp.c64 = *cam;
  Cam32& c = cp.c32;
  c.width = cam->width;
  c.height = cam->height;
  c.fx = (float)cam->fx; c.fy = (float)cam->fy; c.cx = (float)cam->cx; c.cy = (float)cam->cy;
  for (int k = 0; k < 9; ++k) c.R[k] = (float)cam->R[k];
  for (int k = 0; k < 3; ++k) { c.t[k] = (float)cam->t[k]; c.center[k] = (float)cam->center[k]; }
  // stream-ordered upload; from pageable memory the driver stages it at once, so the
  // caller may reuse `cam` immediately (a captured frame graph then replays it)
  cudaMemcpyAsync(ws->at<CamPair>(ws->L.cam), &cp, sizeof(CamPair), cudaMemcpyHostToDevice, S(stream));
  return cuda_status();
}

}  // extern "C"

template <bool FULL, bool COLOR, typename TS>
static void launch_project(rs_workspace* ws, const rs_scene* scene, const int32_t* active_idx, uint32_t items,
                           const rs_options* opts, void* full, int32_t* full_bbox, cudaStream_t st) {
  const unsigned grid = (items + kProjThreads - 1) / kProjThreads;
  const TS* planes = static_cast<const TS*>(scene->planes);
  const TS* sh = static_cast<const TS*>(scene->sh);
  CamPair* cp = ws->at<CamPair>(ws->L.cam);
  if (ws->f64)
    launch(project64_kernel<FULL, COLOR, TS>, grid, kProjThreads, 0, st, planes, sh, scene->plane_stride,
           scene->sh_degree, active_idx, items, scene->n, &cp->c64, opt64(*opts), ws->at<Rec>(ws->L.recs),
           ws->at<Rec64>(ws->L.recs64), ws->at<uint32_t>(ws->L.keysB), ws->at<uint32_t>(ws->L.rows), ws->ctr(),
           ws->at<Sticky>(ws->L.sticky), static_cast<double*>(full), reinterpret_cast<int4*>(full_bbox));
  else
    launch(project_kernel<FULL, COLOR, TS>, grid, kProjThreads, 0, st, planes, sh, scene->plane_stride,
           scene->sh_degree, active_idx, items, scene->n, &cp->c32, opt32(*opts), ws->at<Rec>(ws->L.recs),
           ws->at<uint32_t>(ws->L.keysB), ws->at<uint32_t>(ws->L.rows), ws->ctr(), ws->at<Sticky>(ws->L.sticky),
           static_cast<float*>(full), reinterpret_cast<int4*>(full_bbox));
}

extern "C" {

static int32_t project_impl(rs_workspace* ws, const rs_scene* scene, const int32_t* active_idx, int64_t m,
                            const rs_camera* cam, const rs_options* opts, void* full, int32_t* full_bbox,
                            bool color, void* stream) {
  if (!ws || !scene || !valid_options(opts) || !scene->planes || !scene->sh || scene->sh_degree < 0 ||
      scene->sh_degree > 3 || scene->n < 0 || scene->plane_stride < scene->n ||
      (scene->dtype != RS_F32 && scene->dtype != RS_F64) || (reinterpret_cast<uintptr_t>(scene->sh) & 15))
    return RS_EINVAL;
  const int64_t items = active_idx ? m : scene->n;
  if (items < 0) return RS_EINVAL;
  if (items > ws->n_cap) return RS_ENOMEM_WORKSPACE;
  cudaStream_t st = S(stream);
  // zero counters, histograms, ranges and the compaction look-back in one memset
  cudaMemsetAsync(ws->base, 0, ws->L.frame_bytes, st);
  if (cam) {
    const int32_t s = rs_set_camera(ws, cam, stream);
    if (s != RS_OK) return s;
  } else if (!ws->have_cam) {
    return RS_EINVAL;  // cam == NULL reuses the camera of the last rs_set_camera
  }
  ws->n_items = (uint32_t)items;
  ws->binned = false;
  ws->has_color = color || full;
  ws->f64 = opts->precision == RS_F64;
  if (items > 0) {
    const uint32_t n = (uint32_t)items;
    const bool d = scene->dtype == RS_F64;
    if (full) {
      if (d) launch_project<true, true, double>(ws, scene, active_idx, n, opts, full, full_bbox, st);
      else launch_project<true, true, float>(ws, scene, active_idx, n, opts, full, full_bbox, st);
    } else if (color) {
      if (d) launch_project<false, true, double>(ws, scene, active_idx, n, opts, nullptr, nullptr, st);
      else launch_project<false, true, float>(ws, scene, active_idx, n, opts, nullptr, nullptr, st);
    } else {
      if (d) launch_project<false, false, double>(ws, scene, active_idx, n, opts, nullptr, nullptr, st);
      else launch_project<false, false, float>(ws, scene, active_idx, n, opts, nullptr, nullptr, st);
    }
  }
  return cuda_status();
}

int32_t rs_project(rs_workspace* ws, const rs_scene* scene, const int32_t* active_idx, int64_t m,
                   const rs_camera* cam, const rs_options* opts, void* stream) {
  return project_impl(ws, scene, active_idx, m, cam, opts, nullptr, nullptr, true, stream);
}

int32_t rs_project_full(rs_workspace* ws, const rs_scene* scene, const int32_t* active_idx, int64_t m,
                        const rs_camera* cam, const rs_options* opts, void* out_proj, int32_t* out_bbox,
                        void* stream) {
  if (!out_proj || !out_bbox) return RS_EINVAL;
  return project_impl(ws, scene, active_idx, m, cam, opts, out_proj, out_bbox, true, stream);
}

int32_t rs_bin(rs_workspace* ws, void* stream) {
  if (!ws || ws->W <= 0) return RS_EINVAL;
  cudaStream_t st = S(stream);
  const uint32_t n = ws->n_items;
  if (n > 0) {
    // depth sort of the n_visible binned items (the projection wrote every item's key;
    // culled items carry kInvalidKey)
    const uint32_t* nvis = &ws->ctr()->n_visible;
    const uint32_t *keys_res, *items_sorted;
    bool sorted = false;
    // one cooperative kernel (compaction fused into pass 0, 4 passes, grid barriers) for frames
    // of up to ~1M items, where the launch chain's per-kernel latency dominates (configs[1]:
    // 52 vs 65 us); larger frames keep the onesweep launches (configs[2]: 112 vs 153 us)
    const int G_dsort = std::min(ws->sms, kMaxDsortCtas);
    // (the per-CTA digit counts are 16-bit: at most ceil(n / G) keys per CTA)
    if (n <= kBsortMaxItems && dsort_mode() == 1) {  // small frames: one CTA, shared memory only
      const cudaError_t e = ws->f64
          ? launch_ex(bsort_kernel<true>, 1, kBsortThreads, sizeof(BsortSmem), st, ws->at<uint32_t>(ws->L.keysB), n,
                      ws->at<uint32_t>(ws->L.keysA), ws->at<uint32_t>(ws->L.valsA), ws->ctr())
          : launch_ex(bsort_kernel<false>, 1, kBsortThreads, sizeof(BsortSmem), st, ws->at<uint32_t>(ws->L.keysB), n,
                      ws->at<uint32_t>(ws->L.keysA), ws->at<uint32_t>(ws->L.valsA), ws->ctr());
      if (e == cudaSuccess) {
        keys_res = ws->at<uint32_t>(ws->L.keysA);
        items_sorted = ws->at<uint32_t>(ws->L.valsA);
        sorted = true;
      } else {
        cudaGetLastError();
      }
    }
    if (!sorted && (n + G_dsort - 1) / G_dsort < 65536 &&
        (dsort_mode() == 2 || (dsort_mode() == 1 && n <= kDsortMaxItems))) {
      static const int g_env = [] {  // RS_DSORT_CTAS: grid override (A/B measurements)
        const char* e = std::getenv("RS_DSORT_CTAS");
        return e ? std::atoi(e) : 0;
      }();
      const int G = g_env > 0 ? std::min(g_env, G_dsort) : G_dsort;
      static const int force_bins = [] {  // RS_DSORT_BINS=256: always 4 passes of 8-bit digits (tests, A/B)
        const char* e = std::getenv("RS_DSORT_BINS");
        return e ? std::atoi(e) : 0;
      }();
      static const uint32_t red_max = [] {  // RS_DSORT_RED_MAX: the atomics/barrier switch (tests, A/B)
        const char* e = std::getenv("RS_DSORT_RED_MAX");
        return e ? (uint32_t)std::strtoul(e, nullptr, 10) : kDsortRedMax;
      }();
      const cudaError_t e = ws->f64
          ? launch_coop(dsort_kernel<true>, G, kDsortThreads, sizeof(DsortSmem), st, ws->at<uint32_t>(ws->L.keysB), n,
                        ws->at<uint32_t>(ws->L.keysA), ws->at<uint32_t>(ws->L.valsA), ws->at<uint32_t>(ws->L.keysC),
                        ws->at<uint32_t>(ws->L.valsB), ws->at<uint32_t>(ws->L.dtab), ws->ctr(), red_max, force_bins)
          : launch_coop(dsort_kernel<false>, G, kDsortThreads, sizeof(DsortSmem), st, ws->at<uint32_t>(ws->L.keysB), n,
                        ws->at<uint32_t>(ws->L.keysA), ws->at<uint32_t>(ws->L.valsA), ws->at<uint32_t>(ws->L.keysC),
                        ws->at<uint32_t>(ws->L.valsB), ws->at<uint32_t>(ws->L.dtab), ws->ctr(), red_max, force_bins);
      if (e == cudaSuccess) {
        keys_res = ws->at<uint32_t>(ws->L.keysA);
        items_sorted = ws->at<uint32_t>(ws->L.valsA);
        sorted = true;
      } else {
        cudaGetLastError();  // not launchable here (e.g. an SM partition): the launch chain below
      }
    }
    if (!sorted) {
      launch(compact_hist_kernel, (n + kCompactKeys - 1) / kCompactKeys, 256, 0, st,
             ws->at<uint32_t>(ws->L.keysB), n, ws->at<uint32_t>(ws->L.keysA), ws->at<uint32_t>(ws->L.valsA),
             ws->at<unsigned long long>(ws->L.proj_lb), ws->ctr(), kSortThreads * kDepthItems,
             ws->at<uint32_t>(ws->L.hist), ws->at<uint32_t>(ws->L.lbA));
      run_sort<uint32_t, kDepthItems>(ws, ws->at<uint32_t>(ws->L.keysA), ws->at<uint32_t>(ws->L.keysA),
                                      ws->at<uint32_t>(ws->L.keysB), ws->at<uint32_t>(ws->L.valsA),
                                      ws->at<uint32_t>(ws->L.valsA), ws->at<uint32_t>(ws->L.valsB), nvis, 0, n, 32,
                                      0, 0, ws->f64, st, &keys_res, &items_sorted);
    }
    if (ws->f64)  // fp32-rounded depth keys: runs of equal keys re-ordered by the fp64 depth
      launch(tiefix_kernel, std::min((n + 255) / 256, (uint32_t)ws->sms * 8), 256, 0, st, keys_res,
             const_cast<uint32_t*>(items_sorted), nvis, ws->at<Rec64>(ws->L.recs64));
    // row segments: per rank chunk and row counts, their per-row prefix, each segment placed
    // in row-major depth-stable order; per-tile ranges, expansion into the per-tile lists
    // (segbin.cuh)
    Counters* ctr = ws->ctr();
    const uint32_t seg_cap = (uint32_t)seg_capacity(ws->n_cap, ws->pair_cap);
    const uint32_t tab_stride = (uint32_t)rowtab_stride(ws->n_cap);
    const unsigned rc = (n + kRankChunk - 1) / kRankChunk;
    static const int slots = [] {  // RS_EXPAND_SLOTS: chunk slots per SM of the expansion grids (A/B)
      const char* e = std::getenv("RS_EXPAND_SLOTS");
      return e ? std::max(std::atoi(e), 1) : 16;
    }();
    const unsigned gx = (unsigned)std::min<int64_t>(seg_cap / kExpandChunk + ws->TH + 1, (int64_t)ws->sms * slots);
    // expansion: the sparse chunks grid-strided (column groups x chunk slots), the dense ones on
    // persistent ticketed CTAs on the workspace's second stream, concurrently
    const unsigned groups = (ws->TW + kExpandCols - 1) / kExpandCols;
    const dim3 eg((groups + RS_EXPAND_GROUPS - 1) / RS_EXPAND_GROUPS, gx), dg(ws->sms * 6);
    const int T = ws->TW * ws->TH;
    launch(segrows_kernel, rc, 256, 0, st, items_sorted, ws->at<uint32_t>(ws->L.rows), ctr, ws->TH, tab_stride,
           ws->at<uint32_t>(ws->L.rowtab));
    launch(segscan_kernel, ws->TH, 256, 0, st, ws->at<uint32_t>(ws->L.rowtab), tab_stride, ctr, ws->TH, seg_cap,
           ws->at<uint32_t>(ws->L.rowcnt), ws->at<uint32_t>(ws->L.rowstart), ws->at<uint32_t>(ws->L.chunkstart),
           ws->at<Sticky>(ws->L.sticky));
    launch(segplace_kernel, rc, 256, 64 * ws->TH, st, items_sorted, ws->at<Rec>(ws->L.recs), ctr, ws->TH,
           ws->at<uint32_t>(ws->L.rowtab), tab_stride, ws->at<uint32_t>(ws->L.rowstart),
           ws->at<uint32_t>(ws->L.segitem), ws->at<uint32_t>(ws->L.segspan), ws->at<float4>(ws->L.geom));
    launch(chunk_count_kernel, gx, 256, 0, st, ws->at<uint32_t>(ws->L.segspan),
           ws->at<uint32_t>(ws->L.rowstart), ws->at<uint32_t>(ws->L.chunkstart), ws->TH, ws->TW,
           ws->at<uint32_t>(ws->L.chunkcnt), ws->at<uint2>(ws->L.chunkinfo), expand_dense_span(), ctr,
           ws->at<uint32_t>(ws->L.densel));
    launch(tile_chunks_kernel, (T + 7) / 8, 256, 0, st, ws->at<uint32_t>(ws->L.chunkstart), ws->TH, ws->TW,
           ws->at<uint32_t>(ws->L.chunkcnt), ws->at<uint32_t>(ws->L.tilecnt),
           ws->at<unsigned long long>(ws->L.scanpart), ws->at<uint32_t>(ws->L.scancls));
    launch(tile_scan_kernel, (T + kScanTiles - 1) / kScanTiles, kScanTiles, 0, st, ws->at<uint32_t>(ws->L.tilecnt), T,
           ctr, (uint32_t)ws->pair_cap, ws->at<uint2>(ws->L.ranges), ws->at<Sticky>(ws->L.sticky),
           ws->at<uint32_t>(ws->L.tileord), ws->at<unsigned long long>(ws->L.scanpart), ws->at<uint32_t>(ws->L.scancls));
    cudaEventRecord(ws->ev_fork, st);
    cudaStreamWaitEvent(ws->aux, ws->ev_fork, 0);
    g_pdl_class = kPdlExpand;
    launch(expand_dense_kernel, dg, 256, 0, ws->aux, ws->at<uint32_t>(ws->L.segitem),
           ws->at<uint32_t>(ws->L.segspan), ws->at<uint2>(ws->L.chunkinfo), ws->at<uint32_t>(ws->L.densel),
           ws->TW, ws->at<uint32_t>(ws->L.chunkcnt), ws->at<uint2>(ws->L.ranges), ctr,
           ws->at<uint32_t>(ws->L.pitem));
    cudaEventRecord(ws->ev_join, ws->aux);
    launch(expand_kernel, eg, 256, 0, st, ws->at<uint32_t>(ws->L.segitem), ws->at<uint32_t>(ws->L.segspan),
           ws->at<uint2>(ws->L.chunkinfo), ws->at<uint32_t>(ws->L.chunkstart), ws->TH, ws->TW,
           ws->at<uint32_t>(ws->L.chunkcnt), ws->at<uint2>(ws->L.ranges), ctr, ws->at<uint32_t>(ws->L.pitem),
           expand_major_thresh());
    cudaStreamWaitEvent(st, ws->ev_join, 0);
    g_pdl_class = kPdlChain;
  } else {  // no items: no tile scan ran -- the blends' CTA -> tile map is the identity
    const int T = ws->TW * ws->TH;
    launch(tile_order_identity_kernel, (T + 255) / 256, 256, 0, st, ws->at<uint32_t>(ws->L.tileord), T);
  }
  ws->binned = true;
  return cuda_status();
}

static const uint32_t* final_pair_items(const rs_workspace* ws) { return ws->at<uint32_t>(ws->L.pitem); }

int32_t rs_blend_ex(rs_workspace* ws, const rs_options* opts, const rs_outputs* out_p, void* scores_v,
                    uint32_t flags, void* stream) {
  if (!ws || !valid_options(opts) || !ws->binned) return RS_EINVAL;
  if ((opts->precision == RS_F64) != ws->f64) return RS_EINVAL;  // not the precision of the projection
  rs_outputs out{};
  if (out_p) out = *out_p;
  if ((out.rgb != nullptr) != (out.alpha != nullptr) || (out.rgb != nullptr) != (out.count != nullptr) ||
      (out.rgb64 != nullptr) != (out.alpha64 != nullptr) || (out.rgb64 != nullptr) != (out.count64 != nullptr))
    return RS_EINVAL;
  const bool color = out.rgb || out.rgb64 || out.depth || out.tau;
  if ((out.tau != nullptr) != (out.last != nullptr)) return RS_EINVAL;
  if (out.tau && ws->f64) return RS_EINVAL;  // the training outputs are fp32-path only
  if (color && !ws->has_color) return RS_EINVAL;  // projected by a score-only rs_render
  if (!color && !scores_v) return RS_EINVAL;
  const bool stats = (flags & RS_FLAG_COUNT_EVALS) != 0;
  cudaStream_t st = S(stream);
  const int T = ws->TW * ws->TH;
  const uint2* ranges = ws->at<uint2>(ws->L.ranges);
  const uint32_t* items = final_pair_items(ws);
  const Rec* recs = ws->at<Rec>(ws->L.recs);
  const float4* geom = ws->at<float4>(ws->L.geom);  // ellipse row geometry (warp quarter masks)
  const uint32_t* order = ws->at<uint32_t>(ws->L.tileord);  // CTA -> tile (tile_scan_kernel)
  Counters* ctr = ws->ctr();
  g_pdl_class = kPdlBlend;
  struct Restore {
    ~Restore() { g_pdl_class = kPdlChain; }
  } restore;
  if (ws->f64) {
    const Out64 o64{static_cast<double*>(out.rgb), static_cast<double*>(out.alpha), static_cast<double*>(out.depth),
                    out.count, out.rgb64, out.alpha64, out.count64};
    const Opt64 op = opt64(*opts);
    const Rec64* r64 = ws->at<Rec64>(ws->L.recs64);
    auto* sc = static_cast<unsigned long long*>(scores_v);
    // exp64_tab's normal range and non-negative thresholds (integer compares, blend64.cuh)
    const bool fast = opts->alpha_cut >= 1e-300 && opts->alpha_max >= 0.0 && opts->alpha_max <= 1e300 &&
                      opts->tau_stop >= 0.0 && opts->lowpass >= 0.0;
#define RS_B64(C, I, K, F) \
  launch(blend64_kernel<C, I, K, F>, T, kBlend64Threads, 0, st, ranges, items, recs, r64, geom, order, ctr, ws->W, \
         ws->H, ws->TW, op, o64, sc, ws->at<double>(ws->L.exptab))
#define RS_B64_F(C, I, K) \
  if (fast) { RS_B64(C, I, K, true); } else { RS_B64(C, I, K, false); }
    if (color && sc) {
      if (stats) { RS_B64_F(true, true, true); } else { RS_B64_F(true, true, false); }
    } else if (color) {
      if (stats) { RS_B64_F(true, false, true); } else { RS_B64_F(true, false, false); }
    } else {
      if (stats) { RS_B64_F(false, true, true); } else { RS_B64_F(false, true, false); }
    }
#undef RS_B64_F
#undef RS_B64
    return cuda_status();
  }
  const Out32 o32{static_cast<float*>(out.rgb), static_cast<float*>(out.alpha), static_cast<float*>(out.depth),
                  out.count, out.rgb64, out.alpha64, out.count64, out.tau, out.last};
  const Opt32 op = opt32(*opts);
  uint32_t* scores = static_cast<uint32_t*>(scores_v);
  const bool one_px = (flags & RS_FLAG_BLEND_1PX) != 0 && !out.tau;  // the training outputs: 2-px kernel
#define RS_BLEND(C, I, K, F)                                                                              \
  if (one_px)                                                                                             \
    launch(blend_kernel<C, I, K, F>, T, kBlendThreads, 0, st, ranges, items, recs, ctr, ws->W, ws->H,     \
           ws->TW, op, o32, scores);                                                                       \
  else                                                                                                    \
    launch(blend2_kernel<C, I, K, F>, T, kBlend2Threads, 0, st, ranges, items, recs, geom, order, ctr,    \
           ws->W, ws->H, ws->TW, op, o32, scores)
#define RS_BLEND_F(C, I, K) \
  if (fast) { RS_BLEND(C, I, K, true); } else { RS_BLEND(C, I, K, false); }
  // exact-range exp2 is only needed for degenerate options (see blend.cuh FAST)
  const bool fast = op.alpha_cut >= 1e-30f;
  if (out.tau) {  // training forward (rasterize_cached): records tau and the last composite per pixel
    if (scores) {
      if (fast) launch(blend2_kernel<true, true, false, true, true>, T, kBlend2Threads, 0, st, ranges, items,
                       recs, geom, order, ctr, ws->W, ws->H, ws->TW, op, o32, scores);
      else launch(blend2_kernel<true, true, false, false, true>, T, kBlend2Threads, 0, st, ranges, items, recs,
                  geom, order, ctr, ws->W, ws->H, ws->TW, op, o32, scores);
    } else {
      if (fast) launch(blend2_kernel<true, false, false, true, true>, T, kBlend2Threads, 0, st, ranges, items,
                       recs, geom, order, ctr, ws->W, ws->H, ws->TW, op, o32, scores);
      else launch(blend2_kernel<true, false, false, false, true>, T, kBlend2Threads, 0, st, ranges, items, recs,
                  geom, order, ctr, ws->W, ws->H, ws->TW, op, o32, scores);
    }
  } else if (color && scores) {
    if (stats) { RS_BLEND_F(true, true, true); } else { RS_BLEND_F(true, true, false); }
  } else if (color) {
    if (stats) { RS_BLEND_F(true, false, true); } else { RS_BLEND_F(true, false, false); }
  } else {
    if (stats) { RS_BLEND_F(false, true, true); } else { RS_BLEND_F(false, true, false); }
  }
#undef RS_BLEND_F
#undef RS_BLEND
  return cuda_status();
}

int32_t rs_blend(rs_workspace* ws, const rs_options* opts, void* out_rgb, void* out_alpha, void* out_depth,
                 int32_t* out_count, void* scores, uint32_t flags, void* stream) {
  if (out_rgb && (!out_alpha || !out_depth || !out_count)) return RS_EINVAL;
  const rs_outputs out{out_rgb, out_alpha, out_depth, out_count, nullptr, nullptr, nullptr, nullptr, nullptr};
  return rs_blend_ex(ws, opts, &out, scores, flags, stream);
}

int32_t rs_render_ex(rs_workspace* ws, const rs_scene* scene, const int32_t* active_idx, int64_t m,
                     const rs_camera* cam, const rs_options* opts, const rs_outputs* out, void* scores,
                     uint32_t flags, void* stream) {
  // a score-only frame (no image outputs) projects without the SH colour
  const bool color = out && (out->rgb || out->rgb64 || out->depth || out->tau);
  int32_t s = project_impl(ws, scene, active_idx, m, cam, opts, nullptr, nullptr, color, stream);
  if (s != RS_OK) return s;
  if ((s = rs_bin(ws, stream)) != RS_OK) return s;
  return rs_blend_ex(ws, opts, out, scores, flags, stream);
}

int32_t rs_render(rs_workspace* ws, const rs_scene* scene, const int32_t* active_idx, int64_t m,
                  const rs_camera* cam, const rs_options* opts, void* out_rgb, void* out_alpha, void* out_depth,
                  int32_t* out_count, void* scores, uint32_t flags, void* stream) {
  if (out_rgb && (!out_alpha || !out_depth || !out_count)) return RS_EINVAL;
  const rs_outputs out{out_rgb, out_alpha, out_depth, out_count, nullptr, nullptr, nullptr, nullptr, nullptr};
  return rs_render_ex(ws, scene, active_idx, m, cam, opts, &out, scores, flags, stream);
}

int32_t rs_backward(rs_workspace* ws, const rs_scene* scene, const int32_t* active_idx, int64_t m,
                    const rs_options* opts, const float* grad_image, const float* tau, const int32_t* last,
                    float* g_pos, float* g_sh, float* g_ls, float* g_quat, float* g_logit, float* g_mean2d,
                    uint8_t* touched, void* stream) {
  if (!ws || !scene || !valid_options(opts) || !grad_image || !tau || !last || !g_pos || !g_sh || !g_ls || !g_quat ||
      !g_logit || !g_mean2d || !touched || !ws->binned || !ws->has_color || ws->f64 ||
      opts->precision != RS_F32 || scene->dtype != RS_F32)
    return RS_EINVAL;  // the training pair is the fp32 path
  const int64_t items = active_idx ? m : scene->n;
  if (items != (int64_t)ws->n_items) return RS_EINVAL;  // not the frame rs_render_ex just produced
  cudaStream_t st = S(stream);
  const int64_t n = scene->n;
  if (active_idx || items == 0) {  // Gaussians outside the list keep zero gradients; else
    cudaMemsetAsync(g_pos, 0, (size_t)n * 12, st);  // chain_kernel writes every item's
    cudaMemsetAsync(g_sh, 0, (size_t)n * 192, st);
    cudaMemsetAsync(g_ls, 0, (size_t)n * 12, st);
    cudaMemsetAsync(g_quat, 0, (size_t)n * 16, st);
    cudaMemsetAsync(g_logit, 0, (size_t)n * 4, st);
    cudaMemsetAsync(g_mean2d, 0, (size_t)n * 4, st);
    cudaMemsetAsync(touched, 0, (size_t)n, st);
  }
  if (items == 0) return cuda_status();
  cudaMemsetAsync(ws->at<float>(ws->L.sgrad), 0, (size_t)items * 4 * kSGrad, st);
  cudaMemsetAsync(ws->at<uint8_t>(ws->L.titem), 0, (size_t)items, st);
  const Opt32 op = opt32(*opts);
  auto* bwd = op.alpha_cut >= 1e-30f ? backward2_kernel<true> : backward2_kernel<false>;
  launch(bwd, ws->TW * ws->TH, kBwd2Threads, 0, st, ws->at<uint2>(ws->L.ranges), final_pair_items(ws),
         ws->at<Rec>(ws->L.recs), ws->at<float4>(ws->L.geom), ws->at<uint32_t>(ws->L.tileord), ws->ctr(), ws->W,
         ws->H, ws->TW, op, grad_image, tau, last, ws->at<float>(ws->L.sgrad), ws->at<uint8_t>(ws->L.titem));
  launch(chain_kernel, (unsigned)((items + 127) / 128), 128, 0, st, static_cast<const float*>(scene->planes),
         static_cast<const float*>(scene->sh), scene->plane_stride, scene->sh_degree, active_idx, (uint32_t)items,
         &ws->at<CamPair>(ws->L.cam)->c32, op, ws->at<float>(ws->L.sgrad), ws->at<uint8_t>(ws->L.titem), g_pos,
         g_sh, g_ls, g_quat, g_logit, g_mean2d, touched);
  return cuda_status();
}

int32_t rs_read_stats(rs_workspace* ws, rs_stats* out, void* stream) {
  if (!ws || !out) return RS_EINVAL;
  Counters c;
  if (cudaMemcpyAsync(&c, ws->ctr(), sizeof(c), cudaMemcpyDeviceToHost, S(stream)) != cudaSuccess) return RS_ECUDA;
  if (cudaStreamSynchronize(S(stream)) != cudaSuccess) return RS_ECUDA;
  out->n_items = c.n_items;
  out->n_visible = c.n_visible;
  out->n_pairs = c.n_pairs;
  out->overflow = c.overflow;
  out->evals = c.evals;
  out->composites = c.composites;
  out->pairs_needed = c.pairs_needed;
  out->bad_index = c.bad_index;
  out->_pad = 0;
  return RS_OK;
}

int32_t rs_read_overflow(rs_workspace* ws, uint32_t* out_overflowed, uint64_t* out_pairs_needed_max,
                         int32_t reset, void* stream) {
  if (!ws || !out_overflowed || !out_pairs_needed_max) return RS_EINVAL;
  Sticky h;
  Sticky* d = ws->at<Sticky>(ws->L.sticky);
  if (cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, S(stream)) != cudaSuccess) return RS_ECUDA;
  if (reset && cudaMemsetAsync(d, 0, sizeof(Sticky), S(stream)) != cudaSuccess) return RS_ECUDA;
  if (cudaStreamSynchronize(S(stream)) != cudaSuccess) return RS_ECUDA;
  *out_overflowed = h.overflowed;
  *out_pairs_needed_max = h.pairs_needed_max;
  return RS_OK;
}

int32_t rs_read_sticky(rs_workspace* ws, uint32_t* out_overflowed, uint64_t* out_pairs_needed_max,
                       uint32_t* out_bad_index, int32_t reset, void* stream) {
  if (!out_bad_index) return RS_EINVAL;
  Sticky h;
  if (!ws || !out_overflowed || !out_pairs_needed_max) return RS_EINVAL;
  Sticky* d = ws->at<Sticky>(ws->L.sticky);
  if (cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, S(stream)) != cudaSuccess) return RS_ECUDA;
  if (reset && cudaMemsetAsync(d, 0, sizeof(Sticky), S(stream)) != cudaSuccess) return RS_ECUDA;
  if (cudaStreamSynchronize(S(stream)) != cudaSuccess) return RS_ECUDA;
  *out_overflowed = h.overflowed;
  *out_pairs_needed_max = h.pairs_needed_max;
  *out_bad_index = h.bad_index;
  return RS_OK;
}

int32_t rs_get_buffers(rs_workspace* ws, rs_buffers* out) {
  if (!ws || !out) return RS_EINVAL;
  out->records = ws->at<void>(ws->L.recs);
  out->records64 = ws->at<void>(ws->L.recs64);
  out->items_sorted = ws->at<uint32_t>(ws->L.valsA);  // 4 depth passes end in A
  out->pair_items = final_pair_items(ws);
  out->ranges = ws->at<uint32_t>(ws->L.ranges);
  out->counters = ws->at<uint32_t>(ws->L.ctr);
  out->tiles_x = ws->TW;
  out->tiles_y = ws->TH;
  return RS_OK;
}

size_t rs_compact_workspace_size(int64_t n) {
  return align_up(((size_t)std::max<int64_t>(n, 0) / kCompactPerBlock + 2) * 8 + 256);
}

static int32_t compact_impl(const uint8_t* flags, int64_t n, int32_t* out_idx, uint32_t* out_count, void* scratch,
                            size_t scratch_bytes, void* stream, bool bits) {
  if (n < 0 || !out_count || (n > 0 && (!flags || !out_idx)) || n > 0x7fffffffLL) return RS_EINVAL;
  if (scratch_bytes < rs_compact_workspace_size(n) || !scratch) return RS_ENOMEM_WORKSPACE;
  cudaStream_t st = S(stream);
  cudaMemsetAsync(out_count, 0, 4, st);
  if (n == 0) return cuda_status();
  const int blocks = (int)((n + kCompactPerBlock - 1) / kCompactPerBlock);
  cudaMemsetAsync(scratch, 0, (size_t)blocks * 8 + 256, st);
  uint32_t* ticket = reinterpret_cast<uint32_t*>(scratch);
  unsigned long long* status = reinterpret_cast<unsigned long long*>(static_cast<unsigned char*>(scratch) + 256);
  if (bits)
    compact_kernel<true><<<blocks, kCompactThreads, 0, st>>>(flags, n, out_idx, out_count, status, ticket);
  else
    compact_kernel<false><<<blocks, kCompactThreads, 0, st>>>(flags, n, out_idx, out_count, status, ticket);
  return cuda_status();
}

int32_t rs_compact(const uint8_t* flags, int64_t n, int32_t* out_idx, uint32_t* out_count, void* scratch,
                   size_t scratch_bytes, void* stream) {
  return compact_impl(flags, n, out_idx, out_count, scratch, scratch_bytes, stream, false);
}

int32_t rs_compact_bits(const uint8_t* bits, int64_t n, int32_t* out_idx, uint32_t* out_count, void* scratch,
                        size_t scratch_bytes, void* stream) {
  return compact_impl(bits, n, out_idx, out_count, scratch, scratch_bytes, stream, true);
}

int32_t rs_check_finite(const rs_scene* scene, uint32_t* out_bad, void* stream) {
  if (!scene || !out_bad || scene->n < 0 || (scene->n > 0 && (!scene->planes || !scene->sh)) ||
      scene->plane_stride < scene->n || (scene->dtype != RS_F32 && scene->dtype != RS_F64))
    return RS_EINVAL;
  cudaStream_t st = S(stream);
  cudaMemsetAsync(out_bad, 0, 4, st);
  if (scene->n > 0) {
    if (scene->dtype == RS_F64)
      finite_kernel<double><<<1184, 256, 0, st>>>(static_cast<const double*>(scene->planes),
                                                  static_cast<const double*>(scene->sh), scene->n,
                                                  scene->plane_stride, out_bad);
    else
      finite_kernel<float><<<1184, 256, 0, st>>>(static_cast<const float*>(scene->planes),
                                                 static_cast<const float*>(scene->sh), scene->n,
                                                 scene->plane_stride, out_bad);
  }
  return cuda_status();
}

int32_t rs_rspl_unpack(const float* payload, int64_t n, float* planes, int64_t plane_stride, float* sh,
                       uint32_t* out_bad, void* stream) {
  if (n < 0 || plane_stride < n || !out_bad || (n > 0 && (!payload || !planes || !sh)) ||
      (reinterpret_cast<uintptr_t>(payload) & 15) || (reinterpret_cast<uintptr_t>(sh) & 15))
    return RS_EINVAL;
  cudaStream_t st = S(stream);
  cudaMemsetAsync(out_bad, 0, 4, st);
  if (n > 0)
    rspl_unpack_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(payload, n, planes, plane_stride, sh, out_bad);
  return cuda_status();
}

int32_t rs_rspl_pack(const float* planes, int64_t plane_stride, const float* sh, int64_t n, float* payload,
                     void* stream) {
  if (n < 0 || plane_stride < n || (n > 0 && (!payload || !planes || !sh)) ||
      (reinterpret_cast<uintptr_t>(payload) & 15) || (reinterpret_cast<uintptr_t>(sh) & 15))
    return RS_EINVAL;
  if (n > 0)
    rspl_pack_kernel<<<(unsigned)((n + 255) / 256), 256, 0, S(stream)>>>(planes, plane_stride, sh, n, payload);
  return cuda_status();
}

int32_t rs_pack_bits(const uint8_t* flags, int64_t n, uint8_t* bits, void* stream) {
  if (n < 0 || (n > 0 && (!flags || !bits))) return RS_EINVAL;
  if (n > 0) pack_bits_kernel<<<(unsigned)((n + 255) / 256), 256, 0, S(stream)>>>(flags, n, bits);
  return cuda_status();
}

int32_t rs_sq_diff_sum(const double* a, const double* b, int64_t n, double* out_sum, void* stream) {
  if (n < 0 || !out_sum || (n > 0 && (!a || !b))) return RS_EINVAL;
  cudaStream_t st = S(stream);
  cudaMemsetAsync(out_sum, 0, sizeof(double), st);
  if (n > 0) sq_diff_sum_kernel<<<(unsigned)std::min<int64_t>((n + 255) / 256, 1184), 256, 0, st>>>(a, b, n, out_sum);
  return cuda_status();
}

size_t rs_ssim_workspace_size(int32_t height, int32_t width, int32_t channels, int32_t win) {
  if (height < win || width < win || channels <= 0 || win <= 0) return 0;
  return (size_t)3 * (height - win + 1) * (width - win + 1) * channels * sizeof(double);
}

int32_t rs_ssim(const double* x, const double* y, int32_t height, int32_t width, int32_t channels, int32_t win,
                const double* kernel, double* out_sum, double* grad, void* scratch, size_t scratch_bytes,
                void* stream) {
  if (!x || !y || !kernel || !out_sum || win <= 0 || win > kMaxSsimWin || height < win || width < win ||
      channels <= 0)
    return RS_EINVAL;
  if (grad && (!scratch || scratch_bytes < rs_ssim_workspace_size(height, width, channels, win)))
    return RS_ENOMEM_WORKSPACE;
  cudaStream_t st = S(stream);
  cudaMemsetAsync(out_sum, 0, sizeof(double), st);
  const int64_t nwin = (int64_t)(height - win + 1) * (width - win + 1) * channels;
  double* maps = grad ? static_cast<double*>(scratch) : nullptr;
  ssim_window_kernel<<<(unsigned)((nwin + 255) / 256), 256, 0, st>>>(x, y, height, width, channels, win, kernel,
                                                                    out_sum, maps);
  if (grad) {
    const int64_t npx = (int64_t)height * width * channels;
    ssim_grad_kernel<<<(unsigned)((npx + 255) / 256), 256, 0, st>>>(x, y, height, width, channels, win, kernel,
                                                                     maps, 1.0 / (double)nwin, grad);
  }
  return cuda_status();
}

int32_t rs_nearest_cluster(const double* centers, int32_t k, const double* positions, int64_t m, int32_t* out,
                           void* stream) {
  if (k <= 0 || m < 0 || !centers || (m > 0 && (!positions || !out))) return RS_EINVAL;
  if (m > 0)
    nearest_cluster_kernel<<<(unsigned)((m + 255) / 256), 256, 0, S(stream)>>>(centers, k, positions, m, out);
  return cuda_status();
}

int32_t rs_max_merge(float* dst, const float* src, int64_t n, void* stream) {
  if (n < 0 || (n > 0 && (!dst || !src))) return RS_EINVAL;
  if (n > 0)
    max_merge_kernel<<<(unsigned)std::min<int64_t>((n + 255) / 256, 4096), 256, 0, S(stream)>>>(
        reinterpret_cast<uint32_t*>(dst), reinterpret_cast<const uint32_t*>(src), n);
  return cuda_status();
}

}  // extern "C"
