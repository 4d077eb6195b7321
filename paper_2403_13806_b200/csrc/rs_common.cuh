// rs_common.cuh -- shared device types of the render-and-prune path.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

#include "../../include/radsplat.h"

namespace rs {

constexpr int kTile = 16;          // 16x16 pixel tiles, one CTA of 256 threads each
constexpr int kBlendThreads = 256;
constexpr int kProjThreads = 128;  // projection CTA
constexpr uint32_t kInvalidKey = 0xffffffffu;
constexpr int kPlanes = 59;

// Projected Gaussian, 64 B = 4 x 16 B so a batch is staged with four
// 128-bit loads per thread and read back from shared memory as broadcasts.
//   a = {mean x, mean y, na, nb}   na,nb,nc = -0.5*log2(e) * (ia, 2*ib, ic)
//   b = {nc, opacity, cut2, depth} cut2: log2 power below which alpha < alpha_cut
//   c = {r, g, b, gid bits}        gid = scene index (for importance scatter)
//   d = {x0 | x1<<16, y0 | y1<<16, cx0 | cx1<<16 | tight<<31, cy0 | cy1<<16}
//       [x0,x1)x[y0,y1): the half-open 3-sigma pixel bbox of render.py:133-137;
//       [cx0,cx1)x[cy0,cy1): a sub-box outside which no pixel can reach
//       alpha >= alpha_cut (culling only -- never changes a result, §4 DESIGN.md);
//       bit 31 of d.w ("ell"): the box came from the ellipse, so the tile binning
//       lists per tile row only the columns the ellipse reaches (rows.cuh)
struct __align__(16) Rec {
  float4 a, b, c;
  int4 d;
};
static_assert(sizeof(Rec) == 64, "record must be 64 B");

// fp64 record of an RS_F64 frame (96 B = 6 x 16 B), the reference's projected
// quantities in double (render.py:95-158), the conic pre-scaled by -1/2 (exact):
// (na, nb, nc) = -(ia/2, ib, ic/2), so the blend's
// x = fma(nc dy, dy, fma(nb dy, dx, (na dx) dx)) is -q/2 of render.py:254-256 with
// fused roundings, alpha = min(o e^x, alpha_max). lnc = ln(alpha_cut / o) - 1e-6 is
// a conservative skip bound (x < lnc => alpha < alpha_cut): the exp is not
// evaluated, no result changes. The binning uses the fp32 Rec written next to it
// (boxes, row geometry, depth key).
struct __align__(16) Rec64 {
  double mx, my, na, nb, nc, o, depth, lnc;
  double r, g, b;
  uint32_t gid, pad;
};
static_assert(sizeof(Rec64) == 96, "fp64 record must be 96 B");

// Device-side views of the boundary structs (include/radsplat.h): the fp32 path
// works on the camera and options rounded once on the host (round to nearest,
// = numpy astype(float32)); the fp64 path reads rs_camera / rs_options as is.
struct Cam32 {
  int32_t width, height;
  float fx, fy, cx, cy;
  float R[9];
  float t[3];
  float center[3];
};
struct Opt32 {
  float alpha_max, alpha_cut, tau_stop, near_limit, lowpass, sigma_bound;
};
struct Opt64 {
  double alpha_max, alpha_cut, tau_stop, near_limit, lowpass, sigma_bound;
};
// typed rs_outputs (RS_F32 / RS_F64 frames)
struct Out32 {
  float* rgb;
  float* alpha;
  float* depth;
  int32_t* count;
  double* rgb64;
  double* alpha64;
  int64_t* count64;
  float* tau;
  int32_t* last;
};
struct Out64 {
  double* rgb;
  double* alpha;
  double* depth;
  int32_t* count;
  double* rgb64;
  double* alpha64;
  int64_t* count64;
};
// the camera as it lives in the workspace: both precisions, uploaded together
struct CamPair {
  rs_camera c64;
  Cam32 c32;
};

__device__ __forceinline__ int lo16(int v) { return v & 0xffff; }
__device__ __forceinline__ int hi16(int v) { return (int)((unsigned)v >> 16); }
__device__ __forceinline__ int4 bbox_of(const int4 d) { return make_int4(lo16(d.x), hi16(d.x), lo16(d.y), hi16(d.y)); }
// culling box; bit 31 of d.z flags a box derived from the ellipse (then every pixel
// outside it has p2 < cut2, so a per-pixel box test is redundant)
__device__ __forceinline__ int4 cullbox_of(const int4 d) {
  return make_int4(lo16(d.z), hi16(d.z) & 0x7fff, lo16(d.w), hi16(d.w) & 0x7fff);
}
__device__ __forceinline__ bool cullbox_ell(const int4 d) { return d.w < 0; }
__device__ __forceinline__ bool cullbox_tight(const int4 d) { return d.z < 0; }

// Device-side counters, mirrors rs_stats (first four words) + sort bookkeeping.
// Programmatic dependent launch (api.cu launch()): wait for the previous kernel of the stream
// to complete (its writes visible), then let the next one be scheduled. No-ops for a kernel
// launched without the attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

struct Counters {
  uint32_t n_items, n_visible, n_pairs, overflow;  // n_pairs = min(P, pair capacity)
  unsigned long long evals, composites;
  unsigned long long pairs_needed;                 // true P (sizing hint after overflow)
  uint32_t tickets[12];  // onesweep chunk tickets, one per pass
  uint32_t spare0, spare1;
  uint32_t proj_ticket;  // logical block ticket of the depth-key compaction
  uint32_t n_segs;       // row segments of the binned items (segbin.cuh)
  uint32_t n_dense;      // dense expansion chunks listed by chunk_count_kernel
  uint32_t dense_work;   // (dense chunk, column group) tickets of expand_dense_kernel
  uint32_t emit_done;    // finished segscan CTAs (the last one scans the row totals)
  uint32_t bad_index;    // an active_idx entry outside [0, n) was skipped
  uint32_t gbar[2];      // grid barrier {arrivals, generation} of the cooperative kernels
};
static_assert(sizeof(Counters) == 128, "Counters is 128 B");

enum : unsigned long long { kLbAgg = 1ull << 62, kLbInc = 2ull << 62, kLbMask = (1ull << 62) - 1 };

// Decoupled look-back over 64-bit status words (flag in the top 2 bits);
// one warp reads 32 predecessors per step.
__device__ __forceinline__ unsigned long long warp_lookback(volatile unsigned long long* st, uint32_t b, int lane) {
  unsigned long long excl = 0;
  int j = (int)b - 1;
  while (j >= 0) {
    const int k = j - lane;  // lane 0 = nearest predecessor
    const unsigned long long s = k >= 0 ? st[k] : (unsigned long long)kLbInc;  // before block 0: inclusive zero
    const unsigned ready = __ballot_sync(0xffffffffu, (s & ~(unsigned long long)kLbMask) != 0);
    const unsigned inc = __ballot_sync(0xffffffffu, (s & (unsigned long long)kLbInc) != 0) & ready;
    const unsigned notready = ~ready;
    // use the window up to (and including) the nearest inclusive entry, or up to the first
    // unpublished entry, whichever comes first
    const int first_inc = inc ? __ffs(inc) - 1 : 32;
    const int first_nr = notready ? __ffs(notready) - 1 : 32;
    const int take = first_inc < first_nr ? first_inc + 1 : first_nr;  // lanes [0, take)
    unsigned long long v = (lane < take && k >= 0) ? (s & (unsigned long long)kLbMask) : 0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    excl += v;
    if (first_inc < first_nr) break;
    j -= take;
  }
  return excl;
}

// Overflow record that outlives the per-frame counter reset: a batch of frames
// (e.g. a scoring pass) is launched without host syncs and checked once.
struct Sticky {
  uint32_t overflowed, bad_index;
  unsigned long long pairs_needed_max;
};

}  // namespace rs
