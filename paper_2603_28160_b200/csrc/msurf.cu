// libmsurf.so — B200 (sm_100a) kernels for the FSM surface-topography hot path
// of arXiv 2603.28160 (reference package `millsurf`), behind the C ABI in
// include/msurf.h (design and measurements: DESIGN.md §4).
//
//  * sweep_kernel<MODE, DIAG, ONE>: engine.py:215-313 for all (pass, tooth,
//    step, edge point) of one or many surfaces. One CTA = one (job, pass,
//    tooth, tile of 128 time steps). Phase 1: one thread per step hoists the
//    fp64 trig (correctly rounded double-double sincos) and the transform, and
//    builds a per-(step, 32-point chunk) 2-D cull mask in fp32 with a proven
//    margin (generalises the x-only row cull of engine.py:272-287); live steps
//    are compacted in time order. Phase 2: lane = live step (tilt: two
//    consecutive live steps), warp = (group of live steps, 32-point chunk);
//    per point the affine transform in the exact reference / extended-model
//    op order, the cell index from an fma + magic-number add (near-boundary
//    points deferred to an exact fix-up with the reference's IEEE division),
//    a time-neighbour run filter through lane shuffles, and RED.MIN on
//    order-preserving u64 keys. ONE: the job descriptor is a by-value kernel
//    parameter (constant-bank operands).
//  * decode / areal pass1+pass2 / plane passes / profiles / graymap:
//    deterministic fixed-partition warp-shuffle + block reductions and
//    HBM-streaming kernels (roughness.py:76-188, surface_io.py:100-131).
//  * microbenchmarks for the fp64 and RED.MIN roofline denominators.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <string>

#include "msurf.h"
#include "msurf_trig.cuh"

namespace {

// Sweep CTA shapes (measured on configs 1-5). Batched job
// arrays and the tilt mode: one warp per CTA over a 64-step tile (two phase-1
// rounds, no CTA-wide barrier). Single non-tilt surfaces (configs 1, 4): four
// warps over 128 steps (fewer, larger CTAs balance better there).
constexpr int kBatchTile = 64, kBatchThreads = 32;   // msurf_sweep (job arrays)
constexpr int kTiltTile = 64, kTiltThreads = 32;     // msurf_sweep_job, EXT_TILT
constexpr int kWideTile = 128, kWideThreads = 128;   // msurf_sweep_job, REF / EXT
constexpr int kCapThreads = 256;                     // msurf_sweep_job_capped (EXT_TILT, 64-step tiles)
#ifndef MSURF_STAGE_THREADS
#define MSURF_STAGE_THREADS 64
#endif
constexpr int kStageThreads = MSURF_STAGE_THREADS;   // staged phase-1 CTAs (64-step tiles)
#ifndef MSURF_MIN_BLOCKS_ONE
#define MSURF_MIN_BLOCKS_ONE 32  // 1-warp CTAs with a by-value job: 64 registers (no spills since the folded locate)
#endif
#ifndef MSURF_MIN_BLOCKS
#define MSURF_MIN_BLOCKS 24  // 1-warp CTAs with the job array: 80 registers
#endif

// CTAs per SM a sweep variant's register budget is sized for
constexpr int sweep_min_blocks(bool one, int threads) {
  return threads == 32 ? (one ? MSURF_MIN_BLOCKS_ONE : MSURF_MIN_BLOCKS) : (one ? 8 : 6) * (128 / threads);
}

constexpr int kThreads = 256;      // reduction / stream kernels
constexpr int kWarps = kThreads / 32;
#ifndef MSURF_LANE_POINT
#define MSURF_LANE_POINT 1  // extended modes: phase 2 with lane = edge point (see kLanePoint)
#endif
#ifndef MSURF_PAIR_STEPS
#define MSURF_PAIR_STEPS 2  // 0: never, 1: always, 2: tilt mode only (see kPairSteps)
#endif
#ifndef MSURF_KUNROLL
#define MSURF_KUNROLL 8
#endif
#ifndef MSURF_TILE_CULL
#define MSURF_TILE_CULL 1  // tile-level chunk pre-cull before phase 1 (see kTileCull)
#endif
#ifndef MSURF_CAP_SHIFT
#define MSURF_CAP_SHIFT 5  // surface-cap tiles of (1 << shift)^2 nodes
#endif
constexpr int kCapShift = MSURF_CAP_SHIFT, kCapTile = 1 << kCapShift;
#ifndef MSURF_SHORT_LAUNCH
#define MSURF_SHORT_LAUNCH 3e8  // step-points of a (pass, tooth) launch below which it is "short"
#endif
constexpr double kShortLaunch = MSURF_SHORT_LAUNCH;
#ifndef MSURF_TILE_CULL_ALL
#define MSURF_TILE_CULL_ALL 1  // ... also for by-value REF / EXT launches (A/B knob)
#endif
constexpr int kKUnroll = MSURF_KUNROLL;

thread_local std::string g_err;

int set_err(const std::string& s) {
  g_err = s;
  return 1;
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_err(std::string(what) + ": " + cudaGetErrorString(e));
  return 0;
}

// ----------------------------------------------------------- key encoding
// Order-preserving map fp64 -> u64 (unsigned compare == IEEE compare for
// non-NaN; -0 is canonicalised to +0 first, IEEE treats them equal).
__device__ __forceinline__ uint64_t enc_key_raw(double z) {
  // key = bits ^ (sign ? ~0 : 2^63) on the two 32-bit halves: 3 integer ops
  const unsigned hi = (unsigned)__double2hiint(z), lo = (unsigned)__double2loint(z);
  const unsigned sgn = (unsigned)((int)hi >> 31);
  return ((uint64_t)(hi ^ (sgn | 0x80000000u)) << 32) | (uint64_t)(lo ^ sgn);
}
__device__ __forceinline__ uint64_t enc_key(double z) {
  return enc_key_raw(__dadd_rn(z, 0.0));  // -0 -> +0 first (IEEE treats them equal)
}
__device__ __forceinline__ double dec_key(uint64_t k) {
  const uint64_t b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)b);
}

// ---------------------------------------------------------- cell location
// Reference: idx = floor((w - lo)/dd + 0.5) with a true IEEE division
// (engine.py:298-300, surface_grid.py:85-86).
// Fast path: tq = fma(w, 1/dd, 0.5 - lo/dd) differs from the reference's
// RN(RN((w-lo)/dd) + 0.5) by < 2^-30 while |w/dd|, |lo/dd|, |tq| < 2^18
// (host-checked grid bound). Adding 1.5*2^20 rounds tq to a multiple of
// 2^-32: for |tq| < 2^19 the high word then holds exponent 1043 and
// floor(tq) + 2^19 in its 20 mantissa bits, and the low word is the fraction
// in units of 2^-32. So floor = hi - (1043 << 20 | 2^19) (any other exponent
// means |tq| >= 2^19, i.e. far outside every supported grid, and lands out
// of range by construction), and "within 2^-29 of an integer" is
// (lo + 8) < 16 unsigned. Only those rare near-boundary points take the exact
// reference sequence: bit-identical indices at two DP ops per axis.
constexpr int kMagicHi = (1043 << 20) | (1 << 19);

__device__ __noinline__ int cell_index_exact(double w, double lo, double dd) {
  const double tq = __dadd_rn(__ddiv_rn(__dsub_rn(w, lo), dd), 0.5);
  return __double2int_rz(floor(tq));  // saturates far outside; range checks reject
}

// Z-map key address of node (i, jj) (jj relative to the job's j_lo), row
// major. (4x4-node blocks, one 128-B line each, were measured: config 4's
// RED.MIN touch 27.4 -> 19.1 lines per instruction but its sweep only gains
// 2 %, config 3's lane = point REDs touch more lines.)
template <int MODE>
__device__ __forceinline__ int key_idx(int i, int jj, int ldk) {
  return i * ldk + jj;
}

// Fire-and-forget global atomic min (RED.E.MIN.64): the explicit .global
// form avoids the generic-address shared-memory fallback atomicMin compiles to.
// No "memory" clobber: nothing in a sweep reads the keys back (later kernels
// do, after the launch boundary), and a clobber would pin every later
// shared-memory read of the point loop (the next points' records) behind the
// RED, serialising the unrolled iterations. MSURF_RED_CLOBBER=1 restores it
// (A/B only).
#ifndef MSURF_RED_CLOBBER
#define MSURF_RED_CLOBBER 0
#endif
#if MSURF_RED_CLOBBER
#define MSURF_RED_MEM : "memory"
#else
#define MSURF_RED_MEM
#endif
__device__ __forceinline__ void red_min_u64(unsigned long long* p, unsigned long long v) {
#ifdef MSURF_NO_RED  // timing experiment only: the RED replaced by a never-taken store
  if (v == 1ull) *p = v;
#else
  asm volatile("red.relaxed.gpu.global.min.u64 [%0], %1;" ::"l"(p), "l"(v) MSURF_RED_MEM);
#endif
}


// predicated form: no branch around the RED
__device__ __forceinline__ void red_min_u64_if(unsigned long long* p, unsigned long long v, bool pred) {
#ifdef MSURF_NO_RED
  if (pred && v == 1ull) *p = v;
  return;
#endif
  asm volatile(
      "{ .reg .pred q; setp.ne.u32 q, %2, 0; @q red.relaxed.gpu.global.min.u64 [%0], %1; }" ::"l"(p),
      "l"(v), "r"((unsigned)pred) MSURF_RED_MEM);
}

__device__ __forceinline__ unsigned warp_sum_u(unsigned v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// RED trace (MSURF_SWEEP_TRACE, roofline only): every warp-wide RED.MIN of
// the main point loops appends one record of 32 key offsets from
// g_trace_base (0xffffffff = lane inactive). msurf_red_lines histograms the
// records by the number of distinct 128-byte lines they touch, which with the
// per-shape RED.MIN rates of msurf_microbench(32 + L) gives the time the
// sweep's own RED stream needs at the L2 atomic units' measured throughput.
// The near-boundary fix-up REDs (~1e-9 of points) are not traced.
__device__ unsigned* g_trace;                    // [cap][32] offsets
__device__ unsigned long long g_trace_cap;       // records
__device__ unsigned long long* g_trace_ctr;      // [0] records issued, [1] active lanes
__device__ const unsigned long long* g_trace_base;

__device__ __forceinline__ void trace_red(const unsigned long long* p, bool pred, int lane) {
  const unsigned m = __ballot_sync(0xffffffffu, pred);
  if (!m) return;
  unsigned long long slot = 0;
  if (lane == 0) {
    slot = atomicAdd(g_trace_ctr, 1ull);
    atomicAdd(g_trace_ctr + 1, (unsigned long long)__popc(m));
  }
  slot = __shfl_sync(0xffffffffu, slot, 0);
  if (slot < g_trace_cap) g_trace[slot * 32 + lane] = pred ? (unsigned)(p - g_trace_base) : 0xffffffffu;
}

// 2-D box test of one tool-frame box [xl xh yl yh zl zh] rotated by (c, s),
// after the lead tilt, in fp32 against a window given by its centre
// offsets (ox, oy = tool offset - window centre) and half-widths (hx, hy)
// that already include the caller's margin: every term is bounded by the box
// extent R and the offsets, so the fp32 result is within a few ulp(R + |o|)
// of the exact one; callers add >= 4e-6 (R + |o|) + 1e-6 mm to hx, hy.
template <int MODE>
__device__ __forceinline__ bool tool_box_hits_f32(const float* b, float c, float sn, float ox, float oy, float hx,
                                                  float hy, float tilt_c, float tilt_s) {
  const float ns = -sn;
  const float xl = b[0], xh = b[1], yl = b[2], yh = b[3];
  const float x_lo = fminf(c * xl, c * xh) + fminf(sn * yl, sn * yh) + ox;
  const float x_hi = fmaxf(c * xl, c * xh) + fmaxf(sn * yl, sn * yh) + ox;
  float v_lo = fminf(ns * xl, ns * xh) + fminf(c * yl, c * yh);
  float v_hi = fmaxf(ns * xl, ns * xh) + fmaxf(c * yl, c * yh);
  if (MODE == MSURF_MODE_EXT_TILT) {
    const float a1 = tilt_c * v_lo, a2 = tilt_c * v_hi;
    const float b1 = tilt_s * b[4], b2 = tilt_s * b[5];
    v_lo = fminf(a1, a2) - fmaxf(b1, b2);
    v_hi = fmaxf(a1, a2) - fminf(b1, b2);
  }
  return (x_hi >= -hx) & (x_lo <= hx) & (v_hi + oy >= -hy) & (v_lo + oy <= hy);
}

// one edge point under one lane's step transform: the magic-number high
// words of both cell coordinates, the near-boundary flag, the deposit key and
// (tilt) the key's high word for the neighbour comparisons. REF keeps the
// workpiece x', y' in the reference's exact op order; the extended modes fold
// the offsets into the cell coordinate (see eval_point).
struct PointEval {
  double xw, yw;
  int hi_x, hi_y;
  bool near;
  uint64_t key;
  unsigned zh;  // high word of the order-preserving key (tilt neighbour compares)

  // cell coordinates from mx = fma(a, inv, c) + 1.5*2^20: floor and fraction
  // straight from the bits (see kMagicHi)
  __device__ __forceinline__ PointEval cells(double ax, double cx, double ay, double cy, double inv) {
    const double mx = __dadd_rn(__fma_rn(ax, inv, cx), 0x1.8p20);
    const double my = __dadd_rn(__fma_rn(ay, inv, cy), 0x1.8p20);
    hi_x = __double2hiint(mx);
    hi_y = __double2hiint(my);
    near = (((unsigned)__double2loint(mx) + 8u) < 16u) | (((unsigned)__double2loint(my) + 8u) < 16u);
#ifdef MSURF_FORCE_NEAR
    near = true;  // test build: every point takes the exact deferred path
#endif
    return *this;
  }
};

// Row transform of one live step as the phase-2 lanes hold it: REF the eight
// composite coefficients; EXT / tilt (c, s, cxp, cyp) with the step's x and y
// offsets folded into the cell-coordinate constants, cxp = fma(xoff, inv, cx0)
// and cyp = fma(ty, inv, cy0) (the offsets themselves stay in shared memory
// for the exact path).
//
// Fast cell location of the extended modes: mx = fma(u, inv, cxp) + 1.5*2^20
// with u = fma(c, x, s*y) is (u + xoff - x_min)/dd + 0.5 up to a few 1e-13
// cells (fma instead of the reference's rounded products, the folded
// constant's rounding), far inside the +-8*2^-32 cell window that flags a
// point as near a boundary; flagged points are re-located with the exact
// reference arithmetic (exact_xy + cell_index_exact). The key is exact: EXT's
// is precomputed, tilt's z' uses the model's own fused v.
template <int MODE>
__device__ __forceinline__ PointEval eval_point(const double4 pt, const double* r, double inv, double cx0,
                                                double cy0, double tilt_c, double tilt_s) {
  PointEval e;
  e.zh = 0u;
  if (MODE == MSURF_MODE_REF) {
    // engine.py:289-296: xw = ((m00*xp + m01*yp) + m02*zp) + m03
    e.xw = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(r[0], pt.x), __dmul_rn(r[1], pt.y)), __dmul_rn(r[2], pt.z)),
                     r[3]);
    e.yw = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(r[4], pt.x), __dmul_rn(r[5], pt.y)), __dmul_rn(r[6], pt.z)),
                     r[7]);
    e.key = (uint64_t)__double_as_longlong(pt.w);
    return e.cells(e.xw, cx0, e.yw, cy0, inv);
  }
  const double uu = __fma_rn(r[0], pt.x, __dmul_rn(r[1], pt.y));
  const double vv = __fma_rn(r[0], pt.y, -__dmul_rn(r[1], pt.x));
  if (MODE == MSURF_MODE_EXT_TILT) {
    // lead-tilt model: z' = fma(sin(tau), v, cos(tau) z + zoff),
    // y' - ty = fma(cos(tau), v, -sin(tau) z); pt = (x, y, sin(tau) z, cos(tau) z + zoff)
    const double zz = __fma_rn(tilt_s, vv, pt.w);
    e.key = enc_key_raw(zz);  // pt.w is never -0 (host-canonical), so neither is zz
    e.zh = (unsigned)(e.key >> 32);
    return e.cells(uu, r[2], __fma_rn(tilt_c, vv, -pt.z), r[3], inv);
  }
  e.key = (uint64_t)__double_as_longlong(pt.z);
  return e.cells(uu, r[2], vv, r[3], inv);
}

// exact workpiece x', y' of an extended-mode point (the deferred near-boundary
// path): EXT in the reference's op order on tool-frame points (u = c x + s y,
// v = -s x + c y), so all-zero extensions reproduce the reference bits; tilt
// in the model's fused form
template <int MODE>
__device__ __forceinline__ void exact_xy(const double4 pt, double c, double s, double xoff, double ty,
                                         double tilt_c, double& xw, double& yw) {
  if (MODE == MSURF_MODE_EXT_TILT) {
    const double uu = __fma_rn(c, pt.x, __dmul_rn(s, pt.y));
    const double vv = __fma_rn(c, pt.y, -__dmul_rn(s, pt.x));
    xw = __dadd_rn(uu, xoff);
    yw = __dadd_rn(__fma_rn(tilt_c, vv, -pt.z), ty);
  } else {
    const double uu = __dadd_rn(__dmul_rn(c, pt.x), __dmul_rn(s, pt.y));
    const double vv = __dadd_rn(__dmul_rn(-s, pt.x), __dmul_rn(c, pt.y));
    xw = __dadd_rn(uu, xoff);
    yw = __dadd_rn(vv, ty);
  }
}

// Time-neighbour pre-reduction across lanes (consecutive live steps of one
// point): within a run of lanes whose point sits in one cell only the run's
// minimum deposits. Constant z' (REF/EXT): the run's first lane. Tilt: lanes
// that are a local minimum (< predecessor, <= successor).
template <int MODE>
__device__ __forceinline__ void dedupe(int lane, int idx, bool inside, unsigned zh, bool& dep) {
  const int idx_prev = __shfl_up_sync(0xffffffffu, idx, 1);
  if (MODE == MSURF_MODE_EXT_TILT) {
    // Compare the high words of the order-preserving keys: zh > zh_neighbour
    // proves z' > z'_neighbour, so a lane is skipped only when a same-cell
    // neighbour is provably lower, and every chain of skips ends at a
    // deposited lane whose z' is lower still (equal high words keep both
    // deposits). Lane 0 / lane 31 get their own values back from the edge
    // shuffles, which never skip: no lane test needed.
    const unsigned zh_prev = __shfl_up_sync(0xffffffffu, zh, 1);
    const int idx_next = __shfl_down_sync(0xffffffffu, idx, 1);
    const unsigned zh_next = __shfl_down_sync(0xffffffffu, zh, 1);
    dep = inside & !((idx == idx_prev) & (zh > zh_prev)) & !((idx == idx_next) & (zh > zh_next));
  } else {
    dep = inside & ((lane == 0) | (idx != idx_prev));
  }
}

// advance a warp's (group, chunk) unit cursor by `warps` units
template <int WARPS>
__device__ __forceinline__ void next_unit(int& g, int& q, int nchunk) {
  q += WARPS;
  while (q >= nchunk) {
    q -= nchunk;
    ++g;
  }
}

// tile index inside a job -> (pass, tooth, step tile). MSURF_TILE_ORDER 0:
// pass-major, then tooth, then time (consecutive CTAs = consecutive step
// tiles of one tooth); 1: pass-major, then time, then tooth (the teeth of one
// step tile are adjacent, so the CTAs in flight cover a narrower time window)
#ifndef MSURF_TILE_ORDER
#define MSURF_TILE_ORDER 0
#endif
__device__ __forceinline__ void tile_coords(unsigned loc, unsigned nst, int teeth, int& pass, int& tooth, int& st) {
  if (MSURF_TILE_ORDER == 0) {
    const unsigned rem = loc / nst;
    st = (int)(loc - rem * nst);
    tooth = (int)(rem % (unsigned)teeth);
    pass = (int)(rem / (unsigned)teeth);
  } else {
    const unsigned per_pass = nst * (unsigned)teeth;
    pass = (int)(loc / per_pass);
    const unsigned r = loc - (unsigned)pass * per_pass;
    st = (int)(r / (unsigned)teeth);
    tooth = (int)(r - (unsigned)st * (unsigned)teeth);
  }
}

// tile pre-cull: the tooth box at the tile's mid angle and mid feed position,
// widened by the largest displacement any of its points makes within the
// tile (rotation: arc <= Rt * |dtheta|; feed: |v_f| dt/2 per step). A tile
// the box cannot reach is skipped before any per-step work — for windowed
// strips and narrow grids most tiles are (config 3: ~80 %). Conservative like
// the per-step pre-cull (same fp32 margins). Jobs with host trig tables or a
// trajectory record keep every tile.
template <int MODE, int TILE>
__device__ __forceinline__ bool tile_may_hit(const msurf_job& J, int pass, int tooth, int st) {
  if (J.trig_table || (J.traj && pass == 0)) return true;
  const int nchunk = (J.points + 31) >> 5;
  const float rt_f = __ldg(reinterpret_cast<const float*>(J.chunk_f32) + (long long)tooth * nchunk * 8 + 5);
  float box_f[6];
#pragma unroll
  for (int k = 0; k < 6; ++k) box_f[k] = (float)J.tooth_box[tooth * 6 + k];
  const double dd = J.spacing;
  const long long s0 = J.step_lo + (long long)st * TILE;
  const long long s1 = min(s0 + (long long)TILE, (long long)J.step_hi) - 1;
  const double half_t = 0.5 * (double)(s1 - s0) * J.dt;
  const double tm = J.t_start + (0.5 * (double)(s0 + s1)) * J.dt;
  const double th = J.tooth_base[tooth] - J.omega * tm;
  const double wxc = J.x_min + 0.5 * (double)J.m * dd, wxh = 0.5 * (double)J.m * dd + 1.5 * dd;
  const double wyc = J.y_min + 0.5 * (double)(J.j_lo + J.j_hi) * dd;
  const double wyh = 0.5 * (double)(J.j_hi - J.j_lo) * dd + 1.5 * dd;
  const double kd = rint(th * MSURF_TWO_OVER_PI);
  const double r = __fma_rn(-kd, MSURF_PIO2_2, __fma_rn(-kd, MSURF_PIO2_1, th));
  float sf, cf;
  __sincosf((float)r, &sf, &cf);
  const int quad = ((int)(long long)kd) & 3;
  float ca = cf, sa = sf;
  if (quad == 1) { ca = -sf; sa = cf; }
  else if (quad == 2) { ca = -cf; sa = -sf; }
  else if (quad == 3) { ca = sf; sa = -cf; }
  const float oxf = (float)(J.pass_x0[pass] - wxc);
  const float oyf = (float)(J.y0 + J.feed_speed * tm - wyc);
  const float rot = (float)(fabs(J.omega) * half_t * (double)rt_f);
  const float feed = (float)(fabs(J.feed_speed) * half_t);
  const float mg = (float)(1e-4 + fabs(J.vib_amp)) + 4e-6f * (rt_f + fabsf(oxf) + fabsf(oyf)) + 1e-6f +
                   1.001f * rot + 1e-6f;
  return tool_box_hits_f32<MODE>(box_f, ca, sa, oxf, oyf, (float)wxh + mg, (float)wyh + mg + 1.001f * feed,
                                 (float)J.tilt_c, (float)J.tilt_s);
}

// One phase-2 unit of the paired-step (tilt) loop: chunk q's up-to-32 points
// under the lane's two consecutive live steps A, B (transforms ra / rb, the
// chunk live at them: on_a / on_b; xa / xb -> each step's (x offset, feed
// position) for the exact path). Called by the sweep kernel on its own
// shared-memory rows and by sweep_units_kernel on staged ones.
template <int MODE, int DIAG>
__device__ __forceinline__ void pair_unit(const msurf_job& J, const double4* __restrict__ pts, double4* ptstage,
                                          const double* ra, const double* rb, bool on_a, bool on_b,
                                          const double* xrows, int xstride, int rta, int rtb, int q, int npts, int lane,
                                          double inv, double cx0, double cy0, unsigned span_i, unsigned span_j,
                                          int jbias, int j_lo, int ldk, unsigned long long* __restrict__ keys,
                                          double tilt_c, double tilt_s, double dd, unsigned& n_dep, unsigned& n_atom) {
  const int ibias_a = on_a ? kMagicHi : kMagicHi - (1 << 30);
  const int ibias_b = on_b ? kMagicHi : kMagicHi - (1 << 30);
  const int p_end = min(32, npts - q * 32);
  // stage the chunk's 32 point records (1 KB, coalesced) for broadcast
  // reads; slots past the chunk's end hold zeros (finite, masked below)
  __syncwarp();
  {
    double4 v = make_double4(0.0, 0.0, 0.0, 0.0);
    if (lane < p_end) {
      const double2* src = reinterpret_cast<const double2*>(pts + q * 32 + lane);
      const double2 a = __ldg(src), b = __ldg(src + 1);
      v = make_double4(a.x, a.y, b.x, b.y);
    }
    ptstage[lane] = v;
  }
  __syncwarp();
  // Near-boundary points (probability ~1e-9 each) are not resolved inline:
  // they are flagged, kept out of the neighbour comparisons (treated as
  // outside), and deposited after the chunk with the exact reference index
  // — an extra deposit is always safe, a skipped one never is.
  bool anynear = false;
  // one point per iteration evaluated under both of the lane's steps (two
  // independent fp64 chains). Neighbours in time: A's predecessor is the
  // previous lane's B, B's successor the next lane's A (two shuffles each),
  // A-B within the lane in registers. The edge lanes get their own values
  // back from the shuffles, i.e. compare with their other step, which is a
  // neighbour anyway: no lane tests in the tilt filter.
#pragma unroll kKUnroll
  for (int k = 0; k < p_end; ++k) {
    const double4 pt = ptstage[k];
    PointEval ea = eval_point<MODE>(pt, ra, inv, cx0, cy0, tilt_c, tilt_s);
    PointEval eb = eval_point<MODE>(pt, rb, inv, cx0, cy0, tilt_c, tilt_s);
    const int ia = ea.hi_x - ibias_a, ja = ea.hi_y - jbias;
    const int ib = eb.hi_x - ibias_b, jb = eb.hi_y - jbias;
    anynear |= (ea.near & on_a) | (eb.near & on_b);
    const bool in_a = ((unsigned)ia <= span_i) & ((unsigned)ja <= span_j) & !ea.near;
    const bool in_b = ((unsigned)ib <= span_i) & ((unsigned)jb <= span_j) & !eb.near;
    const int idx_a = in_a ? key_idx<MODE>(ia, ja, ldk) : -1;
    const int idx_b = in_b ? key_idx<MODE>(ib, jb, ldk) : -1;
    const int idx_bp = __shfl_up_sync(0xffffffffu, idx_b, 1);  // A's predecessor (lane 0: own B)
    bool dep_a, dep_b;
    if (MODE == MSURF_MODE_EXT_TILT) {
      const unsigned zh_bp = __shfl_up_sync(0xffffffffu, eb.zh, 1);
      const int idx_an = __shfl_down_sync(0xffffffffu, idx_a, 1);  // B's successor (lane 31: own A)
      const unsigned zh_an = __shfl_down_sync(0xffffffffu, ea.zh, 1);
      const bool ab = idx_a == idx_b;
      dep_a = in_a & !((idx_a == idx_bp) & (ea.zh > zh_bp)) & !(ab & (ea.zh > eb.zh));
      dep_b = in_b & !(ab & (eb.zh > ea.zh)) & !((idx_b == idx_an) & (eb.zh > zh_an));
    } else {
      // constant z' per point: only each run's first step deposits
      dep_a = in_a & ((lane == 0) | (idx_a != idx_bp));
      dep_b = in_b & (idx_b != idx_a);
    }
    if (DIAG) {
      n_dep += (unsigned)in_a + (unsigned)in_b;
      n_atom += (unsigned)dep_a + (unsigned)dep_b;
    }
    red_min_u64_if(keys + idx_a, (unsigned long long)ea.key, dep_a);
    red_min_u64_if(keys + idx_b, (unsigned long long)eb.key, dep_b);
    if (DIAG == 2) {
      trace_red(keys + idx_a, dep_a, lane);
      trace_red(keys + idx_b, dep_b, lane);
    }
  }
  if (__builtin_expect(__any_sync(0xffffffffu, anynear), 0)) {
    for (int k = 0; k < p_end; ++k) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const double4 pt = ptstage[k];
        PointEval e = eval_point<MODE>(pt, h ? rb : ra, inv, cx0, cy0, tilt_c, tilt_s);
        if (!(e.near & (h ? on_b : on_a))) continue;
        if (MODE != MSURF_MODE_REF) {
          const int sl = h ? rtb : rta;
          exact_xy<MODE>(pt, h ? rb[0] : ra[0], h ? rb[1] : ra[1], xrows[sl * xstride + 4], xrows[sl * xstride + 5],
                         tilt_c, e.xw, e.yw);
        }
        const int ie = cell_index_exact(e.xw, J.x_min, dd);
        const int je = cell_index_exact(e.yw, J.y_min, dd) - j_lo;
        const bool in = ((unsigned)ie <= span_i) & ((unsigned)je <= span_j);
        if (in) red_min_u64(keys + key_idx<MODE>(ie, je, ldk), (unsigned long long)e.key);
        if (DIAG) {
          n_dep += in;
          n_atom += in;
        }
      }
    }
  }
}

// One phase-2 unit of the lane = step loop (constant-z' modes and the tilt
// mode's unpaired form): the up-to-32 points of chunk q, already staged in
// ptstage, under the lane's step transform r (live slot rt; `on`: the chunk
// is live at the lane's step). Deposits through the time-neighbour filter;
// near-boundary points re-located exactly afterwards.
template <int MODE, int DIAG, int RW>
__device__ __forceinline__ void step_unit(const msurf_job& J, const double4* ptstage, const double (&r)[RW], int rt,
                                          bool on, int q, int npts, int lane, double inv, double cx0, double cy0,
                                          unsigned span_i, unsigned span_j, int jbias, int j_lo, int ldk,
                                          unsigned long long* __restrict__ keys, double tilt_c, double tilt_s,
                                          double dd, const double* rowv, unsigned& n_dep, unsigned& n_atom) {
  // lanes whose step is not live for this chunk: i index pushed far out of
  // range, so the per-point range test also covers `on`
  const int ibias = on ? kMagicHi : kMagicHi - (1 << 30);
  const int p_end = min(32, npts - q * 32);
        // Near-boundary points (probability ~1e-9 each) are not resolved inline:
        // they are flagged, kept out of the neighbour comparisons (treated as
        // outside), and deposited after the chunk with the exact reference index
        // — an extra deposit is always safe, a skipped one never is.
        bool anynear = false;
        // Two points per iteration with no divergent branch between their
        // evaluations (the compiler interleaves the two dependent fp64 chains).
        // Near-boundary points (probability ~1e-9 each) are not resolved inline:
        // they are flagged, kept out of the neighbour comparisons (treated as
        // outside), and deposited after the chunk with the exact reference index
        // — an extra deposit is always safe, a skipped one never is.
        // 8 iterations (16 points) per unrolled body: the scheduler can overlap
        // one pair's shuffles/REDs with the next pair's fp64 chain (measured:
        // 1.11 -> 1.07 ms on config 2; 16 iterations: slower, i-cache)
  #pragma unroll kKUnroll
        for (int k = 0; k < p_end; k += 2) {
          const int ibias_b = (k + 1 < p_end) ? ibias : kMagicHi - (1 << 30);
          PointEval ea = eval_point<MODE>(ptstage[k], r, inv, cx0, cy0, tilt_c, tilt_s);
          PointEval eb = eval_point<MODE>(ptstage[k + 1], r, inv, cx0, cy0, tilt_c, tilt_s);
          const int ia = ea.hi_x - ibias, ja = ea.hi_y - jbias;
          const int ib = eb.hi_x - ibias_b, jb = eb.hi_y - jbias;
          // near flags of live points (the fast index may be off by one there, so
          // the range test must not filter them)
          anynear |= (ea.near | (eb.near & (k + 1 < p_end))) & on;
          const bool in_a = ((unsigned)ia <= span_i) & ((unsigned)ja <= span_j) & !ea.near;
          const bool in_b = ((unsigned)ib <= span_i) & ((unsigned)jb <= span_j) & !eb.near;
          const int idx_a = in_a ? key_idx<MODE>(ia, ja, ldk) : -1;
          const int idx_b = in_b ? key_idx<MODE>(ib, jb, ldk) : -1;
          bool dep_a, dep_b;
          dedupe<MODE>(lane, idx_a, in_a, ea.zh, dep_a);
          dedupe<MODE>(lane, idx_b, in_b, eb.zh, dep_b);
          if (DIAG) {
            n_dep += (unsigned)in_a + (unsigned)in_b;
            n_atom += (unsigned)dep_a + (unsigned)dep_b;
          }
          red_min_u64_if(keys + idx_a, (unsigned long long)ea.key, dep_a);
          red_min_u64_if(keys + idx_b, (unsigned long long)eb.key, dep_b);
          if (DIAG == 2) {
            trace_red(keys + idx_a, dep_a, lane);
            trace_red(keys + idx_b, dep_b, lane);
          }
        }
        if (__builtin_expect(__any_sync(0xffffffffu, anynear), 0)) {
          for (int k = 0; k < p_end; ++k) {
            const double4 pt = ptstage[k];
            PointEval e = eval_point<MODE>(pt, r, inv, cx0, cy0, tilt_c, tilt_s);
            if (!(e.near & on)) continue;
            if (MODE != MSURF_MODE_REF)
              exact_xy<MODE>(pt, r[0], r[1], rowv[rt * 8 + 4], rowv[rt * 8 + 5], tilt_c, e.xw, e.yw);
            const int ie = cell_index_exact(e.xw, J.x_min, dd);
            const int je = cell_index_exact(e.yw, J.y_min, dd) - j_lo;
            const bool in = on & ((unsigned)ie <= span_i) & ((unsigned)je <= span_j);
            if (in) red_min_u64(keys + key_idx<MODE>(ie, je, ldk), (unsigned long long)e.key);
            if (DIAG) {
              n_dep += in;
              n_atom += in;
            }
          }
        }
}

// staging of a capped (pass, tooth) launch (msurf_job.stage; EXT_TILT, 64-step
// tiles): header [tiles, units, cursor], then per live tile a record
// {n_live; rows[64][6] = (c, s, cxp, cyp, x offset, feed position);
// masks[64][mask_words]}, then the (tile << 32 | chunk) unit list
constexpr long long kStageHeader = 64;
__host__ __device__ inline long long stage_rec_bytes(int mask_words) { return 8 + 64 * 48 + 64 * 8LL * mask_words; }

#pragma nv_diag_suppress 177  // tile_done is unused in the ONE instantiations
template <int MODE, int DIAG, bool ONE, int TILE, int NTHR, bool STAGE = false>
__global__ void __launch_bounds__(NTHR, sweep_min_blocks(ONE, NTHR))
    sweep_kernel(const msurf_job* __restrict__ jobs, int n_jobs,
                 const int64_t* __restrict__ prefix, int mask_words, const __grid_constant__ msurf_job jp,
                 const unsigned long long* __restrict__ list, unsigned* __restrict__ list_count) {
  constexpr int kTileSteps = TILE;               // time steps per CTA
  constexpr int kSweepThreads = NTHR;            // threads per CTA
  // phase-1 rounds of NTHR steps; a CTA wider than its tile (NTHR > TILE: more
  // warps for phase 2) leaves threads >= TILE idle in phase 1
  constexpr int kSubSteps = TILE >= NTHR ? TILE / NTHR : 1;
  constexpr int kSweepWarps = NTHR / 32;
  static_assert((TILE % NTHR == 0 || NTHR % TILE == 0) && NTHR % 32 == 0, "tile / CTA shape");
  constexpr int RW = MODE == MSURF_MODE_REF ? 8 : 4;  // doubles of row data per live step
  // lane = two consecutive live steps (one broadcast point record serves both,
  // half the neighbour exchange in registers): faster for the tilt mode
  // (config 2: 0.99 -> 0.95 ms, config 5: 59.4 -> 54.1 ms) whose neighbour
  // filter needs both neighbours; slower for the constant-z modes (configs 3, 4)
  constexpr bool kPairSteps = MSURF_PAIR_STEPS == 1 || (MSURF_PAIR_STEPS == 2 && MODE == MSURF_MODE_EXT_TILT);
  // lane = one edge point of a 32-point chunk, the warp walking the tile's
  // live steps in time order (warp-uniform transforms broadcast from shared
  // memory): a RED instruction then covers 32 neighbouring edge points — a
  // short radial segment, fewer 128-byte lines — instead of one point's 32
  // positions along its arc (one line per lane at the cutting front), and a
  // point's consecutive steps meet in one lane, so same-cell runs reduce in
  // registers (exact run minimum) before one RED. Measured:
  // faster for the batched flat-end surfaces (config 3: 28.5 -> 16.9 lines per
  // RED, sweep 6.39 -> 5.76 ms); slower for the by-value single surfaces
  // (config 4 4.97 -> 5.36 ms: 6.6-cell point spacing, fewer active lanes per
  // RED) and for the tilt mode (config 5 50.5 -> 66 ms: more instructions per
  // evaluation than the paired-step loop), which keep lane = step.
  constexpr bool kLanePoint = MSURF_LANE_POINT && MODE == MSURF_MODE_EXT && !ONE;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* rowv = reinterpret_cast<double*>(smem_raw);                        // [T][8] by live slot
  uint64_t* masks = reinterpret_cast<uint64_t*>(rowv + kTileSteps * 8);      // [T][W] by thread
  uint64_t* mslot = masks + kTileSteps * mask_words;                         // [T][W] by live slot
  __shared__ msurf_job Js;
  // ONE: a single job passed by value -> its fields are constant-bank operands
  // (no registers, no shared-memory loads); else the CTA's job from the array
  const msurf_job& J = ONE ? jp : Js;
  __shared__ int warp_cnt[kSweepWarps];
  __shared__ unsigned warp_eval[kSweepWarps];
  __shared__ unsigned warp_eng[kSweepWarps];
  __shared__ double4 ptstage[kSweepWarps][32];  // per-warp copy of the current chunk's point records

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  // ONE: one CTA per tile of the by-value job (blockIdx.x = tile). Else
  // persistent CTAs walk the pre-culled tile list (tile_list_kernel): entry =
  // job << 32 | tile index inside the job, taken from a global cursor in list
  // order, so the tiles in flight stay a narrow window of the list (their
  // Z-maps share L2) and uneven tiles balance themselves
  __shared__ unsigned s_i;
  const unsigned list_n = ONE ? 0u : list_count[0];
  long long local = blockIdx.x;
  for (;;) {
  if constexpr (!ONE) {
    if constexpr (kSweepWarps == 1) __syncwarp(); else __syncthreads();  // previous tile done with Js / s_i
    if (tid == 0) s_i = atomicAdd(list_count + 1, 1u);
    if constexpr (kSweepWarps == 1) __syncwarp(); else __syncthreads();
    const unsigned i = s_i;
    if (i >= list_n) return;
    const unsigned long long e = list[i];
    {
      const unsigned long long* src = reinterpret_cast<const unsigned long long*>(jobs + (e >> 32));
      unsigned long long* dst = reinterpret_cast<unsigned long long*>(&Js);
      for (int w = tid; w < (int)(sizeof(msurf_job) / 8); w += kSweepThreads) dst[w] = src[w];
    }
    if constexpr (kSweepWarps == 1) __syncwarp(); else __syncthreads();
    local = (long long)(e & 0xffffffffull);
  }
  {
  // tile -> (pass, tooth, step tile) in 32-bit arithmetic (grids are < 2^31 tiles)
  const unsigned nst = (unsigned)((J.step_hi - J.step_lo + kTileSteps - 1) / kTileSteps);
  int pass, tooth, st;
  tile_coords((unsigned)local, nst, J.tooth_n ? J.tooth_n : J.teeth, pass, tooth, st);
  tooth += J.tooth_lo;  // a launch may cover a tooth range; per-tooth arrays are indexed by the tooth
  const int npts = J.points;
  const int nchunk = (npts + 31) >> 5;
  const double dd = J.spacing;
  const double4* __restrict__ pts = reinterpret_cast<const double4*>(J.pts) + (long long)tooth * npts;

  // this tooth's fp32 chunk cull records (host-made, L1-resident after the
  // first warp touches them) and the bound Rt >= |xc| + |yc| + |yz|
  const float4* __restrict__ cf4 = reinterpret_cast<const float4*>(J.chunk_f32) + (long long)tooth * nchunk * 2;
  const float rt_f = __ldg(reinterpret_cast<const float*>(cf4) + 5);
  float box_f[6];
#pragma unroll
  for (int k = 0; k < 6; ++k) box_f[k] = (float)J.tooth_box[tooth * 6 + k];
  if (ONE && !tile_may_hit<MODE, TILE>(J, pass, tooth, st)) return;  // uniform across the CTA

  const double inv = 1.0 / dd;
  const double cx0 = 0.5 - J.x_min * inv;
  const double cy0 = 0.5 - J.y_min * inv;

  // surface-cap cull (msurf_job.zcap; tilt by-value launches, not in the
  // DIAG=1 counting variant): cell coordinates of a chunk's workpiece box
  // from its window-relative centre, and the tile grid of the job's slab
  const bool zc_on = (DIAG != 1) && ONE && MODE == MSURF_MODE_EXT_TILT && J.zcap != nullptr;
  float zc_k = 0.f, zc_bi = 0.f, zc_bj = 0.f;
  int zc_imax = 0, zc_jmax = 0, zc_tw = 0;
  if (zc_on) {
    const double wxc0 = J.x_min + 0.5 * (double)J.m * dd;
    const double wyc0 = J.y_min + 0.5 * (double)(J.j_lo + J.j_hi) * dd;
    zc_k = (float)inv;
    zc_bi = (float)((wxc0 - J.x_min) * inv + 0.5);
    zc_bj = (float)((wyc0 - J.y_min) * inv + 0.5 - (double)J.j_lo);
    zc_imax = (int)J.m;
    zc_jmax = (int)(J.j_hi - J.j_lo);
    zc_tw = (zc_jmax >> kCapShift) + 1;
  }

  // ---------------- tile-level chunk pre-cull (tilt mode, not in the DIAG=1
  // counting variant): every chunk's window / stock-height / surface-cap test
  // once per tile, at the tile's mid angle and feed position, widened by the
  // largest motion any step of the tile can make — rotation: the chunk centre
  // moves <= (|xc| + |yc|) |omega| half_t; feed: |v_f| half_t; vibration:
  // |amp| — plus the float-sincos error and fp32 margins five times the
  // per-step ones, so the tile mask is a superset of every step's mask (caps
  // read earlier are higher ones). Phase 1 then tests only the tile's chunks,
  // and a tile whose mask is empty skips its rows, double-double sincos
  // included. Ball-end raster tiles are mostly empty: a tooth over the stock
  // top or over an already cut region cuts nothing for 64 steps.
  // by-value surfaces of every mode (a config-4 sub-strip's window leaves most
  // chunks of a tile dead); the batched small surfaces (config 3) sit under
  // the whole tool, so there the per-tile pass is pure overhead (measured +4 %)
  constexpr bool kTileCull = MSURF_TILE_CULL && DIAG != 1 && (MODE == MSURF_MODE_EXT_TILT || (ONE && MSURF_TILE_CULL_ALL));
  uint64_t* tmask = mslot + kTileSteps * mask_words;  // [W] chunks live somewhere in the tile
  bool tc_on = false;
  if constexpr (kTileCull) {
    tc_on = !J.trig_table && !J.traj;
    if (tc_on) {
      const long long s0 = J.step_lo + (long long)st * kTileSteps;
      const long long s1 = min(s0 + (long long)kTileSteps, (long long)J.step_hi) - 1;
      const double half_t = 0.5 * (double)(s1 - s0) * J.dt;
      const double tm = J.t_start + (0.5 * (double)(s0 + s1)) * J.dt;
      const double th = J.tooth_base[tooth] - J.omega * tm;
      const double kd = rint(th * MSURF_TWO_OVER_PI);
      const double r = __fma_rn(-kd, MSURF_PIO2_2, __fma_rn(-kd, MSURF_PIO2_1, th));
      float sf, cf;
      __sincosf((float)r, &sf, &cf);
      const int quad = ((int)(long long)kd) & 3;
      float ca = cf, sa = sf;
      if (quad == 1) { ca = -sf; sa = cf; }
      else if (quad == 2) { ca = -cf; sa = -sf; }
      else if (quad == 3) { ca = sf; sa = -cf; }
      const double wxc = J.x_min + 0.5 * (double)J.m * dd, wxh = 0.5 * (double)J.m * dd + 1.5 * dd;
      const double wyc = J.y_min + 0.5 * (double)(J.j_lo + J.j_hi) * dd;
      const double wyh = 0.5 * (double)(J.j_hi - J.j_lo) * dd + 1.5 * dd;
      const float oxm = (float)(J.pass_x0[pass] - wxc);
      const float oym = (float)(J.y0 + J.feed_speed * tm - wyc);
      const float rot = (float)(fabs(J.omega) * half_t);               // radians
      const float vib = (float)(1.001 * fabs(J.vib_amp));             // mm, x only
      const float feed = (float)(1.001 * fabs(J.feed_speed) * half_t);  // mm, y only
      const float mgx = 2e-5f * (rt_f + fabsf(oxm) + vib) + 1e-5f;
      const float mgy = 2e-5f * (rt_f + fabsf(oym) + feed) + 1e-5f;
      const float hx = (float)wxh + mgx + vib, hy = (float)wyh + mgy + feed;
      // the per-step test's conventions: no tilt terms outside the tilt mode
      const float tcc = MODE == MSURF_MODE_EXT_TILT ? (float)J.tilt_c : 1.0f;
      const float tsz = MODE == MSURF_MODE_EXT_TILT ? (float)J.tilt_s : 0.0f;
      unsigned* tm32 = reinterpret_cast<unsigned*>(tmask);
      for (int qb = warp * 32; qb < mask_words * 64; qb += kSweepThreads) {
        const int q = qb + lane;
        bool hit = false;
        if (q < nchunk) {
          const float4 a = __ldg(cf4 + 2 * q);
          const float4 bz = __ldg(cf4 + 2 * q + 1);  // yz, Rt, zfloor, z margin
          // centre motion over the tile + sincos error (<= 1e-6 rc) + slack
          const float mv = fmaf(1.01f * rot + 1e-6f, fabsf(a.x) + fabsf(a.y), 1e-4f);
          const float uc = fmaf(ca, a.x, sa * a.y);
          const float vc = fmaf(ca, a.y, -(sa * a.x));
          const float yc = fmaf(tcc, vc, bz.x) + oym;
          hit = (fabsf(uc + oxm) <= hx + a.z + mv) & (fabsf(yc) <= hy + a.w + mv);
          const float zlow = fmaf(tsz, vc, bz.z) - fabsf(tsz) * mv - 1e-5f;
          hit &= zlow <= bz.w;
          if (zc_on && hit) {
            const float ci = fmaf(uc + oxm, zc_k, zc_bi), cj = fmaf(yc, zc_k, zc_bj);
            const float ri = fmaf(a.z + mgx + mv + vib, zc_k, 2.5f), rj = fmaf(a.w + mgy + mv + feed, zc_k, 2.5f);
            const int i0 = max(0, __float2int_rd(ci - ri)) >> kCapShift;
            const int i1 = min(zc_imax, __float2int_rd(ci + ri)) >> kCapShift;
            const int j0 = max(0, __float2int_rd(cj - rj)) >> kCapShift;
            const int j1 = min(zc_jmax, __float2int_rd(cj + rj)) >> kCapShift;
            if ((i1 - i0) <= (5 << (5 - kCapShift)) && (j1 - j0) <= (5 << (5 - kCapShift))) {  // larger: keep (no lookup)
              float cap = -INFINITY;  // empty range: no in-grid cell at all
              for (int ti = i0; ti <= i1; ++ti)
                for (int tj = j0; tj <= j1; ++tj) cap = fmaxf(cap, __ldca(J.zcap + ti * zc_tw + tj));
              hit = zlow <= cap + bz.w;
            }
          }
        }
        tm32[q >> 5] = __ballot_sync(0xffffffffu, hit);  // each 32-chunk block written by one warp
      }
      if constexpr (kSweepWarps == 1) __syncwarp(); else __syncthreads();
      unsigned long long anyw = 0ull;
      for (int w = 0; w < mask_words; ++w) anyw |= tmask[w];
      if (anyw == 0ull) {  // uniform: no step of this tile can deposit
        if constexpr (ONE) return; else goto tile_done;
      }
    }
  }

  // ---------------- phase 1: one thread per time step (kSubSteps rounds of
  // kSweepThreads steps), live steps appended in time order
  int n_live = 0;
  unsigned n_eval_cta = 0, n_eng_cta = 0;
  for (int h = 0; h < kSubSteps; ++h) {
    bool any = false, engaged = false;
    unsigned my_eval = 0;
    double rd[RW];
    {
      const double wx_lo = J.x_min - 1.5 * dd;
      const double wx_hi = J.x_min + (double)J.m * dd + 1.5 * dd;
      const double wy_lo = J.y_min + (double)J.j_lo * dd - 1.5 * dd;
      const double wy_hi = J.y_min + (double)J.j_hi * dd + 1.5 * dd;
      const bool tin = TILE >= NTHR || tid < TILE;
      const long long s = J.step_lo + (long long)st * kTileSteps + h * kSweepThreads + tid;
      uint64_t* my_mask = masks + (tin ? tid : 0) * mask_words;
      if (tin)
        for (int w = 0; w < mask_words; ++w) my_mask[w] = 0ull;
      if (tin && s < J.step_hi) {
        // engine.py:240-241, kinematics.py:77 — one rounding per op, no FMA
        const double t = __dadd_rn(J.t_start, __dmul_rn((double)s, J.dt));
        const double ty = __dadd_rn(J.y0, __dmul_rn(J.feed_speed, t));
        const double th = __dsub_rn(J.tooth_base[tooth], __dmul_rn(J.omega, t));
        const double x0p = J.pass_x0[pass];
        // Cheap conservative pre-cull of the whole tooth with a float sincos
        // (double Cody-Waite reduction, |error| < 1e-6 in c, s -> < 1e-4 mm of
        // position for a 100 mm tool, covered by the extra margin; vibration
        // covered by its amplitude): most rows of a windowed strip, and the
        // rows far from the grid, never pay for the double-double sincos.
        // window centre / half-widths for the fp32 box tests (margins added below)
        const double wxc = 0.5 * (wx_lo + wx_hi), wxh = 0.5 * (wx_hi - wx_lo);
        const double wyc = 0.5 * (wy_lo + wy_hi), wyh = 0.5 * (wy_hi - wy_lo);
        const float oyf = (float)(ty - wyc);
        const float tcf = (float)J.tilt_c, tsf = (float)J.tilt_s;
        bool maybe = true;
        if (!J.trig_table && !(J.traj && pass == 0)) {
          const double kd = rint(th * MSURF_TWO_OVER_PI);
          const double r = __fma_rn(-kd, MSURF_PIO2_2, __fma_rn(-kd, MSURF_PIO2_1, th));
          float sf, cf;
          __sincosf((float)r, &sf, &cf);
          const int quad = ((int)(long long)kd) & 3;
          float ca = cf, sa = sf;
          if (quad == 1) { ca = -sf; sa = cf; }
          else if (quad == 2) { ca = -cf; sa = -sf; }
          else if (quad == 3) { ca = sf; sa = -cf; }
          // float sincos error < 1e-6 -> < 1e-4 mm at 100 mm; fp32 box terms
          // within 4e-6 (Rt + |o|); vibration covered by its amplitude
          const float oxf = (float)(x0p - wxc);
          const float mg = (float)(1e-4 + fabs(J.vib_amp)) + 4e-6f * (rt_f + fabsf(oxf) + fabsf(oyf)) + 1e-6f;
          maybe = tool_box_hits_f32<MODE>(box_f, ca, sa, oxf, oyf, (float)wxh + mg, (float)wyh + mg, tcf, tsf);
        }
        if (maybe) {
          double c, sn;
          if (J.trig_table) {
            c = J.trig_table[(s * J.teeth + tooth) * 2 + 0];
            sn = J.trig_table[(s * J.teeth + tooth) * 2 + 1];
          } else {
            msurf_sincos(th, &sn, &c);
          }
          const double ns = -sn;
          double xoff = x0p;
          if (MODE != MSURF_MODE_REF && J.vib_amp != 0.0) {
            const double sv = J.vib_table ? J.vib_table[s]
                                          : msurf_sin(__dadd_rn(__dmul_rn(J.vib_omega, t), J.vib_phase));
            xoff = __dadd_rn(xoff, __dmul_rn(J.vib_amp, sv));
          }
          if (MODE == MSURF_MODE_REF) {
            // engine.py:257-264 composite coefficients, exact op order
            const double* e = J.tooth_rows + tooth * 8;
            rd[0] = __dadd_rn(__dmul_rn(c, e[0]), __dmul_rn(sn, e[4]));
            rd[1] = __dadd_rn(__dmul_rn(c, e[1]), __dmul_rn(sn, e[5]));
            rd[2] = __dadd_rn(__dmul_rn(c, e[2]), __dmul_rn(sn, e[6]));
            rd[3] = __dadd_rn(__dadd_rn(__dmul_rn(c, e[3]), __dmul_rn(sn, e[7])), xoff);
            rd[4] = __dadd_rn(__dmul_rn(ns, e[0]), __dmul_rn(c, e[4]));
            rd[5] = __dadd_rn(__dmul_rn(ns, e[1]), __dmul_rn(c, e[5]));
            rd[6] = __dadd_rn(__dmul_rn(ns, e[2]), __dmul_rn(c, e[6]));
            rd[7] = __dadd_rn(__dadd_rn(__dmul_rn(ns, e[3]), __dmul_rn(c, e[7])), ty);
            if (J.traj && pass == 0) {
              // engine.py:266-270: min-z edge point of this (step, tooth)
              const double4 pt = pts[J.min_index[tooth]];
              double* tr = J.traj + (s * J.teeth + tooth) * 3;
              tr[0] = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(rd[0], pt.x), __dmul_rn(rd[1], pt.y)),
                                          __dmul_rn(rd[2], pt.z)), rd[3]);
              tr[1] = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(rd[4], pt.x), __dmul_rn(rd[5], pt.y)),
                                          __dmul_rn(rd[6], pt.z)), rd[7]);
              tr[2] = dec_key((uint64_t)__double_as_longlong(pt.w));
            }
          } else {
            rd[0] = c;
            rd[1] = sn;
            rd[2] = xoff;  // folded into cxp / cyp when stored (see eval_point)
            rd[3] = ty;
          }
          {
            // whole-tooth test with the exact angle (the SURVEY P_eng row count),
            // fp32 with the same proven widening as the chunk test below
            const float oxf = (float)(xoff - wxc);
            const float mg = 4e-6f * (rt_f + fabsf(oxf) + fabsf(oyf)) + 1e-6f;
            engaged = tool_box_hits_f32<MODE>(box_f, (float)c, (float)sn, oxf, oyf, (float)wxh + mg,
                                              (float)wyh + mg, tcf, tsf);
          }
          if (engaged) {
            // per-chunk bounding circles: x = c*xc + s*yc + xoff +- rx,
            // y = cos(tau)*(c*yc - s*xc) + yz + ty +- ry, against the window
            // (centre, half-width) widened by 1.5 cells. Evaluated in fp32 (the
            // fp64 pipe is the sweep's bottleneck): every term is bounded by
            // S = |xc| + |yc| + |yz| + |offset| <= Rt + |offset|, the fp32 result
            // is within ~8 ulp(S) < 1e-6 S of the exact one, and the test is
            // widened by 4e-6 S + 1e-6 mm, so it stays a superset of the exact
            // cull (a false positive costs work, never a result).
            const double ox = xoff - wxc;
            const float cf = (float)c, sf = (float)sn;
            const float oxf = (float)ox;
            const float tcc = MODE == MSURF_MODE_EXT_TILT ? tcf : 1.0f;
            const float mgx = 4e-6f * (rt_f + fabsf(oxf)) + 1e-6f, mgy = 4e-6f * (rt_f + fabsf(oyf)) + 1e-6f;
            const float hx = (float)wxh + mgx;
            const float hy = (float)wyh + mgy;
            // stock-height cull (not in the DIAG=1 counting variant, whose deposit
            // count is the oracle's P_in): z' >= sin(tau) v_centre + zfloor + stock
            // for every point of the chunk (planner.chunk_zfloor); a chunk whose
            // bound is at or above the stock top cannot lower any key below the
            // initial height, so skipping it never changes a result. Same fp32
            // margin as the position tests.
            const float tsz = MODE == MSURF_MODE_EXT_TILT ? tsf : 0.0f;
            int zc_last = -1;  // the lane's last cap lookup (tile range key, value)
            float zc_cap = 0.f;
            unsigned kept = 0;
            unsigned long long bits = 0ull;
            bool last_hit = false;
            // chunks to test: the tile mask's (tile pre-cull on) or all of them;
            // walked word by word, bit by bit (warp-uniform: one tile mask)
            for (int w = 0; w < mask_words; ++w) {
            const int rem = nchunk - 64 * w;
            unsigned long long todo = rem >= 64 ? ~0ull : ((1ull << rem) - 1ull);
            if (tc_on) todo &= tmask[w];
            while (todo) {
              const int q = 64 * w + __ffsll((long long)todo) - 1;
              todo &= todo - 1ull;
              const float4 a = __ldg(cf4 + 2 * q);
              const float4 bz = __ldg(cf4 + 2 * q + 1);  // yz, Rt, zfloor, 0
              const float uc = fmaf(cf, a.x, sf * a.y);
              const float vc = fmaf(cf, a.y, -(sf * a.x));
              bool hit = (fabsf(uc + oxf) <= hx + a.z) & (fabsf(fmaf(tcc, vc, bz.x) + oyf) <= hy + a.w);
              const float zmg = bz.w;  // 4e-6 (Rt + |zfloor|) + 1e-6, rounded up on the host (planner.chunk_f32)
              const float zlow = fmaf(tsz, vc, bz.z);  // lowest reachable z' - stock, this step
              if (DIAG != 1) hit &= zlow <= zmg;
              if (zc_on && hit) {
                // surface cap: the highest current height (- stock) over every 32x32
                // tile the chunk's box can touch, +-1.5 cells for the fp32 roundings
                // (~1e-3 cell); an empty range means no in-grid cell at all. The caps
                // may be rewritten meanwhile by a refresh on another stream (L1-cached
                // loads: a stale cap is a higher one, still an upper bound), and
                // consecutive chunks of a step mostly touch the same tiles: the lane
                // reuses its last lookup.
                const float ci = fmaf(uc + oxf, zc_k, zc_bi), cj = fmaf(fmaf(tcc, vc, bz.x) + oyf, zc_k, zc_bj);
                // half-extents: the chunk's radii plus the same fp32 margins as the
                // window test (in mm), plus 1.5 cells for the fp32 cell coordinate
                const float ri = fmaf(a.z + mgx, zc_k, 1.5f), rj = fmaf(a.w + mgy, zc_k, 1.5f);
                const int i0 = max(0, __float2int_rd(ci - ri)) >> kCapShift;
                const int i1 = min(zc_imax, __float2int_rd(ci + ri)) >> kCapShift;
                const int j0 = max(0, __float2int_rd(cj - rj)) >> kCapShift;
                const int j1 = min(zc_jmax, __float2int_rd(cj + rj)) >> kCapShift;
                // exact key of the tile range (tile indices < 2^13, spans <= 3); others uncached
                const bool cacheable = (i1 - i0) >= 0 && (i1 - i0) <= 3 && (j1 - j0) >= 0 && (j1 - j0) <= 3 &&
                                       i0 < 8192 && j0 < 8192;
                const int key = cacheable ? ((i0 << 17) | (j0 << 4) | ((i1 - i0) << 2) | (j1 - j0)) : -2;
                if (key < 0 || key != zc_last) {
                  float cap = -INFINITY;
                  if ((i1 - i0) <= 1 && (j1 - j0) <= 1 && i0 <= i1 && j0 <= j1) {
                    // the usual case, at most 2 x 2 tiles: four independent loads
                    const float* r0 = J.zcap + i0 * zc_tw;
                    const float* r1 = J.zcap + i1 * zc_tw;
                    cap = fmaxf(fmaxf(__ldca(r0 + j0), __ldca(r0 + j1)), fmaxf(__ldca(r1 + j0), __ldca(r1 + j1)));
                  } else {
                    for (int ti = i0; ti <= i1; ++ti)
                      for (int tj = j0; tj <= j1; ++tj) cap = fmaxf(cap, __ldca(J.zcap + ti * zc_tw + tj));
                  }
                  zc_last = key;
                  zc_cap = cap;
                }
                hit = zlow <= zc_cap + zmg;
              }
              // the step's chunk mask in a register, stored once per 64 chunks
              bits |= (unsigned long long)hit << (q & 63);
              if (q == nchunk - 1) last_hit = hit;
            }
            my_mask[w] = bits;
            kept += 32u * (unsigned)__popcll(bits);
            bits = 0ull;
            }
            if (last_hit) kept -= (unsigned)(32 * nchunk - npts);  // the last chunk is partial
            any = kept != 0;
            my_eval = kept;
          }
        }
      }
    }
    // ordered compaction of live steps (keeps time order for the neighbour merge)
    const unsigned bal = __ballot_sync(0xffffffffu, any);
    const unsigned eng = __popc(__ballot_sync(0xffffffffu, engaged));
    my_eval = warp_sum_u(my_eval);
    int base = n_live;
    if constexpr (kSweepWarps == 1) {
      n_live += __popc(bal);
      n_eval_cta += my_eval;
      n_eng_cta += eng;
    } else {
      if (lane == 0) {
        warp_cnt[warp] = __popc(bal);
        warp_eval[warp] = my_eval;
        warp_eng[warp] = eng;
      }
      __syncthreads();
#pragma unroll
      for (int w = 0; w < kSweepWarps; ++w) {
        if (w < warp) base += warp_cnt[w];
        n_live += warp_cnt[w];
        n_eval_cta += warp_eval[w];
        n_eng_cta += warp_eng[w];
      }
      __syncthreads();  // warp_cnt is rewritten by the next round
    }
    if (any) {
      const int slot = base + __popc(bal & ((1u << lane) - 1u));
      for (int w = 0; w < mask_words; ++w) mslot[slot * mask_words + w] = masks[tid * mask_words + w];
      if (MODE == MSURF_MODE_REF) {
#pragma unroll
        for (int k = 0; k < RW; ++k) rowv[slot * 8 + k] = rd[k];
      } else {
        rowv[slot * 8 + 0] = rd[0];
        rowv[slot * 8 + 1] = rd[1];
        rowv[slot * 8 + 2] = __fma_rn(rd[2], inv, cx0);
        rowv[slot * 8 + 3] = __fma_rn(rd[3], inv, cy0);
        rowv[slot * 8 + 4] = rd[2];
        rowv[slot * 8 + 5] = rd[3];
      }
    }
  }
  if constexpr (kSweepWarps == 1) __syncwarp(); else __syncthreads();
  if (n_live == 0) {
    if (tid == 0 && J.counters && n_eng_cta)
      atomicAdd(J.counters + MSURF_CTR_ENGAGED_ROWS, (unsigned long long)n_eng_cta);
    if constexpr (ONE) return; else goto tile_done;
  }
  if constexpr (STAGE) {
    static_assert(ONE && MODE == MSURF_MODE_EXT_TILT && TILE == 64, "staged shape");
    // staged launch: phase 1's rows and masks + the live units out, phase 2 in
    // sweep_units_kernel
    __shared__ unsigned s_slot;
    unsigned char* sbuf = static_cast<unsigned char*>(J.stage);
    unsigned* hdr = reinterpret_cast<unsigned*>(sbuf);
    if (tid == 0) s_slot = atomicAdd(hdr, 1u);
    if constexpr (kSweepWarps == 1) __syncwarp(); else __syncthreads();
    const unsigned slot = s_slot;
    const long long stride = stage_rec_bytes(mask_words);
    unsigned char* rec = sbuf + kStageHeader + (long long)slot * stride;
    if (tid == 0) *reinterpret_cast<unsigned long long*>(rec) = (unsigned long long)n_live;
    double* rr = reinterpret_cast<double*>(rec + 8);
    for (int i = tid; i < n_live * 6; i += kSweepThreads) rr[i] = rowv[(i / 6) * 8 + (i % 6)];
    unsigned long long* rm = reinterpret_cast<unsigned long long*>(rec + 8 + 64 * 48);
    for (int i = tid; i < n_live * mask_words; i += kSweepThreads) rm[i] = mslot[i];
    const long long max_tiles = (J.step_hi - J.step_lo + 63) / 64;
    unsigned long long* units = reinterpret_cast<unsigned long long*>(sbuf + kStageHeader + max_tiles * stride);
    for (int qb = warp * 32; qb < nchunk; qb += kSweepThreads) {
      const int qq = qb + lane;
      bool live = false;
      if (qq < nchunk)
        for (int s2 = 0; s2 < n_live; ++s2) live |= ((mslot[s2 * mask_words + (qq >> 6)] >> (qq & 63)) & 1ull) != 0;
      const unsigned bal = __ballot_sync(0xffffffffu, live);
      if (bal) {
        unsigned base = 0;
        if (lane == 0) base = atomicAdd(hdr + 1, (unsigned)__popc(bal));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (live) units[base + __popc(bal & ((1u << lane) - 1u))] = ((unsigned long long)slot << 32) | (unsigned)qq;
      }
#ifdef MSURF_STAGE_STATS  // experiment only: lane-slot utilisation of the staged units
      if (qq < nchunk) {
        unsigned cnt = 0;
        for (int s2 = 0; s2 < n_live; ++s2) cnt += (unsigned)((mslot[s2 * mask_words + (qq >> 6)] >> (qq & 63)) & 1ull);
        if (cnt && J.counters) {
          atomicAdd(J.counters + MSURF_CTR_DEPOSITS, 64ull);
          atomicAdd(J.counters + MSURF_CTR_ATOMICS, (unsigned long long)cnt);
        }
      }
#endif
    }
    if (tid == 0 && J.counters) {
      atomicAdd(J.counters + MSURF_CTR_LIVE_ROWS, (unsigned long long)n_live);
      atomicAdd(J.counters + MSURF_CTR_EVAL, (unsigned long long)n_eval_cta);
      atomicAdd(J.counters + MSURF_CTR_ENGAGED_ROWS, (unsigned long long)n_eng_cta);
    }
    return;
  }

  // ---------------- phase 2: lane = live step(s), warp walks the 32 points of a chunk
  // unit = (group of consecutive live steps, 32-point chunk). Each lane keeps
  // its step's transform (tilt: its two steps' transforms) in registers; the
  // chunk's point records are staged once in shared memory and read as warp
  // broadcasts. Consecutive live steps of one point sit in neighbouring
  // lanes (or in one lane's pair): the time-neighbour filter skips a deposit
  // only when a same-cell neighbour provably deposits a key that is not
  // higher, so each monotone run of a point through a cell costs one RED.MIN.
  const unsigned span_i = (unsigned)J.m;
  const int j_lo = (int)J.j_lo;
  const unsigned span_j = (unsigned)(J.j_hi - J.j_lo);
  // j index straight from the magic-number high word, already relative to
  // the owned strip: hi - (kMagicHi + j_lo)
  const int jbias = kMagicHi + j_lo;
  const int ldk = (int)J.ld;
  unsigned long long* __restrict__ keys = reinterpret_cast<unsigned long long*>(J.keys);
  const double tilt_c = J.tilt_c, tilt_s = J.tilt_s;
  unsigned n_dep = 0, n_atom = 0;
  // unit = (group of consecutive live steps, chunk q), dealt round-robin to
  // the warps in (g, q) order; the lane's transforms are reloaded only when g
  // changes, and (g, q) advance without a division
  int g = warp / nchunk, q = warp - (warp / nchunk) * nchunk;
  int g_loaded = -1;
  if constexpr (kLanePoint) {
    constexpr int kSlotWords = kTileSteps / 32;
    for (int qc = warp; qc < nchunk; qc += kSweepWarps) {
      // live slots of this chunk (bit = slot, time order)
      unsigned mw[kSlotWords];
      unsigned anyq = 0u;
#pragma unroll
      for (int w = 0; w < kSlotWords; ++w) {
        const int slot = w * 32 + lane;
        const bool on = slot < n_live && ((mslot[slot * mask_words + (qc >> 6)] >> (qc & 63)) & 1ull);
        mw[w] = __ballot_sync(0xffffffffu, on);
        anyq |= mw[w];
      }
      if (!anyq) continue;  // warp-uniform
      const int pidx = qc * 32 + lane;
      const bool pv = pidx < npts;
      double4 pt = make_double4(0.0, 0.0, 0.0, 0.0);
      if (pv) {
        const double2* src = reinterpret_cast<const double2*>(pts + pidx);
        const double2 a = __ldg(src), b = __ldg(src + 1);
        pt = make_double4(a.x, a.y, b.x, b.y);
      }
      // a lane past the tooth's last point: i index pushed far out of range
      const int ibias = pv ? kMagicHi : kMagicHi - (1 << 30);
      int run_idx = -1;                 // cell of the current run (-1: none)
      unsigned long long run_key = 0;   // tilt: minimum key of the run
#pragma unroll
      for (int w = 0; w < kSlotWords; ++w) {
        unsigned m = mw[w];
        while (m) {  // warp-uniform: two live steps per iteration (two independent fp64 chains)
          const int s1 = w * 32 + __ffs(m) - 1;
          m &= m - 1u;
          const bool two = m != 0u;
          const int s2 = two ? w * 32 + __ffs(m) - 1 : s1;
          m &= m - (two ? 1u : 0u);
          const double4 t1 = *reinterpret_cast<const double4*>(rowv + s1 * 8);
          const double4 t2 = *reinterpret_cast<const double4*>(rowv + s2 * 8);
          const double r1[4] = {t1.x, t1.y, t1.z, t1.w};
          const double r2[4] = {t2.x, t2.y, t2.z, t2.w};
          PointEval e1 = eval_point<MODE>(pt, r1, inv, cx0, cy0, tilt_c, tilt_s);
          PointEval e2 = eval_point<MODE>(pt, r2, inv, cx0, cy0, tilt_c, tilt_s);
          const int ia1 = e1.hi_x - ibias, ja1 = e1.hi_y - jbias;
          const int ia2 = e2.hi_x - ibias, ja2 = e2.hi_y - jbias;
          const bool in1 = ((unsigned)ia1 <= span_i) & ((unsigned)ja1 <= span_j) & !e1.near;
          const bool in2 = ((unsigned)ia2 <= span_i) & ((unsigned)ja2 <= span_j) & !e2.near & two;
          const int idx1 = in1 ? key_idx<MODE>(ia1, ja1, ldk) : -1;
          const int idx2 = in2 ? key_idx<MODE>(ia2, ja2, ldk) : -1;
          bool dep1, dep2;
          unsigned long long k1, k2;
          int a1, a2;
          if (MODE == MSURF_MODE_EXT_TILT) {
            // run minimum: a run ends when the cell changes; its minimum deposits then
            const bool brk1 = idx1 != run_idx;
            dep1 = brk1 & (run_idx >= 0);
            a1 = run_idx;
            k1 = run_key;
            run_key = brk1 ? e1.key : (e1.key < run_key ? e1.key : run_key);
            run_idx = idx1;
            const bool brk2 = two & (idx2 != run_idx);
            dep2 = brk2 & (run_idx >= 0);
            a2 = run_idx;
            k2 = run_key;
            if (two) {
              run_key = brk2 ? e2.key : (e2.key < run_key ? e2.key : run_key);
              run_idx = idx2;
            }
          } else {
            // constant z' per point: each run's first evaluation deposits
            dep1 = in1 & (idx1 != run_idx);
            dep2 = in2 & (idx2 != idx1);
            a1 = idx1;
            a2 = idx2;
            k1 = e1.key;
            k2 = e2.key;
            if (two) run_idx = idx2; else run_idx = idx1;
          }
          if (DIAG) {
            n_dep += (unsigned)in1 + (unsigned)in2;
            n_atom += (unsigned)dep1 + (unsigned)dep2;
          }
          red_min_u64_if(keys + a1, k1, dep1);
          red_min_u64_if(keys + a2, k2, dep2);
          if (DIAG == 2) {
            trace_red(keys + a1, dep1, lane);
            trace_red(keys + a2, dep2, lane);
          }
          // near-boundary evaluations (~1e-9 each): the exact reference index, deposited directly
          if (__builtin_expect(__any_sync(0xffffffffu, pv & (e1.near | (e2.near & two))), 0)) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const PointEval& e = h ? e2 : e1;
              const int sl = h ? s2 : s1;
              if (!(pv & e.near & (h == 0 || two))) continue;
              double xw, yw;
              exact_xy<MODE>(pt, rowv[sl * 8 + 0], rowv[sl * 8 + 1], rowv[sl * 8 + 4], rowv[sl * 8 + 5], tilt_c,
                             xw, yw);
              const int ie = cell_index_exact(xw, J.x_min, dd);
              const int je = cell_index_exact(yw, J.y_min, dd) - j_lo;
              const bool in = ((unsigned)ie <= span_i) & ((unsigned)je <= span_j);
              if (in) red_min_u64(keys + key_idx<MODE>(ie, je, ldk), (unsigned long long)e.key);
              if (DIAG) {
                n_dep += in;
                n_atom += in;
              }
            }
          }
        }
      }
      if (MODE == MSURF_MODE_EXT_TILT) {
        const bool dep = run_idx >= 0;  // the chunk's last run
        if (DIAG) n_atom += (unsigned)dep;
        red_min_u64_if(keys + run_idx, run_key, dep);
        if (DIAG == 2) trace_red(keys + run_idx, dep, lane);
      }
    }
  } else if constexpr (kPairSteps) {
    // unit = (group g of 64 consecutive live steps, chunk q); lane l holds the
    // group's steps 2l (A) and 2l+1 (B), so one broadcast point record serves
    // two evaluations and half of the neighbour exchange stays in registers
    const int groups = (n_live + 63) >> 6;
    int rta = 0, rtb = 0;
    double ra[RW], rb[RW];
    for (; g < groups; next_unit<kSweepWarps>(g, q, nchunk)) {
      const int sa = g * 64 + 2 * lane, sb = sa + 1;
      if (g != g_loaded) {  // warp-uniform
        g_loaded = g;
        rta = sa < n_live ? sa : -1;
        rtb = sb < n_live ? sb : -1;
#pragma unroll
        for (int k = 0; k < RW; ++k) {
          ra[k] = rta >= 0 ? rowv[sa * 8 + k] : 0.0;
          rb[k] = rtb >= 0 ? rowv[sb * 8 + k] : 0.0;
        }
      }
      const bool on_a = rta >= 0 && ((mslot[rta * mask_words + (q >> 6)] >> (q & 63)) & 1ull);
      const bool on_b = rtb >= 0 && ((mslot[rtb * mask_words + (q >> 6)] >> (q & 63)) & 1ull);
      if (!__any_sync(0xffffffffu, on_a | on_b)) continue;
      pair_unit<MODE, DIAG>(J, pts, ptstage[warp], ra, rb, on_a, on_b, rowv, 8, rta, rtb, q, npts, lane, inv, cx0,
                            cy0, span_i, span_j, jbias, j_lo, ldk, keys, tilt_c, tilt_s, dd, n_dep, n_atom);
    }
  } else {
    // unit = (group of 32 live steps, chunk q), lane = one step. Only live
    // units are visited: per group the union of its steps' chunk masks
    // (warp-uniform), the live units dealt round-robin to the CTA's warps in
    // (group, chunk) order (a windowed sub-strip leaves most chunks of a step
    // dead, and testing every (group, chunk) pair cost ~8 % of the issue).
    int rt = 0;
    double r[RW];
    const int groups = (n_live + 31) >> 5;
    unsigned u_rank = 0;  // live units seen so far (uniform)
    for (int gg = 0; gg < groups; ++gg) {
      const int slot = gg * 32 + lane;
      const int rtg = slot < n_live ? slot : -1;
      for (int w = 0; w < mask_words; ++w) {
      const unsigned long long mw = rtg >= 0 ? mslot[rtg * mask_words + w] : 0ull;
      unsigned long long live_q = ((unsigned long long)__reduce_or_sync(0xffffffffu, (unsigned)(mw >> 32)) << 32) |
                                  (unsigned long long)__reduce_or_sync(0xffffffffu, (unsigned)mw);
      while (live_q) {
      const int qb = __ffsll((long long)live_q) - 1;
      live_q &= live_q - 1ull;
      if ((u_rank++ % (unsigned)kSweepWarps) != (unsigned)warp) continue;
      const int q = 64 * w + qb;
      if (gg != g_loaded) {  // warp-uniform
        g_loaded = gg;
        rt = rtg;
#pragma unroll
        for (int k = 0; k < RW; ++k) r[k] = rt >= 0 ? rowv[slot * 8 + k] : 0.0;
      }
      const bool on = (mw >> qb) & 1ull;
      const int p_end = min(32, npts - q * 32);
      // stage the chunk's 32 point records (1 KB, coalesced) for broadcast
      // reads; slots past the chunk's end hold zeros (finite, masked below)
      __syncwarp();
      {
        double4 v = make_double4(0.0, 0.0, 0.0, 0.0);
        if (lane < p_end) {
          const double2* src = reinterpret_cast<const double2*>(pts + q * 32 + lane);
          const double2 a = __ldg(src), b = __ldg(src + 1);
          v = make_double4(a.x, a.y, b.x, b.y);
        }
        ptstage[warp][lane] = v;
      }
      __syncwarp();
      step_unit<MODE, DIAG, RW>(J, ptstage[warp], r, rt, on, q, npts, lane, inv, cx0, cy0, span_i, span_j, jbias,
                                j_lo, ldk, keys, tilt_c, tilt_s, dd, rowv, n_dep, n_atom);
      }  // live chunks of the word
      }  // mask words
    }  // groups
  }

  // counters: one atomic per warp
  if (J.counters) {
    if (DIAG) {
      n_dep = warp_sum_u(n_dep);
      n_atom = warp_sum_u(n_atom);
      if (lane == 0) {
        atomicAdd(J.counters + MSURF_CTR_DEPOSITS, (unsigned long long)n_dep);
        atomicAdd(J.counters + MSURF_CTR_ATOMICS, (unsigned long long)n_atom);
      }
    }
    if (tid == 0) {
      atomicAdd(J.counters + MSURF_CTR_LIVE_ROWS, (unsigned long long)n_live);
      atomicAdd(J.counters + MSURF_CTR_EVAL, (unsigned long long)n_eval_cta);
      atomicAdd(J.counters + MSURF_CTR_ENGAGED_ROWS, (unsigned long long)n_eng_cta);
    }
  }
  }
  tile_done:
  if constexpr (ONE) return;
  }
}
#pragma nv_diag_default 177

// tile list of a job array: one thread per tile (job found by binary search
// in the tile prefix), live tiles appended with one atomic per warp; the
// order is not deterministic and need not be (min and the counters commute)
template <int MODE, int TILE>
__global__ void __launch_bounds__(256)
    tile_list_kernel(const msurf_job* __restrict__ jobs, int n_jobs, const int64_t* __restrict__ prefix,
                     long long n_tiles, unsigned long long* __restrict__ list, unsigned* __restrict__ count) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  bool live = false;
  unsigned long long entry = 0;
  if (t < n_tiles) {
    int lo = 0, hi = n_jobs - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (prefix[mid] <= t) lo = mid; else hi = mid - 1;
    }
    const msurf_job& J = jobs[lo];
    const unsigned local = (unsigned)(t - prefix[lo]);
    const unsigned nst = (unsigned)((J.step_hi - J.step_lo + TILE - 1) / TILE);
    int pass, tooth, st;
    tile_coords(local, nst, J.tooth_n ? J.tooth_n : J.teeth, pass, tooth, st);
    tooth += J.tooth_lo;
    live = tile_may_hit<MODE, TILE>(J, pass, tooth, st);
    entry = ((unsigned long long)lo << 32) | local;
  }
  const unsigned bal = __ballot_sync(0xffffffffu, live);
  if (!bal) return;
  const int lane = threadIdx.x & 31;
  unsigned base = 0;
  if (lane == __ffs(bal) - 1) base = atomicAdd(count, (unsigned)__popc(bal));
  base = __shfl_sync(0xffffffffu, base, __ffs(bal) - 1);
  if (live) list[base + __popc(bal & ((1u << lane) - 1u))] = entry;
}

// phase 2 of a staged launch: persistent one-warp CTAs take (tile, chunk)
// units from the list in order through a global cursor, load the tile's
// staged rows and masks (L2) and run pair_unit: the heavy tiles' units spread
// over every warp of the GPU instead of trailing in their own CTA
// MINB: one-warp CTAs per SM the registers are sized for — 32 (64 registers)
// for long (pass, tooth) launches that fill the GPU on their own; 16 (~100
// registers, more of the point loop's fp64 chains in flight per warp) for
// short ones, where fewer, faster warps shorten the launch (measured: config
// 2 0.532 -> 0.508 ms; config 5's long launches lose with 16: 10.67 -> 11.03)
template <int DIAG, int MINB = 32>
__global__ void __launch_bounds__(32, MINB)
    sweep_units_kernel(const __grid_constant__ msurf_job J, int mask_words) {
  constexpr int MODE = MSURF_MODE_EXT_TILT;
  __shared__ double4 ptstage[32];
  const int lane = threadIdx.x & 31;
  unsigned char* sbuf = static_cast<unsigned char*>(J.stage);
  unsigned* hdr = reinterpret_cast<unsigned*>(sbuf);
  const unsigned n_units = hdr[1];
  const long long stride = stage_rec_bytes(mask_words);
  const long long max_tiles = (J.step_hi - J.step_lo + 63) / 64;
  const unsigned long long* units =
      reinterpret_cast<const unsigned long long*>(sbuf + kStageHeader + max_tiles * stride);
  const int tooth = J.tooth_lo;
  const int npts = J.points;
  const double4* __restrict__ pts = reinterpret_cast<const double4*>(J.pts) + (long long)tooth * npts;
  const double dd = J.spacing;
  const double inv = 1.0 / dd;
  const double cx0 = 0.5 - J.x_min * inv;
  const double cy0 = 0.5 - J.y_min * inv;
  const unsigned span_i = (unsigned)J.m;
  const int j_lo = (int)J.j_lo;
  const unsigned span_j = (unsigned)(J.j_hi - J.j_lo);
  const int jbias = kMagicHi + j_lo;
  const int ldk = (int)J.ld;
  unsigned long long* __restrict__ keys = reinterpret_cast<unsigned long long*>(J.keys);
  unsigned n_dep = 0, n_atom = 0;
  // the next unit's index is fetched while the current unit runs (the cursor
  // atomic's round trip was the kernel's largest stall)
  unsigned u_next = 0;
  if (lane == 0) u_next = atomicAdd(hdr + 2, 1u);
  for (;;) {
    const unsigned u = __shfl_sync(0xffffffffu, u_next, 0);
    if (u >= n_units) break;
    if (lane == 0) u_next = atomicAdd(hdr + 2, 1u);
    const unsigned long long e = units[u];
    const unsigned char* rec = sbuf + kStageHeader + (long long)(e >> 32) * stride;
    const int q = (int)(e & 0xffffffffull);
    const int n_live = (int)*reinterpret_cast<const unsigned long long*>(rec);
    const double* rr = reinterpret_cast<const double*>(rec + 8);
    const unsigned long long* rm = reinterpret_cast<const unsigned long long*>(rec + 8 + 64 * 48);
    const int sa = 2 * lane, sb = sa + 1;
    const int rta = sa < n_live ? sa : -1, rtb = sb < n_live ? sb : -1;
    double ra[4], rb[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      ra[k] = rta >= 0 ? __ldcg(rr + sa * 6 + k) : 0.0;
      rb[k] = rtb >= 0 ? __ldcg(rr + sb * 6 + k) : 0.0;
    }
    const bool on_a = rta >= 0 && ((__ldcg(rm + rta * mask_words + (q >> 6)) >> (q & 63)) & 1ull);
    const bool on_b = rtb >= 0 && ((__ldcg(rm + rtb * mask_words + (q >> 6)) >> (q & 63)) & 1ull);
    pair_unit<MODE, DIAG>(J, pts, ptstage, ra, rb, on_a, on_b, rr, 6, rta, rtb, q, npts, lane, inv, cx0, cy0, span_i,
                          span_j, jbias, j_lo, ldk, keys, J.tilt_c, J.tilt_s, dd, n_dep, n_atom);
  }
  if (DIAG && J.counters) {
    n_dep = warp_sum_u(n_dep);
    n_atom = warp_sum_u(n_atom);
    if (lane == 0) {
      atomicAdd(J.counters + MSURF_CTR_DEPOSITS, (unsigned long long)n_dep);
      atomicAdd(J.counters + MSURF_CTR_ATOMICS, (unsigned long long)n_atom);
    }
  }
}

// --------------------------------------------------------------- fill/decode
// HBM streams: 16-byte vector accesses when the surface size is even (every
// BASELINE grid), grid-stride over a capped grid, one y-block row per surface.
__global__ void __launch_bounds__(kThreads)
    fill_kernel(uint64_t* __restrict__ keys, long long count, const double* __restrict__ value) {
  const uint64_t key = enc_key(value[blockIdx.y]);
  uint64_t* base = keys + (long long)blockIdx.y * count;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long t0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if ((count & 1) == 0 && (reinterpret_cast<uintptr_t>(base) & 15) == 0) {
    ulonglong2* b2 = reinterpret_cast<ulonglong2*>(base);
    const ulonglong2 kk = make_ulonglong2(key, key);
    for (long long i = t0; i < count / 2; i += stride) b2[i] = kk;
  } else {
    for (long long i = t0; i < count; i += stride) base[i] = key;
  }
}

__global__ void __launch_bounds__(kThreads)
    decode_kernel(uint64_t* __restrict__ keys, long long count, const double* __restrict__ sent,
                  unsigned long long* __restrict__ machined) {
  uint64_t* base = keys + (long long)blockIdx.y * count;
  const double sentinel = sent[blockIdx.y];
  unsigned cnt = 0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long t0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if ((count & 1) == 0 && (reinterpret_cast<uintptr_t>(base) & 15) == 0) {
    ulonglong2* b2 = reinterpret_cast<ulonglong2*>(base);
    double2* o2 = reinterpret_cast<double2*>(base);
    for (long long i = t0; i < count / 2; i += stride) {
      const ulonglong2 k = b2[i];
      const double2 hv = make_double2(dec_key(k.x), dec_key(k.y));
      o2[i] = hv;
      cnt += (hv.x < sentinel) + (hv.y < sentinel);
    }
  } else {
    double* out = reinterpret_cast<double*>(base);
    for (long long i = t0; i < count; i += stride) {
      const double hv = dec_key(base[i]);
      out[i] = hv;
      cnt += (hv < sentinel);
    }
  }
  cnt = warp_sum_u(cnt);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(machined + blockIdx.y, (unsigned long long)cnt);
}

// Strip-layout decode: the keys of a surface cut into feed-direction
// sub-strips are stored strip by strip (strip k = columns [c_k, c_k+1) as a
// contiguous rows x w_k block, so each sweep job's L2 working set is one
// contiguous slab); this writes the row-major fp64 heights (surface_grid.py
// layout, leading dimension ld_out) and counts machined cells. Grid: x over
// row blocks, y = strip; 16-byte loads / stores where the width allows.
__global__ void __launch_bounds__(kThreads)
    decode_strips_kernel(const uint64_t* __restrict__ keys, double* __restrict__ out, long long rows,
                         long long ld_out, const long long* __restrict__ col0, const double* __restrict__ sent,
                         unsigned long long* __restrict__ machined) {
  const int k = blockIdx.y;
  const long long c0 = col0[k], w = col0[k + 1] - c0;
  const uint64_t* src = keys + rows * c0;
  const double sentinel = sent[0];
  unsigned cnt = 0;
  for (long long i = blockIdx.x; i < rows; i += gridDim.x) {
    const uint64_t* r = src + i * w;
    double* o = out + i * ld_out + c0;
    for (long long c = threadIdx.x; c < w; c += blockDim.x) {
      const double hv = dec_key(r[c]);
      o[c] = hv;
      cnt += hv < sentinel;
    }
  }
  cnt = warp_sum_u(cnt);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(machined, (unsigned long long)cnt);
}

// ------------------------------------------------------------ reductions
template <int NV>
struct Acc {
  double v[NV];
};

__device__ __forceinline__ double shfl_d(double v, int o) {
  return __shfl_xor_sync(0xffffffffu, v, o);
}

// fixed-order block reduction; kind[k]: 0 sum, 1 max, 2 min
template <int NV>
__device__ void block_reduce(double (&v)[NV], const int (&kind)[NV], double* sh /*[kWarps*NV]*/) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      const double w = shfl_d(v[k], o);
      v[k] = kind[k] == 0 ? v[k] + w : (kind[k] == 1 ? fmax(v[k], w) : fmin(v[k], w));
    }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < NV; ++k) sh[warp * NV + k] = v[k];
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      v[k] = lane < kWarps ? sh[lane * NV + k] : (kind[k] == 0 ? 0.0 : (kind[k] == 1 ? -INFINITY : INFINITY));
    }
#pragma unroll
    for (int o = 4; o; o >>= 1) {
#pragma unroll
      for (int k = 0; k < NV; ++k) {
        const double w = shfl_d(v[k], o);
        v[k] = kind[k] == 0 ? v[k] + w : (kind[k] == 1 ? fmax(v[k], w) : fmin(v[k], w));
      }
    }
  }
}

// double-double warp+block reduction of (hi, lo) in a fixed order: the mean
// of the areal pass is then the correctly rounded sum / n, so a constant
// region has d == 0 exactly (roughness.py:106 on NumPy gives the same)
__device__ void block_reduce_dd(double& hi, double& lo, double* sh /*[2*kWarps]*/) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const msurf_dd x = {hi, lo};
    const msurf_dd y = {shfl_d(hi, o), shfl_d(lo, o)};
    const msurf_dd r = ms_dd_add(x, y);
    hi = r.hi;
    lo = r.lo;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) {
    sh[2 * warp] = hi;
    sh[2 * warp + 1] = lo;
  }
  __syncthreads();
  if (warp == 0) {
    hi = lane < kWarps ? sh[2 * lane] : 0.0;
    lo = lane < kWarps ? sh[2 * lane + 1] : 0.0;
#pragma unroll
    for (int o = 4; o; o >>= 1) {
      const msurf_dd x = {hi, lo};
      const msurf_dd y = {shfl_d(hi, o), shfl_d(lo, o)};
      const msurf_dd r = ms_dd_add(x, y);
      hi = r.hi;
      lo = r.lo;
    }
  }
}

// pass 1 partials per block: [sum_hi, max z, min z, n, n_uncut, sum_lo]
__global__ void __launch_bounds__(kThreads)
    areal_pass1_kernel(const double* __restrict__ h, long long ld, long long sstride,
                       long long i_lo, long long j_lo, long long rows, long long cols,
                       const double* __restrict__ sent, int exclude, double* __restrict__ work) {
  __shared__ double sh[kWarps * 4];
  __shared__ double shd[kWarps * 2];
  const double* hs = h + (long long)blockIdx.y * sstride;
  const double sentinel = sent[blockIdx.y];
  double v[4] = {-INFINITY, INFINITY, 0.0, 0.0};  // max, min, n, n_uncut
  const int kind[4] = {1, 2, 0, 0};
  double shi = 0.0, slo = 0.0;
  const long long r0 = rows * blockIdx.x / gridDim.x, r1 = rows * (blockIdx.x + 1) / gridDim.x;
  for (long long r = r0; r < r1; ++r) {
    const double* row = hs + (i_lo + r) * ld + j_lo;
#pragma unroll 4
    for (long long c = threadIdx.x; c < cols; c += blockDim.x) {
      const double hv = row[c];
      const bool cut = hv < sentinel;
      if (!cut) v[3] += 1.0;
      if (cut || !exclude) {
        const double z = __dmul_rn(hv, 1000.0);  // roughness.py:105 (MM_TO_UM)
        const msurf_dd t = ms_two_sum(shi, z);
        shi = t.hi;
        slo = __dadd_rn(slo, t.lo);
        v[0] = fmax(v[0], z);
        v[1] = fmin(v[1], z);
        v[2] += 1.0;
      }
    }
  }
  {
    const msurf_dd t = ms_fast_two_sum(shi, slo);
    shi = t.hi;
    slo = t.lo;
  }
  block_reduce<4>(v, kind, sh);
  block_reduce_dd(shi, slo, shd);
  if (threadIdx.x == 0) {
    double* o = work + ((long long)blockIdx.y * gridDim.x + blockIdx.x) * 6;
    o[0] = shi; o[1] = v[0]; o[2] = v[1]; o[3] = v[2]; o[4] = v[3]; o[5] = slo;
  }
}

// one block per surface: stats1[s][6] = sum z, max z, min z, n, n_uncut, mean
// (mean = correctly rounded double-double sum / n)
__global__ void __launch_bounds__(kThreads)
    finalize_stats1_kernel(const double* __restrict__ work, int nb, double* __restrict__ out) {
  __shared__ double sh[kWarps * 4];
  __shared__ double shd[kWarps * 2];
  double v[4] = {-INFINITY, INFINITY, 0.0, 0.0};
  const int kind[4] = {1, 2, 0, 0};
  double shi = 0.0, slo = 0.0;
  const double* w = work + (long long)blockIdx.x * nb * 6;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) {
    const msurf_dd x = {shi, slo};
    const msurf_dd y = {w[b * 6 + 0], w[b * 6 + 5]};
    const msurf_dd r = ms_dd_add(x, y);
    shi = r.hi;
    slo = r.lo;
    v[0] = fmax(v[0], w[b * 6 + 1]);
    v[1] = fmin(v[1], w[b * 6 + 2]);
    v[2] += w[b * 6 + 3];
    v[3] += w[b * 6 + 4];
  }
  block_reduce<4>(v, kind, sh);
  block_reduce_dd(shi, slo, shd);
  if (threadIdx.x == 0) {
    double* o = out + (long long)blockIdx.x * 6;
    const double n = v[2];
    double mean = 0.0;
    if (n > 0.0) {
      // (shi + slo) / n rounded once: q = shi/n, remainder via FMA
      const double q = __ddiv_rn(shi, n);
      const double rem = __dadd_rn(__fma_rn(-q, n, shi), slo);
      mean = __dadd_rn(q, __ddiv_rn(rem, n));
    }
    o[0] = __dadd_rn(shi, slo); o[1] = v[0]; o[2] = v[1]; o[3] = n; o[4] = v[3]; o[5] = mean;
  }
}

__global__ void __launch_bounds__(kThreads)
    areal_pass2_kernel(const double* __restrict__ h, long long ld, long long sstride,
                       long long i_lo, long long j_lo, long long rows, long long cols,
                       const double* __restrict__ sent, int exclude,
                       const double* __restrict__ stats1, double* __restrict__ work) {
  __shared__ double sh[kWarps * 4];
  const double* hs = h + (long long)blockIdx.y * sstride;
  const double sentinel = sent[blockIdx.y];
  const double mu = stats1[blockIdx.y * 6 + 5];  // z.mean() (roughness.py:106)
  double v[4] = {0.0, 0.0, 0.0, 0.0};
  const int kind[4] = {0, 0, 0, 0};
  const long long r0 = rows * blockIdx.x / gridDim.x, r1 = rows * (blockIdx.x + 1) / gridDim.x;
  for (long long r = r0; r < r1; ++r) {
    const double* row = hs + (i_lo + r) * ld + j_lo;
#pragma unroll 4
    for (long long c = threadIdx.x; c < cols; c += blockDim.x) {
      const double hv = row[c];
      if (hv < sentinel || !exclude) {
        const double d = __dsub_rn(__dmul_rn(hv, 1000.0), mu);  // roughness.py:105-106, no FMA
        const double d2 = d * d;
        v[0] += fabs(d);
        v[1] += d2;
        v[2] += d2 * d;
        v[3] += d2 * d2;
      }
    }
  }
  block_reduce<4>(v, kind, sh);
  if (threadIdx.x == 0) {
    double* o = work + ((long long)blockIdx.y * gridDim.x + blockIdx.x) * 4;
    for (int k = 0; k < 4; ++k) o[k] = v[k];
  }
}

// one block per surface: reduce nb partials in fixed order; kinds holds 2 bits
// per value (0 sum, 1 max, 2 min)
template <int NV>
__global__ void __launch_bounds__(kThreads)
    finalize_kernel(const double* __restrict__ work, int nb, unsigned kinds, double* __restrict__ out) {
  __shared__ double sh[kWarps * NV];
  double v[NV];
  int kind[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    kind[k] = (int)((kinds >> (2 * k)) & 3u);
    v[k] = kind[k] == 0 ? 0.0 : (kind[k] == 1 ? -INFINITY : INFINITY);
  }
  const double* w = work + (long long)blockIdx.x * nb * NV;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) {
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      const double x = w[b * NV + k];
      v[k] = kind[k] == 0 ? v[k] + x : (kind[k] == 1 ? fmax(v[k], x) : fmin(v[k], x));
    }
  }
  block_reduce<NV>(v, kind, sh);
  if (threadIdx.x == 0)
    for (int k = 0; k < NV; ++k) out[(long long)blockIdx.x * NV + k] = v[k];
}

// least-squares plane leveling (roughness.py:108-113, leveling='plane'):
// pass 1 = the normal-equation sums over the used cells, with i, j the row and
// column offsets inside the ROI and z in um:
// [n, Si, Sj, Sii, Sjj, Sij, Sz, Siz, Sjz, n_uncut]
__global__ void __launch_bounds__(kThreads)
    plane_pass1_kernel(const double* __restrict__ h, long long ld, long long sstride, long long i_lo,
                       long long j_lo, long long rows, long long cols, const double* __restrict__ sent,
                       int exclude, double* __restrict__ work) {
  __shared__ double sh[kWarps * 10];
  const double* hs = h + (long long)blockIdx.y * sstride;
  const double sentinel = sent[blockIdx.y];
  double v[10] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  const int kind[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  const long long r0 = rows * blockIdx.x / gridDim.x, r1 = rows * (blockIdx.x + 1) / gridDim.x;
  for (long long r = r0; r < r1; ++r) {
    const double* row = hs + (i_lo + r) * ld + j_lo;
    const double fi = (double)r;
    for (long long c = threadIdx.x; c < cols; c += blockDim.x) {
      const double hv = row[c];
      const bool cut = hv < sentinel;
      if (!cut) v[9] += 1.0;
      if (cut || !exclude) {
        const double z = hv * 1000.0, fj = (double)c;
        v[0] += 1.0; v[1] += fi; v[2] += fj; v[3] += fi * fi; v[4] += fj * fj; v[5] += fi * fj;
        v[6] += z; v[7] += fi * z; v[8] += fj * z;
      }
    }
  }
  block_reduce<10>(v, kind, sh);
  if (threadIdx.x == 0) {
    double* o = work + ((long long)blockIdx.y * gridDim.x + blockIdx.x) * 10;
    for (int k = 0; k < 10; ++k) o[k] = v[k];
  }
}

// pass 2: d = z - ((a*i + b*j) + c) -> [S|d|, Sd^2, Sd^3, Sd^4, max d, min d]
__global__ void __launch_bounds__(kThreads)
    plane_pass2_kernel(const double* __restrict__ h, long long ld, long long sstride, long long i_lo,
                       long long j_lo, long long rows, long long cols, const double* __restrict__ sent,
                       int exclude, const double* __restrict__ coef, double* __restrict__ work) {
  __shared__ double sh[kWarps * 6];
  const double* hs = h + (long long)blockIdx.y * sstride;
  const double sentinel = sent[blockIdx.y];
  const double a = coef[blockIdx.y * 3 + 0], b = coef[blockIdx.y * 3 + 1], c0 = coef[blockIdx.y * 3 + 2];
  double v[6] = {0.0, 0.0, 0.0, 0.0, -INFINITY, INFINITY};
  const int kind[6] = {0, 0, 0, 0, 1, 2};
  const long long r0 = rows * blockIdx.x / gridDim.x, r1 = rows * (blockIdx.x + 1) / gridDim.x;
  for (long long r = r0; r < r1; ++r) {
    const double* row = hs + (i_lo + r) * ld + j_lo;
    const double ai = a * (double)r;
    for (long long c = threadIdx.x; c < cols; c += blockDim.x) {
      const double hv = row[c];
      if (hv < sentinel || !exclude) {
        const double d = hv * 1000.0 - ((ai + b * (double)c) + c0);
        const double d2 = d * d;
        v[0] += fabs(d); v[1] += d2; v[2] += d2 * d; v[3] += d2 * d2;
        v[4] = fmax(v[4], d); v[5] = fmin(v[5], d);
      }
    }
  }
  block_reduce<6>(v, kind, sh);
  if (threadIdx.x == 0) {
    double* o = work + ((long long)blockIdx.y * gridDim.x + blockIdx.x) * 6;
    for (int k = 0; k < 6; ++k) o[k] = v[k];
  }
}

// one block per (surface, profile): pass A = sum (double-double), counts,
// extrema; mean = correctly rounded sum / n (or the all-reduced first pass of
// a strip-sharded profile, stats_in); pass B = sum |z - mean|.
// out[k][8] = sum z, n_used, n_uncut, max z, min z, sum|z-mean|, mean, 0
__global__ void __launch_bounds__(kThreads)
    profiles_kernel(const double* __restrict__ h, long long sstride, const long long* __restrict__ start,
                    int n_prof, long long len, long long stride, const double* __restrict__ sent,
                    int exclude, const double* __restrict__ stats_in, double* __restrict__ out) {
  __shared__ double sh[kWarps * 4];
  __shared__ double shd[kWarps * 2];
  __shared__ double s_mean;
  const int prof = blockIdx.x;
  const int surf = blockIdx.y;
  const double* base = h + (long long)surf * sstride + start[prof];
  const double sentinel = sent[surf];
  double v[4] = {0.0, 0.0, -INFINITY, INFINITY};  // n_cut, n_uncut, max, min
  const int kind[4] = {0, 0, 1, 2};
  double shi = 0.0, slo = 0.0;
  for (long long k = threadIdx.x; k < len; k += blockDim.x) {
    const double hv = base[k * stride];
    const bool cut = hv < sentinel;
    if (!cut) v[1] += 1.0;
    if (cut || !exclude) {
      const double z = __dmul_rn(hv, 1000.0);
      const msurf_dd t = ms_two_sum(shi, z);
      shi = t.hi;
      slo = __dadd_rn(slo, t.lo);
      v[0] += 1.0;
      v[2] = fmax(v[2], z);
      v[3] = fmin(v[3], z);
    }
  }
  {
    const msurf_dd t = ms_fast_two_sum(shi, slo);
    shi = t.hi;
    slo = t.lo;
  }
  block_reduce<4>(v, kind, sh);
  block_reduce_dd(shi, slo, shd);
  if (threadIdx.x == 0) {
    const long long k = (long long)surf * n_prof + prof;
    double mean = 0.0;
    if (stats_in) {
      mean = stats_in[k * 8 + 0] / stats_in[k * 8 + 1];
    } else if (v[0] > 0.0) {
      const double q = __ddiv_rn(shi, v[0]);
      mean = __dadd_rn(q, __ddiv_rn(__dadd_rn(__fma_rn(-q, v[0], shi), slo), v[0]));
    }
    s_mean = mean;
  }
  __syncthreads();
  const double mu = s_mean;
  double a[1] = {0.0};
  const int ka[1] = {0};
  for (long long k = threadIdx.x; k < len; k += blockDim.x) {
    const double hv = base[k * stride];
    if (hv < sentinel || !exclude) a[0] += fabs(__dsub_rn(__dmul_rn(hv, 1000.0), mu));
  }
  __syncthreads();
  block_reduce<1>(a, ka, sh);
  if (threadIdx.x == 0) {
    double* o = out + ((long long)surf * n_prof + prof) * 8;
    o[0] = __dadd_rn(shi, slo); o[1] = v[0]; o[2] = v[1]; o[3] = v[2]; o[4] = v[3]; o[5] = a[0];
    o[6] = mu; o[7] = 0.0;
  }
}

// ------------------------------------------------------------ microbench
__global__ void mb_dp_kernel(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x * 1e-9, x1 = x0 + 1.0, x2 = x0 + 2.0, x3 = x0 + 3.0;
  double x4 = x0 + 4.0, x5 = x0 + 5.0, x6 = x0 + 6.0, x7 = x0 + 7.0;
  for (int i = 0; i < iters; ++i) {
    x0 = __dadd_rn(__dmul_rn(x0, a), b); x1 = __dadd_rn(__dmul_rn(x1, a), b);
    x2 = __dadd_rn(__dmul_rn(x2, a), b); x3 = __dadd_rn(__dmul_rn(x3, a), b);
    x4 = __dadd_rn(__dmul_rn(x4, a), b); x5 = __dadd_rn(__dmul_rn(x5, a), b);
    x6 = __dadd_rn(__dmul_rn(x6, a), b); x7 = __dadd_rn(__dmul_rn(x7, a), b);
  }
  const double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (s == 12345.678) out[0] = s;
}

__global__ void mb_fma_kernel(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x * 1e-9, x1 = x0 + 1.0, x2 = x0 + 2.0, x3 = x0 + 3.0;
  double x4 = x0 + 4.0, x5 = x0 + 5.0, x6 = x0 + 6.0, x7 = x0 + 7.0;
  for (int i = 0; i < iters; ++i) {
    x0 = __fma_rn(x0, a, b); x1 = __fma_rn(x1, a, b); x2 = __fma_rn(x2, a, b);
    x3 = __fma_rn(x3, a, b); x4 = __fma_rn(x4, a, b); x5 = __fma_rn(x5, a, b);
    x6 = __fma_rn(x6, a, b); x7 = __fma_rn(x7, a, b);
  }
  const double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (s == 12345.678) out[0] = s;
}

// ------------------------------------------------------------ graymap export
// surface_io.py:100-131 (write_graymap): range pass over the machined cells of
// the ROI in mm -> partials [max, min, n_machined] per block
__global__ void __launch_bounds__(kThreads)
    graymap_range_kernel(const double* __restrict__ h, long long ld, long long i_lo, long long j_lo,
                         long long rows, long long cols, const double* __restrict__ sent,
                         double* __restrict__ work) {
  __shared__ double sh[kWarps * 3];
  const double sentinel = sent[0];
  double v[3] = {-INFINITY, INFINITY, 0.0};
  const int kind[3] = {1, 2, 0};
  const long long r0 = rows * blockIdx.x / gridDim.x, r1 = rows * (blockIdx.x + 1) / gridDim.x;
  for (long long r = r0; r < r1; ++r) {
    const double* row = h + (i_lo + r) * ld + j_lo;
    for (long long c = threadIdx.x; c < cols; c += blockDim.x) {
      const double hv = row[c];
      if (hv < sentinel) {
        v[0] = fmax(v[0], hv);
        v[1] = fmin(v[1], hv);
        v[2] += 1.0;
      }
    }
  }
  block_reduce<3>(v, kind, sh);
  if (threadIdx.x == 0) {
    double* o = work + (long long)blockIdx.x * 3;
    o[0] = v[0]; o[1] = v[1]; o[2] = v[2];
  }
}

// pixels: machined -> rint((z - z_lo) * (65535 / (z_hi - z_lo))) (mid-gray when
// z_hi == z_lo), uncut -> 0; image row = y node j, column = x node i, 16-bit
// big-endian. 32x32 node tiles transposed through shared memory so both the
// fp64 reads (along j) and the u16 writes (along i) are coalesced.
__global__ void __launch_bounds__(256)
    graymap_pixels_kernel(const double* __restrict__ h, long long ld, long long i_lo, long long j_lo,
                          long long rows, long long cols, const double* __restrict__ sent,
                          const double* __restrict__ range3, unsigned short* __restrict__ pix) {
  __shared__ unsigned short tile[32][33];
  const double sentinel = sent[0];
  const double z_hi = range3[0], z_lo = range3[1];
  const bool flat = !(z_hi > z_lo);
  const double scale = flat ? 0.0 : __ddiv_rn(65535.0, __dsub_rn(z_hi, z_lo));
  const long long ti = (long long)blockIdx.y * 32, tj = (long long)blockIdx.x * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  for (int a = ty; a < 32; a += 8) {  // a = i offset in tile, tx = j offset
    const long long i = ti + a, j = tj + tx;
    unsigned short p = 0;
    if (i < rows && j < cols) {
      const double hv = h[(i_lo + i) * ld + j_lo + j];
      if (hv < sentinel) p = flat ? (unsigned short)32768 : (unsigned short)rint(__dmul_rn(__dsub_rn(hv, z_lo), scale));
    }
    tile[a][tx] = p;
  }
  __syncthreads();
  for (int b = ty; b < 32; b += 8) {  // b = j offset (image row), tx = i offset (column)
    const long long j = tj + b, i = ti + tx;
    if (i < rows && j < cols) {
      const unsigned short p = tile[tx][b];
      pix[j * rows + i] = (unsigned short)((p >> 8) | (p << 8));
    }
  }
}

// RED.MIN.64 peak with the sweep's access shape: each warp instruction covers
// 32 lanes on consecutive keys (one 256-byte run) at a random warp-uniform
// base inside an L2-resident table
__global__ void mb_atomic_run_kernel(unsigned long long* buf, long long mask, int iters) {
  unsigned long long x = (blockIdx.x * 1315423911ull) ^ ((threadIdx.x >> 5) * 2654435761ull) ^ 0x9e3779b97f4a7c15ull;
  const int lane = threadIdx.x & 31;
  for (int i = 0; i < iters; ++i) {
    x ^= x << 13; x ^= x >> 7; x ^= x << 17;
    red_min_u64(buf + (((x & mask) & ~31ull) + lane), x >> 1);
  }
}

// RED.MIN.64 rate by shape: every warp instruction touches L distinct random
// 128-byte lines of an L2-resident table, lane l on line l % L, key (l / L)
// within it (L = 1: lanes 0-15 only, one key each); warp instructions/s.
// Lanes of one line share a 32-bit LCG stream (one IMAD per RED), so the
// loop issues ~6 instructions per RED and the L2 atomic units, not the
// issue slots, set the rate.
__global__ void mb_atomic_lines_kernel(unsigned long long* buf, unsigned mask_lines, int L, int iters) {
  const int lane = threadIdx.x & 31;
  const int grp = lane % L, pos = lane / L;
  const bool on = pos < 16;
  const unsigned wid = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  unsigned x = (wid * 2654435761u) ^ ((unsigned)(grp + 1) * 0x9e3779b9u);
  unsigned long long* p = buf + pos;
#pragma unroll 4
  for (int i = 0; i < iters; ++i) {
    x = x * 1664525u + 1013904223u;
    if (on) red_min_u64(p + ((unsigned long long)((x >> 7) & mask_lines) << 4), (unsigned long long)(x | 1u));
  }
}

__global__ void mb_atomic_kernel(unsigned long long* buf, long long mask, int iters) {
  unsigned long long x = (blockIdx.x * 1315423911ull) ^ (threadIdx.x * 2654435761ull) ^ 0x9e3779b97f4a7c15ull;
  for (int i = 0; i < iters; ++i) {
    x ^= x << 13; x ^= x >> 7; x ^= x << 17;
    atomicMin(buf + (x & mask), x >> 1);
  }
}

// distinct 128-byte lines per traced RED record -> hist[0..32] (one warp
// per record, grid-stride)
__global__ void __launch_bounds__(256)
    red_lines_kernel(const unsigned* __restrict__ trace, long long n_rec, unsigned long long* hist,
                     unsigned long long* hist_sectors) {
  __shared__ unsigned long long h[33], hs[33];
  for (int i = threadIdx.x; i < 33; i += blockDim.x) h[i] = hs[i] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long r = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5; r < n_rec; r += nw) {
    const unsigned off = __ldcs(trace + r * 32 + lane);
    const bool on = off != ~0u;
    const unsigned act = __ballot_sync(0xffffffffu, on);
    const unsigned same = __match_any_sync(0xffffffffu, on ? (off >> 4) : 0xffffffffu);
    // a lane opens a line if no lower active lane holds the same line
    const bool first = on && ((same & act & ((1u << lane) - 1u)) == 0u);
    const int lines = __popc(__ballot_sync(0xffffffffu, first));
    // the same for the 32-byte sectors (four keys each)
    const unsigned same_s = __match_any_sync(0xffffffffu, on ? (off >> 2) : 0xffffffffu);
    const bool first_s = on && ((same_s & act & ((1u << lane) - 1u)) == 0u);
    const int sectors = __popc(__ballot_sync(0xffffffffu, first_s));
    if (lane == 0) {
      if (hist) atomicAdd(&h[lines], 1ull);
      if (hist_sectors) atomicAdd(&hs[sectors], 1ull);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 33; i += blockDim.x) {
    if (hist && h[i]) atomicAdd(hist + i, h[i]);
    if (hist_sectors && hs[i]) atomicAdd(hist_sectors + i, hs[i]);
  }
}

// the node rows one (pass, tooth) launch can have deposited into: x = fma(c, x_t,
// s y_t) + pass x0 + vibration with |fma(c, x_t, s y_t)| <= max|x_t| + max|y_t|
// over the tooth's tool-frame box, located to the nearest node (+-2 nodes of
// slack cover every rounding). x0 == nullptr: every row.
struct ZBand {
  const double* x0;   // the launch's pass x0 (device)
  const double* box;  // its tooth's box (xl, xh, yl, yh, zl, zh) (device)
  double pad;         // |vibration amplitude|
  double x_min, inv_h;
};

// msurf_zcap_refresh: one CTA per 32x32-node tile of a slab, max key ->
// height - stock rounded up to float (an upper bound for the cull). With a
// band, tiles outside it keep their cap: nothing there changed since it was
// computed, and heights only decrease, so it is still an upper bound.
__global__ void __launch_bounds__(256)
    zcap_kernel(const uint64_t* __restrict__ keys, long long ld, long long rows, long long cols,
                const double* __restrict__ stock, float* __restrict__ zcap, int* stop_reset, ZBand band) {
  if (stop_reset && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) *stop_reset = 0;
  __shared__ unsigned long long wmax[8];
  const long long i0 = (long long)blockIdx.y * kCapTile, j = (long long)blockIdx.x * kCapTile + (threadIdx.x & (kCapTile - 1));
  if (band.x0) {  // CTA-uniform
    const double* b = band.box;
    const double r = fmax(fabs(b[0]), fabs(b[1])) + fmax(fabs(b[2]), fabs(b[3])) + band.pad;
    const double x0 = *band.x0;
    const double lo = (x0 - r - band.x_min) * band.inv_h - 2.0, hi = (x0 + r - band.x_min) * band.inv_h + 2.0;
    if ((double)(i0 + kCapTile - 1) < lo || (double)i0 > hi) return;
  }
  unsigned long long m = 0ull;
  if (j < cols)
    for (long long i = i0 + (threadIdx.x >> kCapShift); i < i0 + kCapTile && i < rows; i += 256 / kCapTile) {
      const unsigned long long k = keys[i * ld + j];
      m = k > m ? k : m;
    }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const unsigned long long v = __shfl_xor_sync(0xffffffffu, m, o);
    m = v > m ? v : m;
  }
  if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < 8; ++w) m = wmax[w] > m ? wmax[w] : m;
    m = wmax[0] > m ? wmax[0] : m;
    const float v = m ? __double2float_ru(__dsub_ru(dec_key(m), stock[0])) : -INFINITY;
    zcap[(long long)blockIdx.y * gridDim.x + blockIdx.x] = v;
  }
}

// smem of one sweep CTA: transforms + masks by thread + masks by slot + the
// tile mask of the tile pre-cull
inline size_t sweep_smem(int tile, int mask_words) {
  return (size_t)tile * 8 * sizeof(double) + (size_t)(2 * tile + 1) * mask_words * sizeof(uint64_t);
}

template <int MODE, int DIAG, bool ONE, int TILE, int NTHR, bool STAGE = false>
cudaError_t launch_shape(int64_t n_tiles, cudaStream_t st, const msurf_job* jobs, int n_jobs, const int64_t* prefix,
                         int mask_words, const msurf_job& job, unsigned long long* list, unsigned* count) {
  auto kern = sweep_kernel<MODE, DIAG, ONE, TILE, NTHR, STAGE>;
  const size_t smem = sweep_smem(TILE, mask_words);
  cudaError_t e = cudaSuccess;
  if (smem > 48 * 1024) e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if constexpr (ONE) {
    kern<<<(unsigned)n_tiles, NTHR, smem, st>>>(nullptr, 1, nullptr, mask_words, job, nullptr, nullptr);
  } else {
    // pre-cull the tiles into the list, then persistent CTAs (a few waves of
    // the resident limit) walk it
    e = cudaMemsetAsync(count, 0, 2 * sizeof(unsigned), st);  // list length, work cursor
    if (e != cudaSuccess) return e;
    tile_list_kernel<MODE, TILE><<<(unsigned)((n_tiles + 255) / 256), 256, 0, st>>>(jobs, n_jobs, prefix, n_tiles,
                                                                                  list, count);
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NTHR, smem);
    const int64_t grid = std::min<int64_t>(n_tiles, (int64_t)sms * std::max(per_sm, 1));
    kern<<<(unsigned)grid, NTHR, smem, st>>>(jobs, n_jobs, prefix, mask_words, job, list, count);
  }
  return cudaSuccess;
}

// tiles of one job for a tile size: passes * teeth * ceil(window / tile)
inline int64_t job_tiles(const msurf_job& j, int tile) {
  return (int64_t)j.passes * (j.tooth_n ? j.tooth_n : j.teeth) * ((j.step_hi - j.step_lo + tile - 1) / tile);
}

template <int MODE, int DIAG>
cudaError_t launch_sweep(int64_t n_tiles, cudaStream_t st, const msurf_job* jobs, int n_jobs,
                         const int64_t* prefix, int mask_words, const msurf_job* one, unsigned long long* list,
                         unsigned* count, bool wide) {
  if (one) {
    if constexpr (MODE == MSURF_MODE_EXT_TILT) {
      if (wide)  // eight warps over 64 steps: heavy tiles finish sooner (short surface-cap launches)
        return launch_shape<MODE, DIAG, true, kTiltTile, kCapThreads>(job_tiles(*one, kTiltTile), st, nullptr, 1,
                                                                     nullptr, mask_words, *one, nullptr, nullptr);
      return launch_shape<MODE, DIAG, true, kTiltTile, kTiltThreads>(job_tiles(*one, kTiltTile), st, nullptr, 1,
                                                                    nullptr, mask_words, *one, nullptr, nullptr);
    } else
      return launch_shape<MODE, DIAG, true, kWideTile, kWideThreads>(job_tiles(*one, kWideTile), st, nullptr, 1,
                                                                    nullptr, mask_words, *one, nullptr, nullptr);
  }
  msurf_job dummy;
  memset(&dummy, 0, sizeof(dummy));
  return launch_shape<MODE, DIAG, false, kBatchTile, kBatchThreads>(n_tiles, st, jobs, n_jobs, prefix, mask_words,
                                                                    dummy, list, count);
}

// small results -> host-mapped page-locked memory (stores over PCIe, no copy engine)
__global__ void readback_kernel(const unsigned long long* __restrict__ src, volatile unsigned long long* dst,
                                long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    dst[i] = src[i];
  __threadfence_system();
}

}  // namespace

// ================================================================ C ABI
extern "C" {

void* msurf_host_alloc(int64_t bytes) {
  void* p = nullptr;
  if (bytes <= 0) return nullptr;
  if (cudaHostAlloc(&p, (size_t)bytes, cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess) {
    cudaGetLastError();
    set_err("msurf_host_alloc: cudaHostAlloc failed");
    return nullptr;
  }
  return p;
}

int msurf_host_free(void* p) {
  if (p && cudaFreeHost(p) != cudaSuccess) return set_err("msurf_host_free: cudaFreeHost failed");
  return 0;
}

int msurf_readback(const void* src, void* host_dst, int64_t bytes, void* stream) {
  if (bytes < 0 || (bytes % 8) || (bytes > 0 && (!src || !host_dst)))
    return set_err("msurf_readback: bad arguments");
  if (bytes == 0) return 0;
  void* dptr = nullptr;
  if (cudaHostGetDevicePointer(&dptr, host_dst, 0) != cudaSuccess) {
    cudaGetLastError();
    return set_err("msurf_readback: destination is not mapped page-locked memory");
  }
  const long long n = bytes / 8;
  const int blocks = (int)std::min<long long>((n + kThreads - 1) / kThreads, 148);
  readback_kernel<<<blocks, kThreads, 0, (cudaStream_t)stream>>>(
      static_cast<const unsigned long long*>(src), static_cast<unsigned long long*>(dptr), n);
  return check_launch("readback_kernel");
}

int msurf_readback_sync(const void* src, void* host_dst, int64_t bytes, void* stream) {
  if (msurf_readback(src, host_dst, bytes, stream)) return 1;
  const cudaError_t e = cudaStreamSynchronize((cudaStream_t)stream);
  if (e != cudaSuccess) return set_err(std::string("msurf_readback_sync: ") + cudaGetErrorString(e));
  return 0;
}

int msurf_copy2d_d2h(void* host_dst, int64_t dst_pitch, const void* src, int64_t src_pitch,
                     int64_t width_bytes, int64_t rows, void* stream) {
  if (!host_dst || !src || rows < 0 || width_bytes < 0 || dst_pitch < width_bytes || src_pitch < width_bytes)
    return set_err("msurf_copy2d_d2h: bad arguments");
  if (rows == 0 || width_bytes == 0) return 0;
  const cudaError_t e = cudaMemcpy2DAsync(host_dst, (size_t)dst_pitch, src, (size_t)src_pitch, (size_t)width_bytes,
                                          (size_t)rows, cudaMemcpyDeviceToHost, (cudaStream_t)stream);
  if (e != cudaSuccess) return set_err(std::string("msurf_copy2d_d2h: ") + cudaGetErrorString(e));
  return 0;
}

int msurf_abi_version(void) { return MSURF_ABI_VERSION; }
int msurf_zcap_tile(void) { return kCapTile; }
const char* msurf_last_error(void) { return g_err.c_str(); }
int msurf_sizeof_job(void) { return (int)sizeof(msurf_job); }
int msurf_tile_steps(void) { return kBatchTile; }

int msurf_fill_keys(uint64_t* keys, int64_t count, int32_t n_surf, const double* value,
                    void* stream) {
  if (count < 0 || n_surf < 1 || (count > 0 && (!keys || !value)))
    return set_err("msurf_fill_keys: bad arguments");
  if (count == 0) return 0;
  long long blocks = (count / 2 + kThreads - 1) / kThreads;
  const long long cap = n_surf > 1 ? 64 : 148 * 16;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  fill_kernel<<<dim3((unsigned)blocks, (unsigned)n_surf), kThreads, 0, (cudaStream_t)stream>>>(
      keys, count, value);
  return check_launch("fill_kernel");
}

static int sweep_impl(const msurf_job* jobs, int32_t n_jobs, const int64_t* tile_prefix, int64_t n_tiles,
                      int32_t mode, int32_t max_points, void* stream, const msurf_job* one, void* scratch) {
  if (!one && n_tiles == 0) return 0;
  if (n_tiles > 0x7fffffffLL) return set_err("msurf_sweep: too many tiles");
  if (one && (job_tiles(*one, 64) == 0)) return 0;
  if (one && job_tiles(*one, 64) > 0x7fffffffLL) return set_err("msurf_sweep_job: too many tiles");
  const int nchunk = (max_points + 31) / 32;
  const int mask_words = (nchunk + 63) / 64;
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = cudaSuccess;
  const bool diag = (mode & MSURF_SWEEP_DIAG) != 0;
  const bool trace = (mode & MSURF_SWEEP_TRACE) != 0;
  const bool wide = (mode & MSURF_SWEEP_WIDE) != 0;
  // scratch: [0, 8) tile count and work cursor, then the tile list (8 bytes per tile)
  unsigned* count = static_cast<unsigned*>(scratch);
  unsigned long long* list = scratch ? static_cast<unsigned long long*>(scratch) + 1 : nullptr;
#define MSURF_LAUNCH(M)                                                                                   \
  e = trace ? launch_sweep<M, 2>(n_tiles, st, jobs, n_jobs, tile_prefix, mask_words, one, list, count, wide)   \
      : diag  ? launch_sweep<M, 1>(n_tiles, st, jobs, n_jobs, tile_prefix, mask_words, one, list, count, wide)   \
              : launch_sweep<M, 0>(n_tiles, st, jobs, n_jobs, tile_prefix, mask_words, one, list, count, wide)
  switch (mode & ~(MSURF_SWEEP_DIAG | MSURF_SWEEP_TRACE | MSURF_SWEEP_WIDE)) {
    case MSURF_MODE_REF: MSURF_LAUNCH(MSURF_MODE_REF); break;
    case MSURF_MODE_EXT: MSURF_LAUNCH(MSURF_MODE_EXT); break;
    case MSURF_MODE_EXT_TILT: MSURF_LAUNCH(MSURF_MODE_EXT_TILT); break;
    default:
      return set_err("msurf_sweep: unknown mode");
  }
#undef MSURF_LAUNCH
  if (e != cudaSuccess) return set_err(std::string("msurf_sweep: launch setup: ") + cudaGetErrorString(e));
  return check_launch("sweep_kernel");
}

int msurf_sweep(const msurf_job* jobs, int32_t n_jobs, const int64_t* tile_prefix,
                int64_t n_tiles, int32_t mode, int32_t max_points, void* scratch, void* stream) {
  if (n_jobs < 1 || !jobs || !tile_prefix || n_tiles < 0 || max_points < 1 || (n_tiles > 0 && !scratch))
    return set_err("msurf_sweep: bad arguments");
  return sweep_impl(jobs, n_jobs, tile_prefix, n_tiles, mode, max_points, stream, nullptr, scratch);
}

int msurf_sweep_job(const msurf_job* job, int32_t mode, int32_t max_points, void* stream) {
  if (!job || max_points < 1) return set_err("msurf_sweep_job: bad arguments");
  return sweep_impl(nullptr, 1, nullptr, 0, mode, max_points, stream, job, nullptr);
}

int msurf_trace_arm(uint32_t* trace, int64_t cap_records, unsigned long long* counters, const uint64_t* base) {
  if ((cap_records > 0 && !trace) || cap_records < 0 || !counters || !base)
    return set_err("msurf_trace_arm: bad arguments");
  unsigned long long cap = (unsigned long long)cap_records;
  cudaError_t e = cudaMemcpyToSymbol(g_trace, &trace, sizeof(trace));
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(g_trace_cap, &cap, sizeof(cap));
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(g_trace_ctr, &counters, sizeof(counters));
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(g_trace_base, &base, sizeof(base));
  if (e != cudaSuccess) return set_err(std::string("msurf_trace_arm: ") + cudaGetErrorString(e));
  return 0;
}

int msurf_red_lines(const uint32_t* trace, int64_t n_records, unsigned long long* hist, void* stream) {
  if (n_records < 0 || !hist || (n_records > 0 && !trace)) return set_err("msurf_red_lines: bad arguments");
  if (n_records == 0) return 0;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  red_lines_kernel<<<(unsigned)sms * 8, 256, 0, (cudaStream_t)stream>>>(trace, n_records, hist, nullptr);
  return check_launch("red_lines_kernel");
}

int msurf_red_sectors(const uint32_t* trace, int64_t n_records, unsigned long long* hist_lines,
                      unsigned long long* hist_sectors, void* stream) {
  if (n_records < 0 || !hist_lines || !hist_sectors || (n_records > 0 && !trace))
    return set_err("msurf_red_sectors: bad arguments");
  if (n_records == 0) return 0;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  red_lines_kernel<<<(unsigned)sms * 8, 256, 0, (cudaStream_t)stream>>>(trace, n_records, hist_lines, hist_sectors);
  return check_launch("red_lines_kernel");
}

static int zcap_refresh(const uint64_t* keys, int64_t ld, int64_t rows, int64_t cols, const double* stock,
                        float* zcap, int32_t* stop_reset, void* stream, const ZBand& band) {
  if (!keys || !stock || !zcap || rows < 1 || cols < 1 || ld < cols) return set_err("msurf_zcap_refresh: bad arguments");
  const long long ti = (rows + kCapTile - 1) / kCapTile, tj = (cols + kCapTile - 1) / kCapTile;
  if (ti > 65535 || tj > 0x7fffffffLL) return set_err("msurf_zcap_refresh: slab too large");
  zcap_kernel<<<dim3((unsigned)tj, (unsigned)ti), 256, 0, (cudaStream_t)stream>>>(keys, ld, rows, cols, stock, zcap,
                                                                                 stop_reset, band);
  return check_launch("zcap_kernel");
}

int msurf_zcap_refresh(const uint64_t* keys, int64_t ld, int64_t rows, int64_t cols, const double* stock,
                       float* zcap, int32_t* stop_reset, void* stream) {
  return zcap_refresh(keys, ld, rows, cols, stock, zcap, stop_reset, stream, ZBand{});
}

// the refresh after (pass, tooth) launch `sub` of a capped job: only the node
// rows that launch can have reached (MSURF_ZCAP_BAND=0: the whole slab)
static int zcap_refresh_after(const msurf_job& sub, const double* stock, void* stream) {
  static const bool on = [] {
    const char* e = getenv("MSURF_ZCAP_BAND");
    return !(e && e[0] == '0');
  }();
  ZBand band{};
  if (on && sub.spacing > 0.0) {
    band.x0 = sub.pass_x0;
    band.box = sub.tooth_box + 6 * sub.tooth_lo;
    band.pad = fabs(sub.vib_amp);
    band.x_min = sub.x_min;
    band.inv_h = 1.0 / sub.spacing;
  }
  return zcap_refresh(sub.keys, sub.ld, sub.m + 1, sub.j_hi - sub.j_lo + 1, stock, const_cast<float*>(sub.zcap),
                      nullptr, stream, band);
}

// one staged (pass, tooth) launch of a capped tilt job: the staging header
// cleared, phase 1 of every tile (rows, masks, live units out), then the
// persistent phase-2 kernel over the units (production variant only)
static int staged_launch(const msurf_job& sub, int32_t max_points, cudaStream_t st) {
  const int nchunk = (max_points + 31) / 32;
  const int mask_words = (nchunk + 63) / 64;
  cudaError_t e = cudaMemsetAsync(sub.stage, 0, 16, st);
  if (e != cudaSuccess) return set_err(std::string("staged_launch: ") + cudaGetErrorString(e));
  // phase 1 with two warps over the 64 steps (one round per CTA instead of two)
  e = launch_shape<MSURF_MODE_EXT_TILT, 0, true, kTiltTile, kStageThreads, true>(job_tiles(sub, kTiltTile), st, nullptr,
                                                                                 1, nullptr, mask_words, sub, nullptr,
                                                                                 nullptr);
  if (e != cudaSuccess) return set_err(std::string("staged_launch: phase 1: ") + cudaGetErrorString(e));
  if (check_launch("sweep_kernel (staged)")) return 1;
  // short launch (the same threshold as engine.ZCAP_LONG_LAUNCH): the
  // register-rich variant (see sweep_units_kernel)
  const bool short_launch = (double)(sub.step_hi - sub.step_lo) * (double)sub.points < kShortLaunch;
  // resident one-warp CTAs of each units-kernel variant, queried once per device
  static int slots[64][2] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return set_err("staged_launch: device index");
  if (!slots[dev][short_launch]) {
    int sms = 148, per_sm = 1;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (short_launch)
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sweep_units_kernel<0, 16>, 32, 0);
    else
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sweep_units_kernel<0, 32>, 32, 0);
    slots[dev][short_launch] = sms * std::max(per_sm, 1);
  }
  const long long units_max = job_tiles(sub, kTiltTile) * nchunk;
  const long long grid = std::min<long long>(units_max, (long long)slots[dev][short_launch]);
  if (grid > 0) {
    if (short_launch)
      sweep_units_kernel<0, 16><<<(unsigned)grid, 32, 0, st>>>(sub, mask_words);
    else
      sweep_units_kernel<0, 32><<<(unsigned)grid, 32, 0, st>>>(sub, mask_words);
  }
  return check_launch("sweep_units_kernel");
}

// staging bytes one capped (pass, tooth) launch of `job` needs
static long long stage_bytes(const msurf_job& job, int32_t max_points) {
  const int nchunk = (max_points + 31) / 32;
  const int mask_words = (nchunk + 63) / 64;
  const long long tiles = (job.step_hi - job.step_lo + 63) / 64;
  return kStageHeader + tiles * stage_rec_bytes(mask_words) + tiles * nchunk * 8;
}

int msurf_stage_bytes(const msurf_job* job, int32_t max_points, int64_t* bytes) {
  if (!job || !bytes || max_points < 1) return set_err("msurf_stage_bytes: bad arguments");
  *bytes = stage_bytes(*job, max_points);
  return 0;
}

int msurf_sweep_job_capped(const msurf_job* job, int32_t mode, int32_t max_points, const double* stock,
                           void* stream) {
  if (!job || !job->zcap || !stock || max_points < 1) return set_err("msurf_sweep_job_capped: bad arguments");
  const long long rows = job->m + 1, cols = job->j_hi - job->j_lo + 1;
  float* zcap = const_cast<float*>(job->zcap);
  const int teeth = job->tooth_n ? job->tooth_n : job->teeth;
  const int n = job->passes * teeth;
  // caps of the freshly filled slab, then (pass, tooth) by (pass, tooth) with
  // the caps refreshed after every launch but the last
  if (msurf_zcap_refresh(job->keys, job->ld, rows, cols, stock, zcap, nullptr, stream)) return 1;
  for (int i = 0; i < n; ++i) {
    msurf_job sub = *job;
    sub.passes = 1;
    sub.pass_x0 = job->pass_x0 + i / teeth;
    sub.tooth_lo = job->tooth_lo + i % teeth;
    sub.tooth_n = 1;
    if (job_tiles(sub, 64) == 0) continue;
    if (sweep_impl(nullptr, 1, nullptr, 0, mode, max_points, stream, &sub, nullptr)) return 1;
    if (i + 1 < n && zcap_refresh_after(sub, stock, stream)) return 1;
  }
  return 0;
}

// library-owned non-blocking streams (no implicit synchronisation with any
// other stream, the legacy one included), per device and thread
// stream k belongs to job slot k / 4 and carries that slot's priority (slot 0
// highest): side-by-side jobs then finish in slot order, so the caller can
// decode and copy out one job's slab while the later ones still sweep
cudaStream_t lib_stream(int k) {
  constexpr int kMax = 48;  // 8 job slots x 4 in-flight launches, then anchors
  static thread_local cudaStream_t pool[64][kMax] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64 || k < 0 || k >= kMax) return nullptr;
  if (!pool[dev][k]) {
    int least = 0, greatest = 0;
    cudaDeviceGetStreamPriorityRange(&least, &greatest);
    const int prio = std::min(least, greatest + k / 4);
    if (cudaStreamCreateWithPriority(&pool[dev][k], cudaStreamNonBlocking, prio) != cudaSuccess) return nullptr;
  }
  return pool[dev][k];
}

void* msurf_anchor_stream(int32_t k) {
  if (k < 0 || k >= 16) return nullptr;
  return lib_stream(32 + k);
}

int msurf_stream_wait(void* waiter, void* signaler) {
  cudaEvent_t ev = nullptr;
  if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) return set_err("msurf_stream_wait: event");
  cudaError_t e = cudaEventRecord(ev, (cudaStream_t)signaler);
  if (e == cudaSuccess) e = cudaStreamWaitEvent((cudaStream_t)waiter, ev, 0);
  cudaEventDestroy(ev);
  if (e != cudaSuccess) return set_err(std::string("msurf_stream_wait: ") + cudaGetErrorString(e));
  return 0;
}

int msurf_sweep_jobs_capped(const msurf_job* jobs, int32_t n_jobs, int32_t mode, int32_t max_points,
                            const int64_t* stocks, int32_t depth, void* stage, int64_t stage_each, int32_t slot0,
                            void* stream) {
  if (!jobs || n_jobs < 1 || !stocks || max_points < 1 || depth < 1 || depth > 4 || slot0 < 0 ||
      slot0 + n_jobs > 8)
    return set_err("msurf_sweep_jobs_capped: bad arguments");
  // fork: job k's (pass, tooth) launches round-robin over `depth` library
  // streams of its own (launch i waits for launch i - depth and the cap refresh
  // after it; neighbours overlap, reading caps at most depth - 1 launches
  // stale, which only weakens the cull); jobs write disjoint slabs. Every
  // stream is joined back into `stream` (graph-capturable fork/join).
  // job j (slot slot0 + j) uses streams 4 (slot0 + j) + [0, depth)
  auto sid = [&](int j, int d) { return 4 * (slot0 + j) + d; };
  cudaStream_t st = (cudaStream_t)stream;
  cudaEvent_t fork = nullptr;
  if (cudaEventCreateWithFlags(&fork, cudaEventDisableTiming) != cudaSuccess) return set_err("events");
  cudaEventRecord(fork, st);
  int rc = 0;
  for (int j = 0; j < n_jobs && rc == 0; ++j)
    for (int d = 0; d < depth; ++d) {
      cudaStream_t q = lib_stream(sid(j, d));
      if (!q) {
        rc = set_err("msurf_sweep_jobs_capped: stream");
        break;
      }
      cudaStreamWaitEvent(q, fork, 0);
    }
  for (int j = 0; j < n_jobs && rc == 0; ++j) {
    const msurf_job* job = jobs + j;
    const double* stock = reinterpret_cast<const double*>(stocks[j]);
    if (!job->zcap || !stock) {
      rc = set_err("msurf_sweep_jobs_capped: job without caps");
      break;
    }
    const long long rows = job->m + 1, cols = job->j_hi - job->j_lo + 1;
    float* zcap = const_cast<float*>(job->zcap);
    const int teeth = job->tooth_n ? job->tooth_n : job->teeth;
    const int n = job->passes * teeth;
    cudaStream_t q0 = lib_stream(sid(j, 0));
    // caps of the freshly filled slab first, seen by every stream of the job
    rc = msurf_zcap_refresh(job->keys, job->ld, rows, cols, stock, zcap, nullptr, q0);
    cudaEvent_t ready = nullptr;
    if (rc == 0 && cudaEventCreateWithFlags(&ready, cudaEventDisableTiming) == cudaSuccess) {
      cudaEventRecord(ready, q0);
      for (int d = 1; d < depth; ++d) cudaStreamWaitEvent(lib_stream(sid(j, d)), ready, 0);
      cudaEventDestroy(ready);
    }
    for (int i = 0; i < n && rc == 0; ++i) {
      cudaStream_t q = lib_stream(sid(j, i % depth));
      msurf_job sub = *job;
      sub.passes = 1;
      sub.pass_x0 = job->pass_x0 + i / teeth;
      sub.tooth_lo = job->tooth_lo + i % teeth;
      sub.tooth_n = 1;
      if (job_tiles(sub, 64) == 0) continue;
      // staged two-kernel form for the production variant when staging is given
      const bool staged = stage && (mode & ~MSURF_MODE_MASK) == 0 && (mode & MSURF_MODE_MASK) == MSURF_MODE_EXT_TILT;
      if (staged) {
        sub.stage = static_cast<unsigned char*>(stage) + (long long)(j * depth + i % depth) * stage_each;
        rc = stage_bytes(sub, max_points) > stage_each ? set_err("msurf_sweep_jobs_capped: staging too small")
                                                       : staged_launch(sub, max_points, q);
      } else {
        sub.stage = nullptr;
        rc = sweep_impl(nullptr, 1, nullptr, 0, mode, max_points, q, &sub, nullptr);
      }
      if (rc == 0 && i + 1 < n) rc = zcap_refresh_after(sub, stock, q);
    }
  }
  for (int j = 0; j < n_jobs; ++j)  // joins are enqueued whatever happened
    for (int d = 0; d < depth; ++d) {
      cudaStream_t q = lib_stream(sid(j, d));
      cudaEvent_t join = nullptr;
      if (!q || cudaEventCreateWithFlags(&join, cudaEventDisableTiming) != cudaSuccess) continue;
      cudaEventRecord(join, q);
      cudaStreamWaitEvent(st, join, 0);
      cudaEventDestroy(join);
    }
  cudaEventDestroy(fork);
  return rc;
}

int msurf_decode(uint64_t* keys, int64_t count, int32_t n_surf, const double* sentinel,
                 unsigned long long* machined, void* stream) {
  if (count < 0 || n_surf < 1 || !keys || !machined || !sentinel)
    return set_err("msurf_decode: bad arguments");
  if (count == 0) return 0;
  long long blocks = (count / 2 + kThreads - 1) / kThreads;
  const long long cap = n_surf > 1 ? 64 : 148 * 16;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  dim3 grid((unsigned)blocks, (unsigned)n_surf);
  decode_kernel<<<grid, kThreads, 0, (cudaStream_t)stream>>>(keys, count, sentinel, machined);
  return check_launch("decode_kernel");
}

int msurf_decode_strips(const uint64_t* keys, double* heights, int64_t rows, int64_t ld_out, int32_t n_strips,
                        const int64_t* col0, const double* sentinel, unsigned long long* machined, void* stream) {
  if (!keys || !heights || !col0 || !sentinel || !machined || rows < 1 || n_strips < 1 || ld_out < 1)
    return set_err("msurf_decode_strips: bad arguments");
  long long blocks = rows < 148 * 8 ? rows : 148 * 8;
  dim3 grid((unsigned)blocks, (unsigned)n_strips);
  decode_strips_kernel<<<grid, kThreads, 0, (cudaStream_t)stream>>>(keys, heights, rows, ld_out,
                                                                    reinterpret_cast<const long long*>(col0),
                                                                    sentinel, machined);
  return check_launch("decode_strips_kernel");
}

// blocks per surface: ~4096 elements per block, at most one per row, at most
// MSURF_RED_BLOCKS; a pure function of the ROI shape, so reductions are
// bit-reproducible run to run
static int red_blocks(int64_t rows, int64_t cols) {
  long long nb = rows * cols / 4096;
  if (nb > rows) nb = rows;
  if (nb > MSURF_RED_BLOCKS) nb = MSURF_RED_BLOCKS;
  return (int)(nb < 1 ? 1 : nb);
}

int msurf_areal_pass1(const double* h, int64_t ld, int64_t surf_stride, int32_t n_surf,
                      int64_t i_lo, int64_t j_lo, int64_t rows, int64_t cols,
                      const double* sentinel, int32_t exclude_uncut, double* work,
                      double* out1, void* stream) {
  if (!h || !work || !out1 || !sentinel || n_surf < 1 || rows < 1 || cols < 1 || i_lo < 0 || j_lo < 0 || ld < cols)
    return set_err("msurf_areal_pass1: bad arguments");
  const int nb = red_blocks(rows, cols);
  cudaStream_t st = (cudaStream_t)stream;
  areal_pass1_kernel<<<dim3(nb, n_surf), kThreads, 0, st>>>(h, ld, surf_stride, i_lo, j_lo, rows, cols,
                                                           sentinel, exclude_uncut, work);
  if (check_launch("areal_pass1_kernel")) return 1;
  finalize_stats1_kernel<<<n_surf, kThreads, 0, st>>>(work, nb, out1);
  return check_launch("finalize_stats1_kernel");
}

int msurf_areal_pass2(const double* h, int64_t ld, int64_t surf_stride, int32_t n_surf,
                      int64_t i_lo, int64_t j_lo, int64_t rows, int64_t cols,
                      const double* sentinel, int32_t exclude_uncut, const double* stats1,
                      double* work, double* out2, void* stream) {
  if (!h || !work || !out2 || !stats1 || !sentinel || n_surf < 1 || rows < 1 || cols < 1 || i_lo < 0 || j_lo < 0 || ld < cols)
    return set_err("msurf_areal_pass2: bad arguments");
  const int nb = red_blocks(rows, cols);
  cudaStream_t st = (cudaStream_t)stream;
  areal_pass2_kernel<<<dim3(nb, n_surf), kThreads, 0, st>>>(h, ld, surf_stride, i_lo, j_lo, rows, cols,
                                                           sentinel, exclude_uncut, stats1, work);
  if (check_launch("areal_pass2_kernel")) return 1;
  finalize_kernel<4><<<n_surf, kThreads, 0, st>>>(work, nb, 0u, out2);
  return check_launch("finalize_kernel<4>");
}

int msurf_areal_plane_pass1(const double* h, int64_t ld, int64_t surf_stride, int32_t n_surf,
                            int64_t i_lo, int64_t j_lo, int64_t rows, int64_t cols,
                            const double* sentinel, int32_t exclude_uncut, double* work, double* out,
                            void* stream) {
  if (!h || !work || !out || !sentinel || n_surf < 1 || rows < 1 || cols < 1 || i_lo < 0 || j_lo < 0 ||
      ld < cols)
    return set_err("msurf_areal_plane_pass1: bad arguments");
  const int nb = red_blocks(rows, cols);
  cudaStream_t st = (cudaStream_t)stream;
  plane_pass1_kernel<<<dim3(nb, n_surf), kThreads, 0, st>>>(h, ld, surf_stride, i_lo, j_lo, rows, cols,
                                                           sentinel, exclude_uncut, work);
  if (check_launch("plane_pass1_kernel")) return 1;
  finalize_kernel<10><<<n_surf, kThreads, 0, st>>>(work, nb, 0u, out);
  return check_launch("finalize_kernel<10>");
}

int msurf_areal_plane_pass2(const double* h, int64_t ld, int64_t surf_stride, int32_t n_surf,
                            int64_t i_lo, int64_t j_lo, int64_t rows, int64_t cols,
                            const double* sentinel, int32_t exclude_uncut, const double* coef,
                            double* work, double* out, void* stream) {
  if (!h || !work || !out || !sentinel || !coef || n_surf < 1 || rows < 1 || cols < 1 || i_lo < 0 ||
      j_lo < 0 || ld < cols)
    return set_err("msurf_areal_plane_pass2: bad arguments");
  const int nb = red_blocks(rows, cols);
  cudaStream_t st = (cudaStream_t)stream;
  plane_pass2_kernel<<<dim3(nb, n_surf), kThreads, 0, st>>>(h, ld, surf_stride, i_lo, j_lo, rows, cols,
                                                           sentinel, exclude_uncut, coef, work);
  if (check_launch("plane_pass2_kernel")) return 1;
  finalize_kernel<6><<<n_surf, kThreads, 0, st>>>(work, nb, (1u << 8) | (2u << 10), out);
  return check_launch("finalize_kernel<6>");
}

int msurf_profiles(const double* h, int64_t surf_stride, int32_t n_surf, const int64_t* start,
                   int32_t n_prof, int64_t len, int64_t stride, const double* sentinel,
                   int32_t exclude_uncut, const double* stats_in, double* out, void* stream) {
  if (!h || !start || !out || !sentinel || n_surf < 1 || n_prof < 1 || len < 1 || stride < 1)
    return set_err("msurf_profiles: bad arguments");
  profiles_kernel<<<dim3(n_prof, n_surf), kThreads, 0, (cudaStream_t)stream>>>(
      h, surf_stride, reinterpret_cast<const long long*>(start), n_prof, len, stride, sentinel,
      exclude_uncut, stats_in, out);
  return check_launch("profiles_kernel");
}

int msurf_graymap_range(const double* h, int64_t ld, int64_t i_lo, int64_t j_lo, int64_t rows, int64_t cols,
                        const double* sentinel, double* work, double* out3, void* stream) {
  if (!h || !sentinel || !work || !out3 || rows < 1 || cols < 1 || i_lo < 0 || j_lo < 0 || ld < cols)
    return set_err("msurf_graymap_range: bad arguments");
  const int nb = red_blocks(rows, cols);
  cudaStream_t st = (cudaStream_t)stream;
  graymap_range_kernel<<<nb, kThreads, 0, st>>>(h, ld, i_lo, j_lo, rows, cols, sentinel, work);
  if (check_launch("graymap_range_kernel")) return 1;
  finalize_kernel<3><<<1, kThreads, 0, st>>>(work, nb, 1u | (2u << 2), out3);
  return check_launch("finalize_kernel<3>");
}

int msurf_graymap_pixels(const double* h, int64_t ld, int64_t i_lo, int64_t j_lo, int64_t rows, int64_t cols,
                         const double* sentinel, const double* range3, uint16_t* pixels, void* stream) {
  if (!h || !sentinel || !range3 || !pixels || rows < 1 || cols < 1 || i_lo < 0 || j_lo < 0 || ld < cols)
    return set_err("msurf_graymap_pixels: bad arguments");
  if ((rows + 31) / 32 > 65535) return set_err("msurf_graymap_pixels: roi too tall");
  dim3 grid((unsigned)((cols + 31) / 32), (unsigned)((rows + 31) / 32));
  graymap_pixels_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(h, ld, i_lo, j_lo, rows, cols, sentinel, range3,
                                                               reinterpret_cast<unsigned short*>(pixels));
  return check_launch("graymap_pixels_kernel");
}

int msurf_microbench(int32_t which, double* result) {
  if (!result) return set_err("msurf_microbench: null result");
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms = 0.f;
  if (which == 0 || which == 1) {
    double* out = nullptr;
    if (cudaMalloc(&out, 8) != cudaSuccess) return set_err("microbench: cudaMalloc");
    const int blocks = sms * 8, threads = 256, iters = 4096;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      if (which == 0) mb_dp_kernel<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
      else mb_fma_kernel<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
    }
    cudaEventElapsedTime(&ms, a, b);
    cudaFree(out);
    const double ops = (double)blocks * threads * iters * 8.0 * (which == 0 ? 2.0 : 1.0);
    *result = ops / (ms * 1e-3);
  } else if (which == 2 || which == 3 || which == 4) {
    unsigned long long* buf = nullptr;
    // 2: 128 MiB of keys (about the L2 size); 3, 4: 32 MiB (L2-resident, the
    // size of one sweep job's Z-map slab)
    const long long n = which == 2 ? (1ll << 24) : (1ll << 22);
    if (cudaMalloc(&buf, n * 8) != cudaSuccess) return set_err("microbench: cudaMalloc");
    cudaMemset(buf, 0xff, n * 8);
    const int blocks = sms * 8, threads = 256, iters = 256;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(a);
      if (which == 4) mb_atomic_run_kernel<<<blocks, threads>>>(buf, n - 1, iters);
      else mb_atomic_kernel<<<blocks, threads>>>(buf, n - 1, iters);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
    }
    cudaEventElapsedTime(&ms, a, b);
    cudaFree(buf);
    *result = (double)blocks * threads * iters / (ms * 1e-3);
  } else if (which >= 33 && which <= 64) {
    // RED.MIN warp instructions/s touching L = which - 32 lines each, 32 MiB table
    const int L = which - 32;
    unsigned long long* buf = nullptr;
    const long long n = 1ll << 22;
    if (cudaMalloc(&buf, n * 8) != cudaSuccess) return set_err("microbench: cudaMalloc");
    cudaMemset(buf, 0xff, n * 8);
    const int blocks = sms * 8, threads = 256, iters = 256;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(a);
      mb_atomic_lines_kernel<<<blocks, threads>>>(buf, (unsigned)((n >> 4) - 1), L, iters);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
    }
    cudaEventElapsedTime(&ms, a, b);
    cudaFree(buf);
    *result = (double)blocks * (threads / 32) * iters / (ms * 1e-3);
  } else {
    return set_err("msurf_microbench: unknown kind");
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return check_launch("microbench");
}

}  // extern "C"
