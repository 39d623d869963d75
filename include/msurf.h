/* msurf.h — C ABI of libmsurf.so, the B200 (sm_100a) FSM surface-topography
 * hot path. Plain POD structs, plain pointers and sizes, explicit CUDA stream
 * (passed as void*), int status + thread-local msurf_last_error().
 *
 * The reference (arXiv 2603.28160, package `millsurf`) is pure Python/NumPy
 * and has no FFI of its own; each entry point below replaces the reference
 * function it cites (file:line under /root/reference/pkg/src/millsurf/), and
 * the Python host package paper_2603_28160_b200 binds them with ctypes
 * (INTEGRATION.md shows the binding a maintainer would add to millsurf).
 *
 * Device buffers are caller-owned (the Python host allocates them with
 * PyTorch); no entry point allocates on the hot path.
 */
#ifndef MSURF_H
#define MSURF_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MSURF_ABI_VERSION 7

/* kinematics mode of a sweep launch (uniform across the jobs of one launch) */
#define MSURF_MODE_REF 0      /* reference composite-matrix order, engine.py:257-296 */
#define MSURF_MODE_EXT 1      /* rotated tool-frame points, z' time-invariant   */
#define MSURF_MODE_EXT_TILT 2 /* rotated tool-frame points + lead tilt (z' per step) */
#define MSURF_MODE_MASK 0xff  /* the kinematics mode bits of a mode word */
/* OR-ed into the mode of msurf_sweep: also count the per-point diagnostics
 * MSURF_CTR_DEPOSITS / MSURF_CTR_ATOMICS (two extra integer ops per point;
 * without it those two counters stay zero) */
#define MSURF_SWEEP_DIAG 0x100
/* OR-ed into the mode: the diagnostics counters plus a trace of every
 * warp-wide RED.MIN of the main point loops into the buffer armed with
 * msurf_trace_arm (roofline measurement only; much slower) */
#define MSURF_SWEEP_TRACE 0x200
/* OR-ed into the mode of msurf_sweep_job (EXT_TILT): eight warps per 64-step
 * CTA instead of one (phase 2 units of heavy tiles spread over more warps) */
#define MSURF_SWEEP_WIDE 0x400

#define MSURF_CTR_LIVE_ROWS 0  /* (step, tooth, pass) rows with >= 1 chunk surviving the 2-D cull */
#define MSURF_CTR_EVAL 1       /* edge points evaluated (points of surviving 32-point chunks)    */
#define MSURF_CTR_DEPOSITS 2   /* evaluated points landing in the owned grid (P_in)              */
#define MSURF_CTR_ATOMICS 3    /* RED.MIN issued after the time-neighbour pre-reduction          */
#define MSURF_CTR_ENGAGED_ROWS 4 /* rows whose whole-tooth 2-D box meets the window (SURVEY P_eng/N) */
#define MSURF_NUM_CTRS 5

/* One surface sweep (one parameter set; one strip of it under sharding).
 * Replaces the per-worker body engine.py:215-313 (_run_step_range) for all
 * steps x teeth x edge points x raster passes of one surface.
 * Layout: 8-byte fields first, then 4-byte fields, no implicit padding. */
typedef struct msurf_job {
  /* grid (surface_grid.py:25-75): node (i,j) at (x_min+i*spacing, y_min+j*spacing) */
  double spacing, x_min, y_min;
  int64_t m, n;      /* cell counts; nodes (m+1) x (n+1)                       */
  int64_t j_lo, j_hi; /* owned feed-direction node columns [j_lo, j_hi]          */
  int64_t ld;        /* keys row pitch in nodes (>= j_hi - j_lo + 1)            */
  uint64_t* keys;    /* device: node (i, j) at keys[i * ld + (j - j_lo)],        *
                      * order-preserving u64 keys of the heights                 */
  /* time (engine.py:152-170, 240-241) */
  double t_start, dt;
  int64_t steps;     /* time steps of one pass (engine.py:170)                   */
  int64_t step_lo, step_hi; /* this job sweeps steps [step_lo, step_hi) of every pass:
                      * the window whose footprint can reach the owned columns */
  double y0, feed_speed, omega;
  /* per-tooth / per-point device arrays */
  const double* tooth_base;  /* [teeth] phase + (2pi)(K-1)/Z (kinematics.py:76)      */
  const double* tooth_rows;  /* REF: [teeth][8] e00 e01 e02 e03 e10 e11 e12 e13      */
  const double* pts;         /* [teeth][points][4] per-point record (16-B aligned):
                              * REF      (xp, yp, zp, key of z')  edge frame
                              * EXT      (xt, yt, key of z', 0)   tool frame
                              * EXT_TILT (xt, yt, sin(tau)*zt, cos(tau)*zt + zoff)  */
  const double* tooth_box;   /* [teeth][6] whole-tooth tool-frame box (P_eng counter)  */
  const double* chunk_circ;  /* [teeth][nchunk][6] cull record per 32-point chunk:
                              * (xc, yc, rx, ry, yz, 0) — see planner._chunk_circles */
  const float* chunk_f32;    /* [teeth][nchunk][8] fp32 copy the kernel's phase-1 cull
                              * reads: (xc, yc, rx, ry, yz, Rt, 0, 0), Rt = the tooth's
                              * bound max|x| + max|y| + max|z| (planner.chunk_f32)    */
  const double* pass_x0;     /* [passes] spindle x of each raster pass               */
  /* extended kinematics */
  double tilt_c, tilt_s, zoff;  /* zoff: surface z offset (EXT_TILT: folded into pts) */
  double vib_amp, vib_omega, vib_phase;
  /* optional host-libm trig tables (parity mode); NULL = device sincos */
  const double* trig_table;  /* [steps][teeth][2] = cos, sin of the tooth angle      */
  const double* vib_table;   /* [steps] sin(vib_omega*t + vib_phase)                  */
  /* optional trajectory record (REF mode, pass 0): per (step, tooth) the
   * workpiece x', y', z' of edge point min_index[tooth] (engine.py:266-270) */
  double* traj;              /* device [steps][teeth][3] or NULL                      */
  const int32_t* min_index;  /* [teeth] argmin of z' (engine.py:189)                  */
  unsigned long long* counters; /* device [MSURF_NUM_CTRS], accumulated             */
  /* optional surface-cap cull (EXT_TILT by-value launches): per 32x32-node tile
   * of this job's slab (row-major, ceil(w/32) tiles per row, w = j_hi-j_lo+1)
   * an upper bound of (current height - stock height), maintained between
   * launches by msurf_zcap_refresh; a (step, chunk) whose lowest reachable z'
   * lies above the bound of every tile it can touch is skipped. NULL = off. */
  const float* zcap;
  /* optional staging (set by msurf_sweep_jobs_capped for its EXT_TILT
   * launches, NULL otherwise): phase 1 writes each live tile's rows and chunk
   * masks plus the list of live (tile, chunk) units here, and a second,
   * persistent kernel balances phase 2 over all warps of the GPU */
  void* stage;
  int32_t teeth, points, passes;
  int32_t tooth_lo;  /* this launch sweeps teeth [tooth_lo, tooth_lo + tooth_n) ... */
  int32_t tooth_n;   /* ... of the `teeth` (0: all); per-tooth arrays stay indexed by the tooth */
  int32_t reserved0;
} msurf_job;

int msurf_abi_version(void);
/* edge length in nodes of a surface-cap tile (msurf_job.zcap holds one float
 * per tile of a job's slab, ceil(rows / t) x ceil(w / t) row-major) */
int msurf_zcap_tile(void);
const char* msurf_last_error(void);
int msurf_sizeof_job(void);

/* Initialise n_surf contiguous surfaces of `count` keys each with the key of
 * value[s] (device array): HeightField init to the stock height, surface_grid.py:107-108. */
int msurf_fill_keys(uint64_t* keys, int64_t count, int32_t n_surf, const double* value,
                    void* stream);

/* The FSM sweep (engine.py:215-313 / 316-357). `jobs` is a DEVICE array of
 * n_jobs descriptors; `tile_prefix` a DEVICE array of n_jobs+1 exclusive
 * prefix sums of tiles per job,
 * tiles(job) = passes*teeth*ceil((step_hi-step_lo)/tile_steps).
 * tile_steps must be msurf_tile_steps(). Deposits are atomicMin on keys, so
 * the result is independent of scheduling (engine.py:316-317 determinism).
 * `scratch` is DEVICE memory of at least 8 * (n_tiles + 1) bytes: the sweep
 * first pre-culls the tiles (a tile whose tooth box cannot reach its job's
 * window does no work) into a list there, then persistent CTAs walk it. */
int msurf_tile_steps(void);
int msurf_sweep(const msurf_job* jobs, int32_t n_jobs, const int64_t* tile_prefix,
                int64_t n_tiles, int32_t mode, int32_t max_points, void* scratch, void* stream);

/* The same sweep for ONE job given as a HOST pointer: the descriptor is
 * passed by value as a kernel parameter, so the kernel reads its fields as
 * constant-bank operands (fewer registers, no per-CTA descriptor copy). The
 * library picks the CTA shape for the mode and sizes the grid itself. Device
 * pointers inside the job are used as in msurf_sweep. */
int msurf_sweep_job(const msurf_job* job, int32_t mode, int32_t max_points, void* stream);

/* Surface-cap refresh for msurf_job.zcap: for every 32x32-node tile of a
 * rows x cols slab of keys (row pitch ld), the maximum height minus stock[0]
 * (device double), rounded up to float, into zcap (row-major tiles,
 * ceil(cols/32) per row). Heights only decrease during a sweep, so a bound
 * taken at any earlier moment stays an upper bound. stop_reset (device int,
 * may be NULL) is zeroed: the flag of the msurf_zcap_watch that follows. */
int msurf_zcap_refresh(const uint64_t* keys, int64_t ld, int64_t rows, int64_t cols, const double* stock,
                       float* zcap, int32_t* stop_reset, void* stream);

/* msurf_sweep_job with the surface-cap cull (EXT_TILT): job->zcap must point
 * at the job's cap tiles. Computes the caps of the (filled) slab, then sweeps
 * the job (pass, tooth) by (pass, tooth) (mode may include MSURF_SWEEP_WIDE)
 * refreshing the caps after each launch, so every launch skips the
 * (step, chunk) pairs that cannot reach below what the earlier ones cut.
 * stock: device double (the stock height). Results equal msurf_sweep_job's. */
int msurf_sweep_job_capped(const msurf_job* job, int32_t mode, int32_t max_points, const double* stock,
                           void* stream);
/* n_jobs capped jobs (HOST array; disjoint slabs, e.g. the L2 sub-strips of a
 * surface) swept concurrently on library-owned non-blocking streams forked
 * from and joined back into `stream` (graph-capturable): each job's (pass,
 * tooth) launches go round-robin over `depth` streams of its own, so up to
 * `depth` of them overlap (caps read at most depth - 1 launches stale: a
 * weaker cull, never another result), depth <= 4. Job j runs in stream slot
 * slot0 + j (<= 8 slots; slot 0 has the highest stream priority, so side-by-
 * side jobs finish in slot order); a caller may issue the jobs of one surface
 * in separate calls with distinct slots and different `stream`s to join each
 * job separately.
 * stocks: HOST array of device pointers to each job's stock height. */
int msurf_sweep_jobs_capped(const msurf_job* jobs, int32_t n_jobs, int32_t mode, int32_t max_points,
                            const int64_t* stocks, int32_t depth, void* stage, int64_t stage_each, int32_t slot0,
                            void* stream);
/* With `stage` (device, n_jobs x depth buffers of stage_each >= msurf_stage_bytes
 * bytes) the production launches run staged: phase 1 of every tile writes
 * its rows, masks and live (tile, chunk) units there, then a persistent
 * kernel balances phase 2 over every warp. NULL: the single-kernel form. */
int msurf_stage_bytes(const msurf_job* job, int32_t max_points, int64_t* bytes);
/* Plumbing for per-job joins: a library-owned non-blocking anchor stream
 * (k < 16), and "waiter waits for everything enqueued on signaler so far"
 * (an event recorded on signaler, waited on by waiter). */
void* msurf_anchor_stream(int32_t k);
int msurf_stream_wait(void* waiter, void* signaler);

/* Decode keys to fp64 heights in place and count machined cells
 * (HeightField.machined_cell_count, surface_grid.py:128-129). Batched over
 * n_surf surfaces of `count` nodes each, contiguous; sentinel[n_surf] (the
 * initial stock height of each surface) and machined[n_surf] are device
 * arrays, machined is accumulated. */
int msurf_decode(uint64_t* keys, int64_t count, int32_t n_surf, const double* sentinel,
                 unsigned long long* machined, void* stream);

/* Decode for a surface whose keys are stored in sub-strip layout: strip k
 * (columns [col0[k], col0[k+1]) of the surface, col0 a DEVICE array of
 * n_strips+1 offsets from the surface's first column) is a contiguous
 * rows x w_k block at keys + rows*col0[k]; writes row-major fp64 heights
 * (node (i, c) at heights[i*ld_out + c]) and adds the machined-cell count to
 * machined[0]. Used for surfaces cut into L2-sized sub-strips: each sweep job
 * then deposits into one contiguous slab. */
int msurf_decode_strips(const uint64_t* keys, double* heights, int64_t rows, int64_t ld_out, int32_t n_strips,
                        const int64_t* col0, const double* sentinel, unsigned long long* machined, void* stream);

/* Areal roughness moments (roughness.py:93-135, leveling='mean').
 * h: device fp64 heights, row-major with leading dimension ld; surface s
 * starts at h + s*surf_stride. ROI rows [i_lo, i_lo+rows), cols [j_lo, j_lo+cols).
 * sentinel[n_surf] device. exclude_uncut=0 counts uncut cells (the host raises
 * DomainError like roughness.py:86-89); =1 skips them. Reductions are
 * deterministic (fixed block partition, fixed-order tree): reruns are
 * bit-identical. work: device scratch of n_surf * MSURF_WORK_DOUBLES doubles
 * (the plane-leveling passes below need * 10).
 * pass1 -> stats1[s][6] = sum z_um, max z_um, min z_um, n_used, n_uncut, mean
 *          (sum in double-double, mean = sum / n rounded once)
 * pass2 reads the mean stats1[s][5] (under strip sharding the caller
 * all-reduces stats1 and recomputes the mean first, so it is global)
 *       -> out2[s][4] = sum|d|, sum d^2, sum d^3, sum d^4 */
#define MSURF_RED_BLOCKS 1024
/* scratch doubles per surface for every reduction below (at most
 * MSURF_RED_BLOCKS blocks x 10 partials: plane pass 1) */
#define MSURF_WORK_DOUBLES (MSURF_RED_BLOCKS * 10)
int msurf_areal_pass1(const double* h, int64_t ld, int64_t surf_stride, int32_t n_surf,
                      int64_t i_lo, int64_t j_lo, int64_t rows, int64_t cols,
                      const double* sentinel, int32_t exclude_uncut, double* work,
                      double* stats1, void* stream);
int msurf_areal_pass2(const double* h, int64_t ld, int64_t surf_stride, int32_t n_surf,
                      int64_t i_lo, int64_t j_lo, int64_t rows, int64_t cols,
                      const double* sentinel, int32_t exclude_uncut, const double* stats1,
                      double* work, double* out2, void* stream);

/* Plane leveling (roughness.py:108-113, leveling='plane'): pass 1 writes the
 * normal-equation sums per surface, out[s][10] = n, Si, Sj, Sii, Sjj, Sij, Sz,
 * Siz, Sjz, n_uncut (i, j = offsets inside the ROI, z in um); the host solves
 * the 3x3 system for z ~ a*i + b*j + c; pass 2 with coef[s][3] = (a, b, c)
 * writes out[s][6] = S|d|, Sd^2, Sd^3, Sd^4, max d, min d of d = z - plane.
 * work: n_surf * MSURF_WORK_DOUBLES doubles. */
int msurf_areal_plane_pass1(const double* h, int64_t ld, int64_t surf_stride, int32_t n_surf,
                            int64_t i_lo, int64_t j_lo, int64_t rows, int64_t cols,
                            const double* sentinel, int32_t exclude_uncut, double* work, double* out,
                            void* stream);
int msurf_areal_plane_pass2(const double* h, int64_t ld, int64_t surf_stride, int32_t n_surf,
                            int64_t i_lo, int64_t j_lo, int64_t rows, int64_t cols,
                            const double* sentinel, int32_t exclude_uncut, const double* coef,
                            double* work, double* out, void* stream);

/* Profile roughness (roughness.py:138-188; Rz = Rp + Rv is the product's
 * extension). Profile p of surface s: `len` samples starting at
 * h + s*surf_stride + start[p], spaced `stride` (1 = feed profile, ld =
 * pick-feed); sentinel[n_surf] device. If stats_in is NULL each block uses
 * its own mean (single GPU); otherwise mean = stats_in[k][0]/stats_in[k][1]
 * of the caller's all-reduced first pass (strip-sharded profiles).
 * out[k = s*n_prof+p][8] = sum z_um, n_used, n_uncut, max z_um, min z_um,
 * sum|z - mean|, mean, 0 */
int msurf_profiles(const double* h, int64_t surf_stride, int32_t n_surf,
                   const int64_t* start, int32_t n_prof, int64_t len, int64_t stride,
                   const double* sentinel, int32_t exclude_uncut, const double* stats_in,
                   double* out, void* stream);

/* Host-side planning arrays of one surface (planner.py, native so a
 * single-surface simulate() spends microseconds before the GPU starts;
 * bitwise identical to the NumPy statement). Scalars (validation, span,
 * engaged half-length, edge->tool rows, helix/runout/tilt constants, noise)
 * come from the Python planner. */
typedef struct msurf_geom_in {
  int32_t mode;              /* MSURF_MODE_*                                          */
  int32_t teeth, points;
  int32_t profile;           /* EXT: 0 insert arc at D/2, 1 ball meridian              */
  double radius;             /* insert / ball radius R                                 */
  double half;               /* insert: engaged half-length (edge l in [-half, half])  */
  double kmax;               /* ball: maximum polar angle                              */
  double tan_beta_over_r;    /* EXT helix: tan(beta)/r_ref, 0 = none                    */
  double tilt_c, tilt_s;     /* EXT_TILT: cos, sin of the lead tilt                     */
  double z0;                 /* REF: spindle z0 (zw = ((e20 x + e21 y) + e22 z) + (e23 + z0)) */
  const double* rows;        /* [teeth][12] edge->tool rows 0..2 (4 columns each)       */
  const double* delta;       /* EXT edge noise [teeth][points] or NULL                  */
  const double* runout_xy;   /* EXT tool-axis runout offsets [teeth][2] or NULL         */
} msurf_geom_in;

/* REF: px/py/pz [points] = edge-frame SoA. EXT: [teeth][points] tool-frame
 * points (profile, noise, rows, helix, runout); stats2 = (z_shift, max|zt|). */
int msurf_plan_geometry(const msurf_geom_in* in, double* px, double* py, double* pz, double* stats2);
/* With the surface z offset zoff: device point records pts [teeth][points][4]
 * (msurf_job.pts), tooth_box [teeth][6], chunk_circ / chunk_box
 * [teeth][nchunk][6], min_index [teeth]; optional zw_out / key_out
 * [teeth][points] (z' and its order-preserving key). */
int msurf_plan_finish(const msurf_geom_in* in, const double* px, const double* py, const double* pz, double zoff,
                      double* pts, double* tooth_box, double* chunk_circ, double* chunk_box, int32_t* min_index,
                      double* zw_out, uint64_t* key_out);

/* The two planning steps for n parameter sets of one geometry family (equal
 * teeth and points, EXT modes), set b in slice b of every output; `threads`
 * host threads split the sets. */
int msurf_plan_geometry_many(const msurf_geom_in* ins, int32_t n, double* px, double* py, double* pz,
                             double* stats2, int32_t threads);
int msurf_plan_finish_many(const msurf_geom_in* ins, int32_t n, const double* px, const double* py, const double* pz,
                           const double* zoff, double* pts, double* tooth_box, double* chunk_circ, double* chunk_box,
                           int32_t* min_index, double* zw_out, uint64_t* key_out, int32_t threads);

/* Graymap export (surface_io.py:100-131, write_graymap) of one fp64 height
 * field (row pitch ld) over the ROI rows [i_lo, i_lo+rows) x cols
 * [j_lo, j_lo+cols). msurf_graymap_range: out3 = (max, min, n) of the
 * machined cells (height < sentinel[0]) in mm; work: MSURF_WORK_DOUBLES.
 * msurf_graymap_pixels: pixels[j * rows + i] (image row = y node, column = x
 * node) = big-endian u16 of rint((z - min) * (65535 / (max - min))) for
 * machined cells, 32768 when max == min, 0 for uncut cells; range3 = out3 of
 * the range pass (device). The caller raises DomainError when n == 0. */
int msurf_graymap_range(const double* h, int64_t ld, int64_t i_lo, int64_t j_lo, int64_t rows, int64_t cols,
                        const double* sentinel, double* work, double* out3, void* stream);
int msurf_graymap_pixels(const double* h, int64_t ld, int64_t i_lo, int64_t j_lo, int64_t rows, int64_t cols,
                         const double* sentinel, const double* range3, uint16_t* pixels, void* stream);

/* Microbenchmarks for the roofline denominators (not in MEASURED_PEAKS.json):
 * which=0: non-FMA DADD/DMUL issue (ops/s), which=1: DFMA (FMA/s),
 * which=2: 64-bit atomicMin (RED.MIN.64) to random addresses in a 128 MiB
 * table (~L2 size), which=3: the same in a 32 MiB (L2-resident) table,
 * which=4: RED.MIN.64 where each warp instruction covers one 256-byte run of
 * consecutive keys at a random base in 32 MiB (ops/s);
 * which=32+L (L = 1..32): warp RED.MIN.64 instructions/s when each touches L
 * distinct random 128-byte lines of a 32 MiB table (lane l on line l % L). Synchronous; creates and destroys its own scratch. */
int msurf_microbench(int32_t which, double* result);

/* RED roof of a workload (roofline measurement, not on the product path).
 * msurf_trace_arm: the next MSURF_SWEEP_TRACE sweeps append one record per
 * warp-wide RED.MIN — 32 u32 key offsets from `base` (0xffffffff = lane
 * inactive) — to `trace` (device, room for cap_records records), counting
 * records issued and active lanes in counters[0..1] (device, caller-zeroed;
 * records beyond the capacity are counted, not stored).
 * msurf_red_lines: hist[L] += records touching L distinct 128-byte lines
 * (hist: 33 device u64, caller-zeroed). With msurf_microbench(32 + L) (warp
 * RED.MIN instructions/s of that shape) this prices the sweep's own RED
 * stream at the L2 atomic throughput. */
int msurf_trace_arm(uint32_t* trace, int64_t cap_records, unsigned long long* counters, const uint64_t* base);
int msurf_red_lines(const uint32_t* trace, int64_t n_records, unsigned long long* hist, void* stream);
/* msurf_red_sectors: the same line histogram plus hist_sectors[S] += records
 * touching S distinct 32-byte sectors (both 33 device u64, caller-zeroed).
 * The L2 atomic units' throughput is close to constant per sector update
 * across warp RED shapes (msurf_microbench(32 + L): 1.2-1.9e11 sectors/s
 * while the line-update rate spans 4x), so the sector count of the sweep's
 * own RED stream over the best measured sector rate is its atomic roof. */
int msurf_red_sectors(const uint32_t* trace, int64_t n_records, unsigned long long* hist_lines,
                      unsigned long long* hist_sectors, void* stream);

/* Small-result readback without the copy engines: msurf_host_alloc returns
 * page-locked host memory mapped into the device address space (NULL on
 * failure); msurf_readback enqueues on `stream` a kernel that stores `bytes`
 * (a multiple of 8) from device memory `src` into such a buffer over PCIe.
 * A D2H cudaMemcpy of a few bytes would queue behind any large D2H copy
 * already in flight (the heights prefetch); these stores do not. The data is
 * valid on the host once the stream has passed the kernel (event sync). */
void* msurf_host_alloc(int64_t bytes);
int msurf_host_free(void* p);
int msurf_readback(const void* src, void* host_dst, int64_t bytes, void* stream);
/* msurf_readback, then block the calling thread until `stream` has passed the
 * kernel (cudaStreamSynchronize): one call per small result on the host
 * path, the data is valid on return. */
int msurf_readback_sync(const void* src, void* host_dst, int64_t bytes, void* stream);

/* Enqueue on `stream` a D2H copy of a rows x width_bytes block (pitches in
 * bytes, cudaMemcpy2DAsync): one feed-direction sub-strip of a row-major
 * height map into the matching columns of a page-locked host map, so the
 * heights of a strip-layout surface cross PCIe strip by strip while the
 * later strips are still being swept. */
int msurf_copy2d_d2h(void* host_dst, int64_t dst_pitch, const void* src, int64_t src_pitch,
                     int64_t width_bytes, int64_t rows, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* MSURF_H */
