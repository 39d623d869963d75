// msurf_plan.cpp — host-side planning arrays for one surface (the O(teeth x
// edge points) part of planner.py), native so a single-surface simulate()
// spends microseconds, not a NumPy-bound fraction of a millisecond, before
// the GPU starts. Every value is bitwise identical to planner.py (the Python
// statement stays the specification; tests/test_native_plan_cpu.py compares
// the two on the reference goldens, the extended cases and the BASELINE
// configs): one IEEE rounding per operation in the order the NumPy
// expressions evaluate (built with -ffp-contract=off), libm sin/cos/sqrt as
// NumPy uses them, reductions that are exact (min/max/argmin, first index on
// ties).
#ifndef _GNU_SOURCE
#define _GNU_SOURCE  // sincos
#endif
#include <math.h>
#include <stdint.h>
#include <string.h>

#include <functional>
#include <vector>

#include "msurf.h"

namespace {

constexpr int kChunk = 32;

inline uint64_t enc_key(double z) {
  z = z + 0.0;  // -0 -> +0
  uint64_t b;
  memcpy(&b, &z, 8);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

inline double key_as_double(uint64_t k) {
  double d;
  memcpy(&d, &k, 8);
  return d;
}

// edge_coordinates (planner.py / geometry.py): l = -half + ((2 half) i)/(n-1),
// endpoints exact; y = 0; z = r - sqrt(r*r - l*l)
void edge_coords(double half, int n, double r, double* x, double* z) {
  const double c = 2.0 * half;
  for (int i = 0; i < n; ++i) x[i] = -half + (c * (double)i) / (double)(n - 1);
  x[0] = -half;
  x[n - 1] = half;
  const double rr = r * r;
  for (int i = 0; i < n; ++i) z[i] = r - sqrt(rr - x[i] * x[i]);
}

// exact min/max of non-NaN values without a libm call (fmin/fmax are PLT calls
// in this build); ties keep the first value, as the tests check bitwise
inline double mn(double a, double b) { return b < a ? b : a; }
inline double mx(double a, double b) { return b > a ? b : a; }

// _chunk_boxes + _chunk_circles + tooth box for one tooth's (x, y, z) rows
void chunk_records(const double* x, const double* y, const double* z, int n, double tc, double ts,
                   double* box /*[nchunk][6]*/, double* circ /*[nchunk][6]*/, double* tbox /*[6]*/) {
  const int nchunk = (n + kChunk - 1) / kChunk;
  for (int k = 0; k < 6; ++k) tbox[k] = (k & 1) ? -INFINITY : INFINITY;
  for (int q = 0; q < nchunk; ++q) {
    const int a = q * kChunk, b = a + kChunk < n ? a + kChunk : n;  // the padding repeats element n-1
    double xl = x[a], xh = x[a], yl = y[a], yh = y[a], zl = z[a], zh = z[a];
    for (int i = a + 1; i < b; ++i) {
      xl = mn(xl, x[i]); xh = mx(xh, x[i]);
      yl = mn(yl, y[i]); yh = mx(yh, y[i]);
      zl = mn(zl, z[i]); zh = mx(zh, z[i]);
    }
    double* bo = box + q * 6;
    bo[0] = xl; bo[1] = xh; bo[2] = yl; bo[3] = yh; bo[4] = zl; bo[5] = zh;
    const double xc = 0.5 * (xl + xh), yc = 0.5 * (yl + yh);
    const double zc = 0.5 * (zl + zh), zr = 0.5 * (zh - zl);
    double m = -INFINITY;
    for (int i = a; i < b; ++i) {
      const double dx = x[i] - xc, dy = y[i] - yc;
      const double s = dx * dx + dy * dy;
      if (s > m) m = s;
    }
    double rho = sqrt(m);
    rho = rho * (1.0 + 1e-12) + 1e-12;
    double* ci = circ + q * 6;
    ci[0] = xc; ci[1] = yc; ci[2] = rho;
    ci[3] = tc * rho + fabs(ts) * (zr * (1.0 + 1e-12) + 1e-12);
    ci[4] = -ts * zc;
    ci[5] = 0.0;
    tbox[0] = mn(tbox[0], xl); tbox[1] = mx(tbox[1], xh);
    tbox[2] = mn(tbox[2], yl); tbox[3] = mx(tbox[3], yh);
    tbox[4] = mn(tbox[4], zl); tbox[5] = mx(tbox[5], zh);
  }
}

}  // namespace

extern "C" {

int msurf_plan_geometry(const msurf_geom_in* in, double* px, double* py, double* pz, double* stats2) {
  if (!in || !px || !py || !pz || in->teeth < 1 || in->points < 2) return 1;
  const int zn = in->teeth, n = in->points;
  const double r = in->radius;
  std::vector<double> ex(n), ez(n), nx(n), nz(n);
  if (in->mode == MSURF_MODE_REF || in->profile == 0) {
    edge_coords(in->half, n, r, ex.data(), ez.data());
    for (int i = 0; i < n; ++i) {
      nx[i] = ex[i] / r;
      nz[i] = -(r - ez[i]) / r;
    }
  } else {
    // ball: kappa_i = (kmax i)/(n-1), last = kmax; n = (sin k, -cos k);
    // e = (r sin k, 0, r - r cos k)
    for (int i = 0; i < n; ++i) {
      const double k = i == n - 1 ? in->kmax : (in->kmax * (double)i) / (double)(n - 1);
      double s, c;
      sincos(k, &s, &c);  // glibc: the same values as sin(k), cos(k) (checked bitwise by the tests)
      nx[i] = s;
      nz[i] = -c;
      ex[i] = r * s;
      ez[i] = r - r * c;
    }
  }
  if (in->mode == MSURF_MODE_REF) {
    // REF: the edge-frame SoA itself (tooth rows are applied on the device)
    for (int i = 0; i < n; ++i) {
      px[i] = ex[i];
      py[i] = 0.0;
      pz[i] = ez[i];
    }
    return 0;
  }
  double zmin_tilt = INFINITY, zmax = 0.0;
  for (int k = 0; k < zn; ++k) {
    const double* e = in->rows + k * 12;
    double* qx = px + (long)k * n;
    double* qy = py + (long)k * n;
    double* qz = pz + (long)k * n;
    const double* dl = in->delta ? in->delta + (long)k * n : nullptr;
    for (int i = 0; i < n; ++i) {
      double x = ex[i], z = ez[i];
      if (dl) {
        x = ex[i] + dl[i] * nx[i];
        z = ez[i] + dl[i] * nz[i];
      }
      const double y = 0.0;
      double ux = ((e[0] * x + e[1] * y) + e[2] * z) + e[3];
      double uy = ((e[4] * x + e[5] * y) + e[6] * z) + e[7];
      const double uz = ((e[8] * x + e[9] * y) + e[10] * z) + e[11];
      if (in->tan_beta_over_r != 0.0) {
        const double psi = z * in->tan_beta_over_r;
        double sps, cps;
        sincos(psi, &sps, &cps);
        const double nxv = cps * ux + sps * uy;
        const double nyv = (-sps) * ux + cps * uy;
        ux = nxv;
        uy = nyv;
      }
      if (in->runout_xy) {
        ux = ux + in->runout_xy[2 * k];
        uy = uy + in->runout_xy[2 * k + 1];
      }
      qx[i] = ux;
      qy[i] = uy;
      qz[i] = uz;
      if (in->mode == MSURF_MODE_EXT_TILT) {
        const double t = in->tilt_c * uz - fabs(in->tilt_s) * sqrt(ux * ux + uy * uy);
        if (t < zmin_tilt) zmin_tilt = t;
      }
      const double az = fabs(uz);
      if (az > zmax) zmax = az;
    }
  }
  if (stats2) {
    stats2[0] = in->mode == MSURF_MODE_EXT_TILT ? -zmin_tilt : 0.0;  // z_shift
    stats2[1] = zmax;                                              // max |zt|
  }
  return 0;
}

int msurf_plan_finish(const msurf_geom_in* in, const double* px, const double* py, const double* pz, double zoff,
                      double* pts, double* tooth_box, double* chunk_circ, double* chunk_box, int32_t* min_index,
                      double* zw_out, uint64_t* key_out) {
  if (!in || !px || !py || !pz || !pts || !tooth_box || !chunk_circ || !chunk_box || !min_index) return 1;
  const int zn = in->teeth, n = in->points;
  const int nchunk = (n + kChunk - 1) / kChunk;
  std::vector<double> zw(n), xt(n), yt(n);
  for (int k = 0; k < zn; ++k) {
    const double* x = in->mode == MSURF_MODE_REF ? px : px + (long)k * n;
    const double* y = in->mode == MSURF_MODE_REF ? py : py + (long)k * n;
    const double* z = in->mode == MSURF_MODE_REF ? pz : pz + (long)k * n;
    double* rec = pts + (long)k * n * 4;
    if (in->mode == MSURF_MODE_REF) {
      // zw = ((e20 x + e21 y) + e22 z) + (e23 + z0); tool-frame x, y for the cull
      const double* e = in->rows + k * 12;
      const double tz = e[11] + in->z0;
      for (int i = 0; i < n; ++i) {
        zw[i] = ((e[8] * x[i] + e[9] * y[i]) + e[10] * z[i]) + tz;
        xt[i] = ((e[0] * x[i] + e[1] * y[i]) + e[2] * z[i]) + e[3];
        yt[i] = ((e[4] * x[i] + e[5] * y[i]) + e[6] * z[i]) + e[7];
      }
    } else {
      for (int i = 0; i < n; ++i) zw[i] = z[i] + zoff;
    }
    int arg = 0;
    for (int i = 1; i < n; ++i)
      if (zw[i] < zw[arg]) arg = i;
    min_index[k] = arg;
    for (int i = 0; i < n; ++i) {
      const uint64_t key = enc_key(zw[i]);
      if (zw_out) zw_out[(long)k * n + i] = zw[i];
      if (key_out) key_out[(long)k * n + i] = key;
      double* r4 = rec + i * 4;
      if (in->mode == MSURF_MODE_REF) {
        r4[0] = x[i]; r4[1] = y[i]; r4[2] = z[i]; r4[3] = key_as_double(key);
      } else if (in->mode == MSURF_MODE_EXT) {
        r4[0] = x[i]; r4[1] = y[i]; r4[2] = key_as_double(key); r4[3] = 0.0;
      } else {
        r4[0] = x[i]; r4[1] = y[i]; r4[2] = in->tilt_s * z[i];
        r4[3] = (in->tilt_c * z[i] + zoff) + 0.0;
      }
    }
    double* cb = chunk_box + (long)k * nchunk * 6;
    double* cc = chunk_circ + (long)k * nchunk * 6;
    double* tb = tooth_box + k * 6;
    if (in->mode == MSURF_MODE_REF) {
      chunk_records(xt.data(), yt.data(), zw.data(), n, 1.0, 0.0, cb, cc, tb);
    } else {
      chunk_records(x, y, z, n, in->tilt_c, in->tilt_s, cb, cc, tb);
    }
  }
  return 0;
}

}  // extern "C"

// ---------------------------------------------------------------- batches
// The same two steps for n parameter sets of one geometry family (equal
// teeth and points): set b reads ins[b] and writes its slice of every output
// (teeth*points, teeth*nchunk*6, ... elements per set). Sets are independent:
// `threads` host threads split them (results do not depend on the split).
#include <unistd.h>

#include <atomic>
#include <condition_variable>
#include <mutex>
#include <thread>

namespace {
// A persistent pool of host workers (created on first use, never joined: the
// process exit ends them), so a 32-set launch group does not pay for thread
// creation on every call. One caller at a time owns the pool; a concurrent
// caller (another planner thread) runs its sets on its own thread instead.
// The split never changes a result: every set is computed by one thread.
struct Pool {
  std::mutex use;  // held by the caller that owns the pool
  std::mutex m;
  std::condition_variable wake, idle;
  std::vector<std::thread> workers;
  const std::function<void(int)>* job = nullptr;
  int n = 0, want = 0, busy = 0;
  std::atomic<int> next{0};
  uint64_t gen = 0;

  explicit Pool(int k) {
    for (int t = 0; t < k; ++t) workers.emplace_back([this] { loop(); });
  }
  void drain() {
    for (int b = next.fetch_add(1); b < n; b = next.fetch_add(1)) (*job)(b);
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      std::unique_lock<std::mutex> lk(m);
      wake.wait(lk, [&] { return gen != seen && want > 0; });
      seen = gen;
      --want;
      ++busy;
      lk.unlock();
      drain();
      lk.lock();
      if (--busy == 0) idle.notify_all();
    }
  }
  // run f(0..n-1) on the caller plus up to `helpers` workers
  void run(int items, int helpers, const std::function<void(int)>& f) {
    {
      std::lock_guard<std::mutex> lk(m);
      job = &f;
      n = items;
      next.store(0);
      want = helpers;
      ++gen;
    }
    wake.notify_all();
    drain();
    std::unique_lock<std::mutex> lk(m);
    want = 0;  // workers that have not started yet stay asleep
    idle.wait(lk, [&] { return busy == 0; });
    job = nullptr;
  }
};

Pool* pool_get() {
  static std::mutex mk;
  static Pool* pool = nullptr;
  static pid_t owner = 0;
  std::lock_guard<std::mutex> lk(mk);
  if (!pool || owner != getpid()) {  // a forked child gets its own (the parent's threads are gone)
    unsigned hw = std::thread::hardware_concurrency();
    int k = hw > 1 ? (int)(hw < 16 ? hw : 16) - 1 : 0;
    pool = new Pool(k);
    owner = getpid();
  }
  return pool;
}

template <class F>
void for_sets(int n, int threads, F&& f) {
  if (threads < 1) threads = 1;
  if (threads > n) threads = n;
  if (threads > 1) {
    Pool* p = pool_get();
    if ((int)p->workers.size() > 0 && p->use.try_lock()) {
      const std::function<void(int)> fn = [&](int b) { f(b); };
      const int helpers = threads - 1 < (int)p->workers.size() ? threads - 1 : (int)p->workers.size();
      p->run(n, helpers, fn);
      p->use.unlock();
      return;
    }
  }
  for (int b = 0; b < n; ++b) f(b);
}
}  // namespace

extern "C" {

int msurf_plan_geometry_many(const msurf_geom_in* ins, int32_t n, double* px, double* py, double* pz,
                             double* stats2, int32_t threads) {
  if (!ins || n < 1) return 1;
  const long per = (long)ins[0].teeth * ins[0].points;
  for (int b = 0; b < n; ++b)
    if (ins[b].teeth != ins[0].teeth || ins[b].points != ins[0].points || ins[b].mode == MSURF_MODE_REF) return 1;
  std::atomic<int> bad{0};
  for_sets(n, threads, [&](int b) {
    if (msurf_plan_geometry(ins + b, px + b * per, py + b * per, pz + b * per, stats2 + 2 * b)) bad = 1;
  });
  return bad.load();
}

int msurf_plan_finish_many(const msurf_geom_in* ins, int32_t n, const double* px, const double* py, const double* pz,
                           const double* zoff, double* pts, double* tooth_box, double* chunk_circ, double* chunk_box,
                           int32_t* min_index, double* zw_out, uint64_t* key_out, int32_t threads) {
  if (!ins || n < 1) return 1;
  const int zn = ins[0].teeth, np = ins[0].points, nchunk = (np + kChunk - 1) / kChunk;
  const long per = (long)zn * np;
  std::atomic<int> bad{0};
  for_sets(n, threads, [&](int b) {
    if (msurf_plan_finish(ins + b, px + b * per, py + b * per, pz + b * per, zoff[b], pts + b * per * 4,
                          tooth_box + (long)b * zn * 6, chunk_circ + (long)b * zn * nchunk * 6,
                          chunk_box + (long)b * zn * nchunk * 6, min_index + (long)b * zn,
                          zw_out ? zw_out + b * per : nullptr, key_out ? key_out + b * per : nullptr))
      bad = 1;
  });
  return bad.load();
}

}  // extern "C"
