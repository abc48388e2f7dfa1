// DVR ray marcher: one thread per pixel ray, index traversal streamed straight into the
// lattice-locked front-to-back integrator.
//
// Reference semantics (paths relative to /root/reference/pkg/src/voxelskip/render.py):
//   Camera.ray_origins :134-149  origin = (eye + ys*up) + xs*right, top row first
//   _ray_setup :273-287, _slab :196-240 (half-open boxes, zero-direction containment)
//   _k_naive :290-302, _dda_runs/_k_grid :305-401, _k_bvh :404-504, _kd_leaves/_k_kd
//   :507-590, _k_hybrid :593-630, _sort_merge :243-270, _k_integrate :633-765,
//   render_frame :869-911 (quantise floor(x*255 + 0.5) clipped).
//
// The reference collects every leaf interval of a ray, sorts and merges them, then
// integrates.  Here the traversals emit intervals already in increasing t (siblings of the
// LBVH and k-d trees are separated by an axis plane and visited near-first; DDA runs are
// monotone), so a one-interval merge window reproduces _sort_merge exactly and the
// integrator consumes intervals as they appear: no per-ray buffers, no overflow re-run.  A
// non-monotone emission (which would make the streaming result differ) raises a flag the
// host turns into an error.
//
// Arithmetic is the reference's: IEEE double, no FMA (the library is built -fmad=false),
// trilinear first-level differences in float32 (numba types f32 - f32 as f32), opacity
// correction 1 - (1 - a)^dt from a host table computed with libm pow (== numba's **).
#include <cfloat>
#include <type_traits>

#include "common.cuh"

// Minimum resident blocks per SM for the two render kernels (register caps; tuned on B200).
#ifndef VS_INTEGRATE_MINB
#define VS_INTEGRATE_MINB 7
#endif
#ifndef VS_SEGMENTS_MINB
#define VS_SEGMENTS_MINB 8
#endif
// Samples the integration loop's gathers run ahead of the shading (1 or 2): two loads in
// flight per warp (rotating slots) take 2-15% off every index kind's frames on the B200; three
// (four slots) spill at the 80-register cap and lose 2-3%.
#ifndef VS_PREFETCH
#define VS_PREFETCH 2
#endif

namespace vs {

constexpr double R_FAR = 1e300;
#ifndef VS_RENDER_TX
#define VS_RENDER_TX 8
#endif
// 128-thread pixel tiles of 8 x 16: a warp covers 8 x 4 pixels (the most coherent ray bundle;
// 16 x 8 tiles measured 2-3% slower, 4 x 32 slower at dense TFs)
constexpr int RENDER_TX = VS_RENDER_TX, RENDER_TY = 128 / VS_RENDER_TX;
constexpr int STACK_CAP = 128;
constexpr int KIND_LBVH_BRICK = 5;  // internal: LBVH leaves by brick DDA

enum RenderFlags { RF_OVERFLOW = 1, RF_ORDER = 2 };

struct Ray {
  double ox, oy, oz, dx, dy, dz, ix, iy, iz;
  bool zx, zy, zz;
};

__device__ __forceinline__ void ray_setup(Ray& r, double ox, double oy, double oz,
                                          const vs_camera_desc& c) {
  r.ox = ox; r.oy = oy; r.oz = oz;
  r.dx = c.dir[0]; r.dy = c.dir[1]; r.dz = c.dir[2];
  r.zx = r.dx == 0.0; r.zy = r.dy == 0.0; r.zz = r.dz == 0.0;
  r.ix = r.zx ? 0.0 : 1.0 / r.dx;
  r.iy = r.zy ? 0.0 : 1.0 / r.dy;
  r.iz = r.zz ? 0.0 : 1.0 / r.dz;
}

// _slab: [l, h) box; returns hit and (t0, t1) with t1 > t0.
__device__ __forceinline__ bool slab(const Ray& r, double lx, double ly, double lz, double hx,
                                     double hy, double hz, double& t0, double& t1) {
  double tmin = -R_FAR, tmax = R_FAR;
  if (r.zx) {
    if (r.ox < lx || r.ox >= hx) return false;
  } else {
    double ta = __dmul_rn(lx - r.ox, r.ix), tb = __dmul_rn(hx - r.ox, r.ix);
    if (ta > tb) { double t = ta; ta = tb; tb = t; }
    if (ta > tmin) tmin = ta;
    if (tb < tmax) tmax = tb;
  }
  if (r.zy) {
    if (r.oy < ly || r.oy >= hy) return false;
  } else {
    double ta = __dmul_rn(ly - r.oy, r.iy), tb = __dmul_rn(hy - r.oy, r.iy);
    if (ta > tb) { double t = ta; ta = tb; tb = t; }
    if (ta > tmin) tmin = ta;
    if (tb < tmax) tmax = tb;
  }
  if (r.zz) {
    if (r.oz < lz || r.oz >= hz) return false;
  } else {
    double ta = __dmul_rn(lz - r.oz, r.iz), tb = __dmul_rn(hz - r.oz, r.iz);
    if (ta > tb) { double t = ta; ta = tb; tb = t; }
    if (ta > tmin) tmin = ta;
    if (tb < tmax) tmax = tb;
  }
  if (tmax <= tmin) return false;
  t0 = tmin;
  t1 = tmax;
  return true;
}

// slab() for a ray with no zero direction component (the branches on r.zx/zy/zz dropped).
__device__ __forceinline__ bool slab_nz(const Ray& r, double lx, double ly, double lz, double hx,
                                        double hy, double hz, double& t0, double& t1) {
  double tmin = -R_FAR, tmax = R_FAR;
  const double o[3] = {r.ox, r.oy, r.oz}, inv[3] = {r.ix, r.iy, r.iz};
  const double l[3] = {lx, ly, lz}, h[3] = {hx, hy, hz};
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    double ta = __dmul_rn(l[a] - o[a], inv[a]), tb = __dmul_rn(h[a] - o[a], inv[a]);
    if (ta > tb) { double t = ta; ta = tb; tb = t; }
    if (ta > tmin) tmin = ta;
    if (tb < tmax) tmax = tb;
  }
  if (tmax <= tmin) return false;
  t0 = tmin;
  t1 = tmax;
  return true;
}

__device__ __forceinline__ bool node_slab(const Ray& r, const int32_t* __restrict__ lo,
                                          const int32_t* __restrict__ hi, int i, double& a,
                                          double& b) {
  const int32_t* l = lo + 3 * i;
  const int32_t* h = hi + 3 * i;
  return slab(r, (double)__ldg(l), (double)__ldg(l + 1), (double)__ldg(l + 2),
              (double)__ldg(h), (double)__ldg(h + 1), (double)__ldg(h + 2), a, b);
}

// Shared per-CTA tables.
struct RenderSmem {
  float4 lut[256];
  double corr[256];
  float u8f[256];
};

// ---- integrator (_k_integrate for one ray), resumable ----------------------------------------
// begin(t0, t1) positions the lattice index k exactly as render.py:664-671; run(S) takes at
// most S samples so the render loop can interleave traversal and sampling across a warp.
struct Integrator {
  const Ray* r;
  const RenderSmem* sm;
  const uint8_t* __restrict__ bins;
  const float* __restrict__ field;  // null: u8 field f32(u/255)
  const uint32_t* __restrict__ quads;  // optional packed (y,z) 2x2 neighbourhoods
  bool idx32, use_tab;
  int nx, ny, nz;
  double entry, dt, inv_dt;
  bool nearest;
  double ert_a;  // early ray termination: stop once acca >= ert_a (2.0 = never: parity mode)
  double accr, accg, accb, acca;
  int taken;  // per-ray lattice samples (< 2^31)
  // active segment
  double t, t1;
  int64_t k;
  bool active;

  // f32(u / 255) exactly (load_raw normalises in float64 then narrows): u/255 in binary is
  // u's 8 bits repeated, so rounding the 64-bit repetition to float and scaling by 2^-64 is
  // the correctly rounded value (checked for all 256 codes) -- no table, no MIO traffic.
  __device__ __forceinline__ static float u8f(uint32_t u) {
    const uint32_t w = u * 0x01010101u;
    const unsigned long long q = ((unsigned long long)w << 32) | w;
    return __fmul_rn(__ull2float_rn(q), __int_as_float(0x1f800000));  // x 2^-64
  }
  __device__ __forceinline__ float fetch(int64_t idx) const {
    if (field) return __ldg(field + idx);
    return u8f(__ldg(bins + idx));
  }

  __device__ __forceinline__ void begin(double t0, double t1_) {
    const int64_t kk = first_k(t0);
    k = kk;
    t = __dadd_rn(entry, __dmul_rn((double)kk, dt));
    t1 = t1_;
    active = t < t1;
  }

  // first lattice index with entry + k*dt >= t0 (render.py:664-671).  The reference's
  // fix-up loops make the result the smallest k >= 0 with t_k >= t0 whatever the initial
  // guess, so the guess uses a multiply by 1/dt instead of the division.
  __device__ __forceinline__ int64_t first_k(double t0) const {
    int64_t kk = (int64_t)ceil(__dmul_rn(t0 - entry, inv_dt));
    if (kk < 0) kk = 0;
    while (kk > 0 && __dadd_rn(entry, __dmul_rn((double)(kk - 1), dt)) >= t0) kk--;
    while (__dadd_rn(entry, __dmul_rn((double)kk, dt)) < t0) kk++;
    return kk;
  }

  __device__ __forceinline__ void sample() {
    sample_at();
    ++k;
    t = __dadd_rn(entry, __dmul_rn((double)k, dt));
  }

  // ---- quad-gather trilinear split in two halves so the next sample's loads can be issued
  // before the current sample's arithmetic (render.py:694-744) ----
  struct Gather {
    uint32_t w0, w1;
    uint32_t fix;  // lazy border fix-ups (bit 0: y0 clamped below, bit 1: z0), see settle()
    double fx, fy, fz;
  };
  __device__ __forceinline__ void gather(double tt, Gather& g) const {
    if (idx32) gather_t<true>(tt, g);
    else gather_t<false>(tt, g);
  }
  // LAZY: leave the clamped-border byte fix-ups to settle(), so the loads can complete while
  // the previous sample is shaded (a fix-up right after the load waits on it even when its
  // predicate is false)
  template <bool IDX32, bool LAZY = false>
  __device__ __forceinline__ void gather_t(double tt, Gather& g) const {
    const double px = __dadd_rn(r->ox, __dmul_rn(tt, r->dx));
    const double py = __dadd_rn(r->oy, __dmul_rn(tt, r->dy));
    const double pz = __dadd_rn(r->oz, __dmul_rn(tt, r->dz));
    const double qx = px - 0.5, qy = py - 0.5, qz = pz - 0.5;
    const double flx = floor(qx), fly = floor(qy), flz = floor(qz);
    g.fx = qx - flx; g.fy = qy - fly; g.fz = qz - flz;
    const int x0r = (int)flx, y0r = (int)fly, z0r = (int)flz;
    const int x0 = min(max(x0r, 0), nx - 1), x1 = min(max(x0r + 1, 0), nx - 1);
    const int y0 = min(max(y0r, 0), ny - 1), z0 = min(max(z0r, 0), nz - 1);
    uint32_t w0, w1;
    {  // the quad volume has < 2^32 words (vs_render rejects larger volumes for it)
      const QuadGeom qg(nx, ny, nz);
      const uint32_t yzw = qg.yz(y0, z0);
      w0 = __ldg(quads + qg.at(x0, yzw));
      w1 = __ldg(quads + qg.at(x1, yzw));
    }
    g.w0 = w0;
    g.w1 = w1;
    g.fix = (y0r < 0 ? 1u : 0u) | (z0r < 0 ? 2u : 0u);
    if (!LAZY) settle(g);
  }
  // clamped low borders: the +1 neighbour is the voxel itself
  __device__ __forceinline__ static void settle(Gather& g) {
    if (g.fix & 1u) { g.w0 = __byte_perm(g.w0, 0, 0x1010); g.w1 = __byte_perm(g.w1, 0, 0x1010); }
    if (g.fix & 2u) { g.w0 = __byte_perm(g.w0, 0, 0x2200); g.w1 = __byte_perm(g.w1, 0, 0x2200); }
  }
  __device__ __forceinline__ double interp(const Gather& g) const {
    if (use_tab) return interp_t<true>(g);
    return interp_t<false>(g);
  }
  template <bool TAB>
  __device__ __forceinline__ double interp_t(const Gather& g) const {
    const uint32_t w0 = g.w0, w1 = g.w1;
    float c000, c001, c010, c011, c100, c101, c110, c111;
    if (TAB) {  // shared-memory table of f32(u/255) (same values, MIO instead of XU)
      const float* tb = sm->u8f;
      c000 = tb[w0 & 0xffu]; c001 = tb[(w0 >> 8) & 0xffu];
      c010 = tb[(w0 >> 16) & 0xffu]; c011 = tb[w0 >> 24];
      c100 = tb[w1 & 0xffu]; c101 = tb[(w1 >> 8) & 0xffu];
      c110 = tb[(w1 >> 16) & 0xffu]; c111 = tb[w1 >> 24];
    } else {
      c000 = u8f(w0 & 0xffu); c001 = u8f((w0 >> 8) & 0xffu);
      c010 = u8f((w0 >> 16) & 0xffu); c011 = u8f(w0 >> 24);
      c100 = u8f(w1 & 0xffu); c101 = u8f((w1 >> 8) & 0xffu);
      c110 = u8f((w1 >> 16) & 0xffu); c111 = u8f(w1 >> 24);
    }
    const float d00 = __fsub_rn(c100, c000), d10 = __fsub_rn(c110, c010);
    const float d01 = __fsub_rn(c101, c001), d11 = __fsub_rn(c111, c011);
    const double c00 = __dadd_rn((double)c000, __dmul_rn((double)d00, g.fx));
    const double c10 = __dadd_rn((double)c010, __dmul_rn((double)d10, g.fx));
    const double c01 = __dadd_rn((double)c001, __dmul_rn((double)d01, g.fx));
    const double c11 = __dadd_rn((double)c011, __dmul_rn((double)d11, g.fx));
    const double c0 = __dadd_rn(c00, __dmul_rn(c10 - c00, g.fy));
    const double c1 = __dadd_rn(c01, __dmul_rn(c11 - c01, g.fy));
    return __dadd_rn(c0, __dmul_rn(c1 - c0, g.fz));
  }
  // the sample's bin by the FP32 filter (common.cuh bin_fast), -1: decide in FP64
  __device__ __forceinline__ int bin_fast(const Gather& g) const {
    return vs::bin_fast(sm->u8f, g.w0, g.w1, __double2float_rn(g.fx), __double2float_rn(g.fy),
                        __double2float_rn(g.fz));
  }
  // floor(v*255 + 0.5) clipped to [0, 255] (render.py:745-748): one floor-converting F2I
  __device__ __forceinline__ static int bin_of(double value) {
    const int bi = __double2int_rd(__dadd_rn(__dmul_rn(value, 255.0), 0.5));
    return bi < 0 ? 0 : (bi > 255 ? 255 : bi);
  }
  // classification + front-to-back compositing of one interpolated value (render.py:745-758)
  __device__ __forceinline__ void shade(double value) { shade_bin(bin_of(value)); }
  __device__ __forceinline__ void shade_bin(int bin) {
    const float4 c = sm->lut[bin];
    if (c.w > 0.0f) {
      const double w = __dmul_rn(1.0 - acca, sm->corr[bin]);
      accr = __dadd_rn(accr, __dmul_rn(w, (double)c.x));
      accg = __dadd_rn(accg, __dmul_rn(w, (double)c.y));
      accb = __dadd_rn(accb, __dmul_rn(w, (double)c.z));
      acca = __dadd_rn(acca, w);
    }
    ++taken;
  }

  // one lattice sample at the current t (no lattice advance)
  __device__ __forceinline__ void sample_at() {
    const int64_t sy = nz, sx = (int64_t)ny * nz;
    const double px = __dadd_rn(r->ox, __dmul_rn(t, r->dx));
    const double py = __dadd_rn(r->oy, __dmul_rn(t, r->dy));
    const double pz = __dadd_rn(r->oz, __dmul_rn(t, r->dz));
    double value;
    if (nearest) {
      int64_t xi = (int64_t)floor(px), yi = (int64_t)floor(py), zi = (int64_t)floor(pz);
      xi = xi < 0 ? 0 : (xi > nx - 1 ? nx - 1 : xi);
      yi = yi < 0 ? 0 : (yi > ny - 1 ? ny - 1 : yi);
      zi = zi < 0 ? 0 : (zi > nz - 1 ? nz - 1 : zi);
      value = (double)fetch(xi * sx + yi * sy + zi);
    } else if (quads) {
      Gather g;
      gather(t, g);
      value = interp(g);
    } else {
      const double qx = px - 0.5, qy = py - 0.5, qz = pz - 0.5;
      int64_t x0 = (int64_t)floor(qx), y0 = (int64_t)floor(qy), z0 = (int64_t)floor(qz);
      const double fx = qx - (double)x0, fy = qy - (double)y0, fz = qz - (double)z0;
      int64_t x1 = x0 + 1, y1 = y0 + 1, z1 = z0 + 1;
      x0 = x0 < 0 ? 0 : (x0 > nx - 1 ? nx - 1 : x0);
      y0 = y0 < 0 ? 0 : (y0 > ny - 1 ? ny - 1 : y0);
      z0 = z0 < 0 ? 0 : (z0 > nz - 1 ? nz - 1 : z0);
      x1 = x1 < 0 ? 0 : (x1 > nx - 1 ? nx - 1 : x1);
      y1 = y1 < 0 ? 0 : (y1 > ny - 1 ? ny - 1 : y1);
      z1 = z1 < 0 ? 0 : (z1 > nz - 1 ? nz - 1 : z1);
      const int64_t b00 = x0 * sx + y0 * sy, b10 = x1 * sx + y0 * sy;
      const int64_t b01 = x0 * sx + y1 * sy, b11 = x1 * sx + y1 * sy;
      const float c000 = fetch(b00 + z0), c100 = fetch(b10 + z0);
      const float c010 = fetch(b01 + z0), c110 = fetch(b11 + z0);
      const float c001 = fetch(b00 + z1), c101 = fetch(b10 + z1);
      const float c011 = fetch(b01 + z1), c111 = fetch(b11 + z1);
      const float d00 = __fsub_rn(c100, c000), d10 = __fsub_rn(c110, c010);
      const float d01 = __fsub_rn(c101, c001), d11 = __fsub_rn(c111, c011);
      const double c00 = __dadd_rn((double)c000, __dmul_rn((double)d00, fx));
      const double c10 = __dadd_rn((double)c010, __dmul_rn((double)d10, fx));
      const double c01 = __dadd_rn((double)c001, __dmul_rn((double)d01, fx));
      const double c11 = __dadd_rn((double)c011, __dmul_rn((double)d11, fx));
      const double c0 = __dadd_rn(c00, __dmul_rn(c10 - c00, fy));
      const double c1 = __dadd_rn(c01, __dmul_rn(c11 - c01, fy));
      value = __dadd_rn(c0, __dmul_rn(c1 - c0, fz));
    }
    shade(value);
  }

  __device__ __forceinline__ void run(int smax) {
    for (int q = 0; q < smax && t < t1 && acca < ert_a; ++q) sample();
    active = t < t1 && acca < ert_a;
  }

  __device__ __forceinline__ void segment(double t0, double t1_) {  // whole segment at once
    begin(t0, t1_);
    while (t < t1 && acca < ert_a) sample();
    active = false;
  }
  __device__ __forceinline__ bool terminated() const { return acca >= ert_a; }
};

// ---- interval generators -----------------------------------------------------------------
// next(a, b, budget): 1 = produced [a, b), 0 = exhausted, 2 = budget (traversal steps) spent.

// Single interval (_k_naive).
struct NaiveGen {
  double a, b;
  bool done;
  __device__ __forceinline__ int next(double& x, double& y, int&) {
    if (done) return 0;
    done = true;
    x = a; y = b;
    return 1;
  }
};

// _dda_runs (render.py:305-378) over [t_in, t_out), resumable.
struct GridDDA {
  const uint8_t* __restrict__ occ;
  int ncx, ncy, ncz;
  double cs, t_out, run_t0, tcur, tnx, tny, tnz;
  int64_t cx, cy, cz, step, max_steps;
  int sx, sy, sz;
  bool open_run, done, fin;

  __device__ __forceinline__ double cross(int64_t c, int s, double o, double inv) const {
    return __dmul_rn(__dmul_rn((double)(c + (s > 0)), cs) - o, inv);
  }
  __device__ void init(const Ray& r, const vs_index_desc& ix, double t_in, double t_out_) {
    occ = ix.occ;
    ncx = ix.ncx; ncy = ix.ncy; ncz = ix.ncz;
    cs = (double)ix.cs;
    t_out = t_out_;
    const double px = __dadd_rn(r.ox, __dmul_rn(t_in, r.dx));
    const double py = __dadd_rn(r.oy, __dmul_rn(t_in, r.dy));
    const double pz = __dadd_rn(r.oz, __dmul_rn(t_in, r.dz));
    cx = (int64_t)floor(__ddiv_rn(px, cs));
    cy = (int64_t)floor(__ddiv_rn(py, cs));
    cz = (int64_t)floor(__ddiv_rn(pz, cs));
    cx = cx < 0 ? 0 : (cx > ncx - 1 ? ncx - 1 : cx);
    cy = cy < 0 ? 0 : (cy > ncy - 1 ? ncy - 1 : cy);
    cz = cz < 0 ? 0 : (cz > ncz - 1 ? ncz - 1 : cz);
    sx = r.zx ? 0 : (r.ix > 0.0 ? 1 : -1);
    sy = r.zy ? 0 : (r.iy > 0.0 ? 1 : -1);
    sz = r.zz ? 0 : (r.iz > 0.0 ? 1 : -1);
    tnx = sx == 0 ? R_FAR : cross(cx, sx, r.ox, r.ix);
    tny = sy == 0 ? R_FAR : cross(cy, sy, r.oy, r.iy);
    tnz = sz == 0 ? R_FAR : cross(cz, sz, r.oz, r.iz);
    open_run = false;
    run_t0 = 0.0;
    tcur = t_in;
    step = 0;
    max_steps = (int64_t)ncx + ncy + ncz + 3;
    done = false;
    fin = false;
  }
  __device__ __forceinline__ int next(const Ray& r, double& x, double& y, int& budget) {
    while (!done) {
      if (budget <= 0) return 2;
      --budget;
      if (step >= max_steps) { done = true; break; }
      double tn = tnx;
      if (tny < tn) tn = tny;
      if (tnz < tn) tn = tnz;
      bool emit = false;
      if (__ldg(occ + (cx * ncy + cy) * ncz + cz)) {
        if (!open_run) { open_run = true; run_t0 = tcur; }
      } else if (open_run) {
        x = run_t0; y = tcur; open_run = false; emit = true;
      }
      ++step;
      if (tn >= t_out) {
        done = true;
      } else {
        if (tnx == tn) { cx += sx; tnx = cross(cx, sx, r.ox, r.ix); }
        if (tny == tn) { cy += sy; tny = cross(cy, sy, r.oy, r.iy); }
        if (tnz == tn) { cz += sz; tnz = cross(cz, sz, r.oz, r.iz); }
        tcur = tn;
        if (cx < 0 || cy < 0 || cz < 0 || cx >= ncx || cy >= ncy || cz >= ncz) done = true;
      }
      if (emit) return 1;
    }
    if (!fin) {
      fin = true;
      if (open_run) { open_run = false; x = run_t0; y = t_out; return 1; }
    }
    return 0;
  }
};

// LBVH leaves without walking the tree.  A leaf's interval is reported by _k_bvh iff its own
// slab interval clipped to [tmin, tmax] is non-empty (ancestor boxes contain it and slab
// intervals are monotone in the box bounds, in floating point too), so the merged union equals
// the merged union of every occupied brick's clipped slab interval.  A 3-D DDA over the brick
// grid visits exactly the bricks whose interval along the ray is non-empty, in increasing t:
// its per-axis crossings are the same expressions slab() evaluates for a brick's faces, and
// simultaneous crossings skip only bricks touched in a single point.  The start brick is the
// one whose per-axis crossing window contains tmin.  Each occupied brick then gets the
// reference's exact clipped slab interval (box hi clipped to dims).
struct BrickDDA {
  const uint32_t* __restrict__ bits;
  int nb[3], dims[3], bs;
  int c[3], s[3];
  double tn[3], tmin, tmax;
  int64_t step, maxsteps;
  bool done;

  __device__ __forceinline__ double plane_t(const Ray& r, int a, int k) const {
    const double o = a == 0 ? r.ox : (a == 1 ? r.oy : r.oz);
    const double inv = a == 0 ? r.ix : (a == 1 ? r.iy : r.iz);
    return __dmul_rn((double)(k * bs) - o, inv);
  }
  __device__ void init(const Ray& r, const vs_index_desc& ix, int nx, int ny, int nz,
                       double tmin_, double tmax_, bool nonempty) {
    bits = ix.brick_bits;
    bs = ix.bs;
    nb[0] = ix.nbx; nb[1] = ix.nby; nb[2] = ix.nbz;
    dims[0] = nx; dims[1] = ny; dims[2] = nz;
    tmin = tmin_; tmax = tmax_;
    done = !nonempty;
    step = 0;
    maxsteps = (int64_t)nb[0] + nb[1] + nb[2] + 3;
    const double cs = (double)bs;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const double o = a == 0 ? r.ox : (a == 1 ? r.oy : r.oz);
      const double d = a == 0 ? r.dx : (a == 1 ? r.dy : r.dz);
      const double inv = a == 0 ? r.ix : (a == 1 ? r.iy : r.iz);
      const bool zero = a == 0 ? r.zx : (a == 1 ? r.zy : r.zz);
      s[a] = zero ? 0 : (inv > 0.0 ? 1 : -1);
      const double p = __dadd_rn(o, __dmul_rn(tmin, d));
      int ca = (int)floor(__ddiv_rn(p, cs));
      ca = ca < 0 ? 0 : (ca > nb[a] - 1 ? nb[a] - 1 : ca);
      if (s[a] > 0) {
        while (ca > 0 && plane_t(r, a, ca) > tmin) --ca;
        while (ca + 1 < nb[a] && plane_t(r, a, ca + 1) <= tmin) ++ca;
        tn[a] = plane_t(r, a, ca + 1);
      } else if (s[a] < 0) {
        while (ca + 1 < nb[a] && plane_t(r, a, ca + 1) > tmin) ++ca;
        while (ca > 0 && plane_t(r, a, ca) <= tmin) --ca;
        tn[a] = plane_t(r, a, ca);
      } else {
        ca = (int)floor(__ddiv_rn(o, cs));
        if (ca < 0 || ca >= nb[a]) done = true;
        tn[a] = R_FAR;
      }
      c[a] = ca;
    }
  }
  __device__ __forceinline__ int next(const Ray& r, double& x, double& y, int& budget) {
    while (!done) {
      if (budget <= 0) return 2;
      --budget;
      if (step++ >= maxsteps) { done = true; break; }
      const int64_t lin = ((int64_t)c[0] * nb[1] + c[1]) * nb[2] + c[2];
      bool emit = false;
      if ((__ldg(bits + (lin >> 5)) >> (lin & 31)) & 1u) {
        double a, b;
        const int l0 = c[0] * bs, l1 = c[1] * bs, l2 = c[2] * bs;
        if (slab(r, (double)l0, (double)l1, (double)l2, (double)min(l0 + bs, dims[0]),
                 (double)min(l1 + bs, dims[1]), (double)min(l2 + bs, dims[2]), a, b)) {
          a = a > tmin ? a : tmin;
          b = b < tmax ? b : tmax;
          if (b > a) { x = a; y = b; emit = true; }
        }
      }
      double tt = tn[0];
      if (tn[1] < tt) tt = tn[1];
      if (tn[2] < tt) tt = tn[2];
      if (tt >= tmax) {
        done = true;
      } else {
#pragma unroll
        for (int a2 = 0; a2 < 3; ++a2) {
          if (tn[a2] == tt) {
            c[a2] += s[a2];
            if (c[a2] < 0 || c[a2] >= nb[a2]) done = true;
            tn[a2] = plane_t(r, a2, c[a2] + (s[a2] > 0));
          }
        }
      }
      if (emit) return 1;
    }
    return 0;
  }
};

// _k_bvh leaf intervals, near-first DFS; the stack holds node ids (a popped node's clipped
// interval is recomputed: same inputs, same doubles).
struct BvhWalk {
  const int32_t *lo, *hi, *left, *right;
  double tmin, tmax;
  int sp;
  int stk[STACK_CAP];

  __device__ void init(const Ray& r, const vs_index_desc& ix, int root, double tmin_,
                       double tmax_) {
    lo = ix.lo; hi = ix.hi; left = ix.left; right = ix.right;
    tmin = tmin_; tmax = tmax_;
    sp = 0;
    double a, b;
    if (root >= 0 && node_slab(r, lo, hi, root, a, b)) {
      a = a > tmin ? a : tmin;
      b = b < tmax ? b : tmax;
      if (b > a) stk[sp++] = root;
    }
  }
  __device__ __forceinline__ int next(const Ray& r, double& x, double& y, int& budget, int* flags) {
    while (sp > 0) {
      if (budget <= 0) return 2;
      --budget;
      const int i = stk[--sp];
      const int li = __ldg(left + i);
      double a, b;
      if (li < 0) {
        node_slab(r, lo, hi, i, a, b);
        x = a > tmin ? a : tmin;
        y = b < tmax ? b : tmax;
        return 1;
      }
      const int ri = __ldg(right + i);
      double la, lb, ra, rb;
      bool hl = node_slab(r, lo, hi, li, la, lb);
      if (hl) { la = la > tmin ? la : tmin; lb = lb < tmax ? lb : tmax; if (lb <= la) hl = false; }
      bool hr = node_slab(r, lo, hi, ri, ra, rb);
      if (hr) { ra = ra > tmin ? ra : tmin; rb = rb < tmax ? rb : tmax; if (rb <= ra) hr = false; }
      if (sp + 2 > STACK_CAP) { *flags |= RF_OVERFLOW; sp = 0; return 0; }
      if (hl && hr) {
        if (la <= ra) { stk[sp++] = ri; stk[sp++] = li; }
        else { stk[sp++] = li; stk[sp++] = ri; }
      } else if (hl) {
        stk[sp++] = li;
      } else if (hr) {
        stk[sp++] = ri;
      }
    }
    return 0;
  }
};

// _kd_leaves: pop, slab-test clipped to [tmin, tmax], leaf -> interval, inner -> far, near.
struct KdWalk {
  const int32_t *lo, *hi, *left, *right, *plane;
  const int8_t* axis;
  double tmin, tmax;
  int sp;
  int stk[STACK_CAP];

  __device__ void init(const vs_index_desc& ix, double tmin_, double tmax_) {
    lo = ix.lo; hi = ix.hi; left = ix.left; right = ix.right; plane = ix.plane; axis = ix.axis;
    tmin = tmin_; tmax = tmax_;
    sp = 0;
    if (ix.root >= 0) stk[sp++] = ix.root;
  }
  __device__ __forceinline__ int next(const Ray& r, double& x, double& y, int& budget, int* flags) {
    while (sp > 0) {
      if (budget <= 0) return 2;
      --budget;
      const int i = stk[--sp];
      double a, b;
      if (!node_slab(r, lo, hi, i, a, b)) continue;
      a = a > tmin ? a : tmin;
      b = b < tmax ? b : tmax;
      if (b <= a) continue;
      const int ax = __ldg(axis + i);
      if (ax < 0) { x = a; y = b; return 1; }
      const double pl = (double)__ldg(plane + i);
      bool front_left;
      const bool zero = ax == 0 ? r.zx : (ax == 1 ? r.zy : r.zz);
      if (zero)
        front_left = (ax == 0 ? r.ox : (ax == 1 ? r.oy : r.oz)) < pl;
      else
        front_left = (ax == 0 ? r.ix : (ax == 1 ? r.iy : r.iz)) > 0.0;
      const int lc = __ldg(left + i), rc = __ldg(right + i);
      const int nr = front_left ? lc : rc, fr = front_left ? rc : lc;
      if (sp + 2 > STACK_CAP) { *flags |= RF_OVERFLOW; sp = 0; return 0; }
      if (fr >= 0) stk[sp++] = fr;
      if (nr >= 0) stk[sp++] = nr;
    }
    return 0;
  }
};

// One-interval merge window over a t-sorted raw stream (= _sort_merge): drop t1 <= t0, merge
// when t0 <= previous t1.  Produces merged segments.
struct MergeState {
  double a, b, last_t0;
  bool open, src_done;
  __device__ __forceinline__ void init() { open = false; src_done = false; last_t0 = -DBL_MAX; a = b = 0.0; }
  // feed one raw interval; returns true and (x, y) when a merged segment is complete
  __device__ __forceinline__ bool feed(double t0, double t1, double& x, double& y, int* flags) {
    if (t0 < last_t0) *flags |= RF_ORDER;
    last_t0 = t0;
    if (t1 <= t0) return false;
    if (open && t0 <= b) {
      if (t1 > b) b = t1;
      return false;
    }
    const bool out = open;
    if (out) { x = a; y = b; }
    a = t0; b = t1; open = true;
    return out;
  }
  __device__ __forceinline__ bool drain(double& x, double& y) {
    if (!open) return false;
    open = false;
    x = a; y = b;
    return true;
  }
};

struct NoGen {};

// Per-kind source of merged segments (members only for the kinds that use them, so the
// brick-DDA path carries no traversal stack).
template <int KIND>
struct SegmentSource {
  typename std::conditional<KIND == VS_KIND_NAIVE, NaiveGen, NoGen>::type naive;
  typename std::conditional<KIND == VS_KIND_GRID || KIND == VS_KIND_HYBRID, GridDDA, NoGen>::type grid;
  typename std::conditional<KIND == KIND_LBVH_BRICK, BrickDDA, NoGen>::type brick;
  typename std::conditional<KIND == VS_KIND_LBVH, BvhWalk, NoGen>::type bvh;
  typename std::conditional<KIND == VS_KIND_KD || KIND == VS_KIND_HYBRID, KdWalk, NoGen>::type kd;
  MergeState m, leaves;
  bool inner_active;

  __device__ void init(const Ray& r, const vs_index_desc& ix, int nx, int ny, int nz, double tmin,
                       double tmax) {
    m.init();
    if constexpr (KIND == VS_KIND_NAIVE) {
      naive.a = tmin; naive.b = tmax; naive.done = false;
    } else if constexpr (KIND == VS_KIND_GRID) {
      grid.init(r, ix, tmin, tmax);
    } else if constexpr (KIND == KIND_LBVH_BRICK) {
      const int n = ix.lbvh_info ? __ldg(ix.lbvh_info) : ix.root + 1;
      brick.init(r, ix, nx, ny, nz, tmin, tmax, n > 0);
    } else if constexpr (KIND == VS_KIND_LBVH) {
      const int n = ix.lbvh_info ? __ldg(ix.lbvh_info) : ix.root + 1;
      bvh.init(r, ix, n > 0 ? 0 : -1, tmin, tmax);
    } else {
      kd.init(ix, tmin, tmax);
      if constexpr (KIND == VS_KIND_HYBRID) { leaves.init(); inner_active = false; }
    }
  }

  // raw intervals of the kind (before the final merge); 1 / 0 / 2 as the generators
  __device__ __forceinline__ int raw(const Ray& r, const vs_index_desc& ix, double& x, double& y,
                                     int& budget, int* flags) {
    if constexpr (KIND == VS_KIND_NAIVE) {
      return naive.next(x, y, budget);
    } else if constexpr (KIND == VS_KIND_GRID) {
      return grid.next(r, x, y, budget);
    } else if constexpr (KIND == KIND_LBVH_BRICK) {
      return brick.next(r, x, y, budget);
    } else if constexpr (KIND == VS_KIND_LBVH) {
      return bvh.next(r, x, y, budget, flags);
    } else if constexpr (KIND == VS_KIND_KD) {
      return kd.next(r, x, y, budget, flags);
    } else {
    // hybrid: merged k-d leaf intervals, each walked by the grid DDA
    while (true) {
      if (inner_active) {
        const int g = grid.next(r, x, y, budget);
        if (g != 0) return g;
        inner_active = false;
      }
      double la, lb;
      bool got = false;
      while (!got) {
        if (leaves.src_done) {
          if (!leaves.drain(la, lb)) return 0;
          got = true;
          break;
        }
        double ka, kb;
        const int k = kd.next(r, ka, kb, budget, flags);
        if (k == 2) return 2;
        if (k == 0) { leaves.src_done = true; continue; }
        got = leaves.feed(ka, kb, la, lb, flags);
      }
      grid.init(r, ix, la, lb);
      inner_active = true;
    }
    }
  }

  // next merged segment: 1 = (x, y), 0 = exhausted, 2 = budget spent
  __device__ __forceinline__ int next(const Ray& r, const vs_index_desc& ix, double& x, double& y,
                                      int& budget, int* flags) {
    while (true) {
      if (m.src_done) return m.drain(x, y) ? 1 : 0;
      double a, b;
      const int k = raw(r, ix, a, b, budget, flags);
      if (k == 2) return 2;
      if (k == 0) { m.src_done = true; continue; }
      if (m.feed(a, b, x, y, flags)) return 1;
    }
  }
};

// Per-call renderer configuration, resolved from the caller's vs_render_opts (no global or
// thread-local state: concurrent callers on other threads / streams never see each other's
// settings).
//   opts bit0: u8 -> f32 by shared-memory table (else the exact 64-bit integer-to-float path)
//   opts bit1: k_integrate_segments evaluates every sample's bin in FP64 (no FP32 bin filter)
//   opts bit2: generic k_segments for the LBVH brick DDA / grid / hybrid / k-d (else flat loops)
//   opts bit4: k_segments_brick evaluates every occupied brick's slab (no run shortcut)
struct RenderCfg {
  int opts = VS_RO_DEFAULT;
  int trav_budget = 1, sample_budget = 1;  // while-while turn sizes of the generic kernels
  double ert_a = 2.0;                      // early ray termination threshold, 2.0 = off
  void* seg_ws = nullptr;                  // two-phase workspace (segments + counts)
  int seg_cap = 0;
};

static RenderCfg render_cfg(const vs_render_opts* o) {
  RenderCfg c;
  if (!o) return c;
  c.opts = o->flags;
  c.trav_budget = o->trav_steps > 0 ? o->trav_steps : (1 << 30);
  c.sample_budget = o->sample_steps > 0 ? o->sample_steps : (1 << 30);
  c.ert_a = o->ert_eps > 0.0 ? 1.0 - o->ert_eps : 2.0;
  return c;
}

template <int KIND>
__global__ void __launch_bounds__(RENDER_TX* RENDER_TY)
    k_render(vs_volume_desc vol, vs_index_desc ix, vs_camera_desc cam, const float* __restrict__ lut,
             const double* __restrict__ corr, double dt, int nearest, vs_rows_desc rows,
             uint8_t* __restrict__ rgba8, double* __restrict__ rgba64, int32_t* __restrict__ samples,
             unsigned long long* __restrict__ total, int* __restrict__ flags_out, int trav_budget,
             int sample_budget, int render_opts, double ert_a) {
  __shared__ RenderSmem sm;
  const int tid = threadIdx.y * RENDER_TX + threadIdx.x;
  for (int k = tid; k < 256; k += RENDER_TX * RENDER_TY) {
    sm.lut[k] = make_float4(lut[4 * k], lut[4 * k + 1], lut[4 * k + 2], lut[4 * k + 3]);
    sm.corr[k] = corr[k];
    sm.u8f[k] = (float)((double)k / 255.0);
  }
  __syncthreads();
  const int i = blockIdx.x * RENDER_TX + threadIdx.x;  // pixel column
  const int l = blockIdx.y * RENDER_TY + threadIdx.y;  // local row
  int64_t taken = 0;
  int flags = 0;
  if (i < cam.width && l < rows.nrows) {
    // local row -> image row: stripes of rows.stripe rows dealt round-robin over rows.nparts
    const int s = l / rows.stripe, w = l % rows.stripe;
    const int j = (s * rows.nparts + rows.part) * rows.stripe + w;
    const double xs = __dmul_rn(((double)i + 0.5) - (double)cam.width / 2.0, cam.scale);
    const double ys = __dmul_rn(((double)cam.height / 2.0 - (double)j) - 0.5, cam.scale);
    const double ox = __dadd_rn(__dadd_rn(cam.eye[0], __dmul_rn(ys, cam.up[0])), __dmul_rn(xs, cam.right[0]));
    const double oy = __dadd_rn(__dadd_rn(cam.eye[1], __dmul_rn(ys, cam.up[1])), __dmul_rn(xs, cam.right[1]));
    const double oz = __dadd_rn(__dadd_rn(cam.eye[2], __dmul_rn(ys, cam.up[2])), __dmul_rn(xs, cam.right[2]));
    Ray r;
    ray_setup(r, ox, oy, oz, cam);
    Integrator I;
    I.r = &r; I.sm = &sm; I.bins = vol.bins; I.field = vol.field;
    I.quads = vol.field ? nullptr : vol.quads;
    I.idx32 = (int64_t)vol.nx * vol.ny * vol.nz < (1LL << 32);
    I.use_tab = (render_opts & 1) != 0;
    I.nx = vol.nx; I.ny = vol.ny; I.nz = vol.nz; I.dt = dt; I.inv_dt = 1.0 / dt; I.nearest = nearest != 0;
    I.ert_a = ert_a;
    I.accr = I.accg = I.accb = I.acca = 0.0;
    I.taken = 0;
    I.active = false;
    double tmin, tmax;
    if (slab(r, 0.0, 0.0, 0.0, (double)vol.nx, (double)vol.ny, (double)vol.nz, tmin, tmax)) {
      I.entry = tmin;  // _k_integrate's own slab of the full volume gives the same entry
      SegmentSource<KIND> src;
      src.init(r, ix, vol.nx, vol.ny, vol.nz, tmin, tmax);
      // while-while: each turn does a bounded amount of traversal (lanes without a segment)
      // and a bounded number of samples (lanes with one), so lanes in the same phase share
      // instructions instead of serialising whole traversals against whole sample loops.
      while (!I.terminated()) {
        if (!I.active) {
          int budget = trav_budget;
          double a, b;
          const int g = src.next(r, ix, a, b, budget, &flags);
          if (g == 0) break;
          if (g == 1) I.begin(a, b);
        }
        if (I.active) I.run(sample_budget);
      }
    }
    taken = I.taken;
    const int64_t pix = (int64_t)l * cam.width + i;
    const double acc[4] = {I.accr, I.accg, I.accb, I.acca};
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const double q = floor(__dadd_rn(__dmul_rn(acc[c], 255.0), 0.5));
      rgba8[4 * pix + c] = (uint8_t)(q < 0.0 ? 0 : (q > 255.0 ? 255 : (int)q));
      if (rgba64) rgba64[4 * pix + c] = acc[c];
    }
    if (samples) samples[pix] = (int32_t)taken;
  }
  if (flags) atomicOr(flags_out, flags);
  if (total) {  // warp-level: no block barrier behind the slowest warp of the tile
    unsigned long long t = (unsigned long long)taken;
    for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if ((tid & 31) == 0 && t) atomicAdd(total, t);
  }
}

// ---- two-phase render: traversal kernel writes each ray's merged segments, the integration
// kernel consumes them (no traversal/sampling divergence inside one warp).  Rays with more
// than `cap` segments are re-traversed by the fused path inside the integration kernel.
__device__ __forceinline__ void pixel_ray(const vs_camera_desc& cam, const vs_rows_desc& rows,
                                          int i, int l, Ray& r) {
  const int s = l / rows.stripe, w = l % rows.stripe;
  const int j = (s * rows.nparts + rows.part) * rows.stripe + w;
  const double xs = __dmul_rn(((double)i + 0.5) - (double)cam.width / 2.0, cam.scale);
  const double ys = __dmul_rn(((double)cam.height / 2.0 - (double)j) - 0.5, cam.scale);
  const double ox = __dadd_rn(__dadd_rn(cam.eye[0], __dmul_rn(ys, cam.up[0])), __dmul_rn(xs, cam.right[0]));
  const double oy = __dadd_rn(__dadd_rn(cam.eye[1], __dmul_rn(ys, cam.up[1])), __dmul_rn(xs, cam.right[1]));
  const double oz = __dadd_rn(__dadd_rn(cam.eye[2], __dmul_rn(ys, cam.up[2])), __dmul_rn(xs, cam.right[2]));
  ray_setup(r, ox, oy, oz, cam);
}

template <int KIND>
__global__ void __launch_bounds__(RENDER_TX* RENDER_TY, VS_SEGMENTS_MINB)
    k_segments(vs_volume_desc vol, vs_index_desc ix, vs_camera_desc cam, vs_rows_desc rows,
               double dt, int2* __restrict__ segs, int* __restrict__ counts, int cap,
               int* __restrict__ flags_out, int step_budget) {
  const int i = blockIdx.x * RENDER_TX + threadIdx.x;
  const int l = blockIdx.y * RENDER_TY + threadIdx.y;
  if (i >= cam.width || l >= rows.nrows) return;
  const int64_t pix = (int64_t)l * cam.width + i;
  const int64_t npix = (int64_t)rows.nrows * cam.width;
  Ray r;
  pixel_ray(cam, rows, i, l, r);
  int n = 0, flags = 0;
  double tmin, tmax;
  if (slab(r, 0.0, 0.0, 0.0, (double)vol.nx, (double)vol.ny, (double)vol.nz, tmin, tmax)) {
    SegmentSource<KIND> src;
    src.init(r, ix, vol.nx, vol.ny, vol.nz, tmin, tmax);
    Integrator L;  // lattice only: k ranges of the merged segments
    L.entry = tmin;
    L.dt = dt;
    L.inv_dt = 1.0 / dt;
    int kprev = -1;
    while (true) {
      // a bounded number of traversal steps per turn keeps the warp's lanes in one flat loop
      int budget = step_budget;
      double a, b;
      const int g = src.next(r, ix, a, b, budget, &flags);
      if (g == 0) break;
      if (g == 2) continue;
      // samples of [a, b) are lattice indices [first_k(a), first_k(b)); ranges are disjoint
      // and increasing, so abutting ones are joined
      const int k0 = (int)L.first_k(a), k1 = (int)L.first_k(b);
      if (k1 <= k0) continue;
      if (n > 0 && k0 == kprev && n <= cap) {
        segs[(int64_t)(n - 1) * npix + pix].y = k1;
      } else {
        if (n < cap) segs[(int64_t)n * npix + pix] = make_int2(k0, k1);
        ++n;
      }
      kprev = k1;
    }
  }
  counts[pix] = n;
  if (flags) atomicOr(flags_out, flags);
}

// k_segments specialised for the LBVH brick DDA: the same DDA steps (BrickDDA::init/next),
// interval merge (_sort_merge via MergeState) and lattice-range emission as the generic
// kernel, written as one flat loop of one DDA step per turn with 32-bit brick indices and no
// generator/budget plumbing between the step and the merge.  SGN >= 0: the (frame-uniform,
// orthographic) ray direction has no zero component and bit a of SGN is the sign of axis a, so
// the per-step sign bookkeeping and slab()'s zero-direction branches compile away; SGN = -1 is
// the general kernel.
template <int SGN>
__global__ void __launch_bounds__(RENDER_TX* RENDER_TY, VS_SEGMENTS_MINB)
    k_segments_brick(vs_volume_desc vol, vs_index_desc ix, vs_camera_desc cam, vs_rows_desc rows,
                     double dt, int2* __restrict__ segs, int* __restrict__ counts, int cap,
                     int* __restrict__ flags_out, int exact_runs) {
  const int i = blockIdx.x * RENDER_TX + threadIdx.x;
  const int l = blockIdx.y * RENDER_TY + threadIdx.y;
  if (i >= cam.width || l >= rows.nrows) return;
  const int64_t pix = (int64_t)l * cam.width + i;
  const int64_t npix = (int64_t)rows.nrows * cam.width;
  Ray r;
  pixel_ray(cam, rows, i, l, r);
  int n = 0, flags = 0;
  double tmin, tmax;
  if (slab(r, 0.0, 0.0, 0.0, (double)vol.nx, (double)vol.ny, (double)vol.nz, tmin, tmax)) {
    const int nb_bricks = ix.lbvh_info ? __ldg(ix.lbvh_info) : ix.root + 1;
    BrickDDA D;
    D.init(r, ix, vol.nx, vol.ny, vol.nz, tmin, tmax, nb_bricks > 0);
    Integrator L;  // lattice only
    L.entry = tmin;
    L.dt = dt;
    L.inv_dt = 1.0 / dt;
    const int bs = D.bs, nby = D.nb[1], nbz = D.nb[2];
    const uint32_t* __restrict__ bits = D.bits;
    int steps = 0;
    const int maxsteps = D.nb[0] + D.nb[1] + D.nb[2] + 3;
    // merge state (MergeState): open interval [ma, mb)
    bool open = false;
    double ma = 0.0, mb = 0.0, last_t0 = -DBL_MAX;
    int kprev = -1;
    auto emit = [&](double a, double b) {
      const int k0 = (int)L.first_k(a), k1 = (int)L.first_k(b);
      if (k1 <= k0) return;
      if (n > 0 && k0 == kprev && n <= cap) {
        segs[(int64_t)(n - 1) * npix + pix].y = k1;
      } else {
        if (n < cap) segs[(int64_t)n * npix + pix] = make_int2(k0, k1);
        ++n;
      }
      kprev = k1;
    };
    bool done = D.done;
    // Run shortcut: inside a run of occupied interior bricks (box hi not clipped to dims) a
    // brick's clipped slab interval is [previous crossing, next crossing] -- slab() evaluates
    // the very plane expressions the DDA's crossings use -- so the merged run just extends to
    // min(next crossing, tmax) and the brick's slab() is skipped (exact_runs: always slab()).
    bool live = false;
    // "interior" (box not clipped to dims) <=> c <= dims / bs - 1 per axis: limits from the
    // kernel parameters (uniform), so no per-step multiplies
    const int ci0 = vol.nx / ix.bs - 1, ci1 = vol.ny / ix.bs - 1, ci2 = vol.nz / ix.bs - 1;
    while (!done) {
      // (a step advances at least one axis by one brick, so with every direction component
      // nonzero the walk leaves the grid within sum(nb) steps: the guard is for SGN = -1)
      if constexpr (SGN < 0) {
        if (steps++ >= maxsteps) break;
      }
      const int lin = (D.c[0] * nby + D.c[1]) * nbz + D.c[2];
      const bool occ = (__ldg(bits + (lin >> 5)) >> (lin & 31)) & 1u;
      const bool interior = D.c[0] <= ci0 && D.c[1] <= ci1 && D.c[2] <= ci2;
      const bool shortcut = occ && live && interior && !exact_runs;
      if (occ && !shortcut) {
        double a, b;
        const int l0 = D.c[0] * bs, l1 = D.c[1] * bs, l2 = D.c[2] * bs;
        const double h0 = (double)min(l0 + bs, D.dims[0]), h1 = (double)min(l1 + bs, D.dims[1]),
                     h2 = (double)min(l2 + bs, D.dims[2]);
        if (SGN >= 0 ? slab_nz(r, (double)l0, (double)l1, (double)l2, h0, h1, h2, a, b)
                     : slab(r, (double)l0, (double)l1, (double)l2, h0, h1, h2, a, b)) {
          a = a > tmin ? a : tmin;
          b = b < tmax ? b : tmax;
          if (b > a) {
            if (a < last_t0) flags |= RF_ORDER;
            last_t0 = a;
            if (open && a <= mb) {
              if (b > mb) mb = b;
            } else {
              if (open) emit(ma, mb);
              ma = a;
              mb = b;
              open = true;
            }
          }
        }
      }
      double tt = D.tn[0];
      if (D.tn[1] < tt) tt = D.tn[1];
      if (D.tn[2] < tt) tt = D.tn[2];
      if (shortcut) mb = tt < tmax ? tt : tmax;
      live = occ && interior && open && mb == tt;
      if (tt >= tmax) break;
#pragma unroll
      for (int a2 = 0; a2 < 3; ++a2) {
        if (D.tn[a2] == tt) {
          if constexpr (SGN >= 0) {
            const int sg = ((SGN >> a2) & 1) ? 1 : -1;
            D.c[a2] += sg;
            if (sg > 0 ? D.c[a2] >= D.nb[a2] : D.c[a2] < 0) done = true;
            D.tn[a2] = D.plane_t(r, a2, D.c[a2] + (sg > 0 ? 1 : 0));
          } else {
            D.c[a2] += D.s[a2];
            if (D.c[a2] < 0 || D.c[a2] >= D.nb[a2]) done = true;
            D.tn[a2] = D.plane_t(r, a2, D.c[a2] + (D.s[a2] > 0));
          }
        }
      }
    }
    if (open) emit(ma, mb);
  }
  counts[pix] = n;
  if (flags) atomicOr(flags_out, flags);
}

// k_segments specialised for the macro-cell grid (_k_grid: _dda_runs then _sort_merge): the
// same GridDDA steps, runs and merge as the generic kernel in one flat loop.  SGN as for
// k_segments_brick (direction sign bits; -1: general).
template <int SGN>
__global__ void __launch_bounds__(RENDER_TX* RENDER_TY, VS_SEGMENTS_MINB)
    k_segments_grid(vs_volume_desc vol, vs_index_desc ix, vs_camera_desc cam, vs_rows_desc rows,
                    double dt, int2* __restrict__ segs, int* __restrict__ counts, int cap,
                    int* __restrict__ flags_out) {
  const int i = blockIdx.x * RENDER_TX + threadIdx.x;
  const int l = blockIdx.y * RENDER_TY + threadIdx.y;
  if (i >= cam.width || l >= rows.nrows) return;
  const int64_t pix = (int64_t)l * cam.width + i;
  const int64_t npix = (int64_t)rows.nrows * cam.width;
  Ray r;
  pixel_ray(cam, rows, i, l, r);
  int n = 0, flags = 0;
  double tmin, tmax;
  if (slab(r, 0.0, 0.0, 0.0, (double)vol.nx, (double)vol.ny, (double)vol.nz, tmin, tmax)) {
    GridDDA G;
    G.init(r, ix, tmin, tmax);
    Integrator L;  // lattice only
    L.entry = tmin;
    L.dt = dt;
    L.inv_dt = 1.0 / dt;
    bool open = false;
    double ma = 0.0, mb = 0.0, last_t0 = -DBL_MAX;
    int kprev = -1;
    auto emit = [&](double a, double b) {
      const int k0 = (int)L.first_k(a), k1 = (int)L.first_k(b);
      if (k1 <= k0) return;
      if (n > 0 && k0 == kprev && n <= cap) {
        segs[(int64_t)(n - 1) * npix + pix].y = k1;
      } else {
        if (n < cap) segs[(int64_t)n * npix + pix] = make_int2(k0, k1);
        ++n;
      }
      kprev = k1;
    };
    auto feed = [&](double a, double b) {  // MergeState::feed
      if (a < last_t0) flags |= RF_ORDER;
      last_t0 = a;
      if (b <= a) return;
      if (open && a <= mb) {
        if (b > mb) mb = b;
        return;
      }
      if (open) emit(ma, mb);
      ma = a;
      mb = b;
      open = true;
    };
    const int ncy = G.ncy, ncz = G.ncz;
    int cx = (int)G.cx, cy = (int)G.cy, cz = (int)G.cz;
    int steps = 0;
    const int max_steps = (int)G.max_steps;
    bool run = false;
    double run_t0 = 0.0, tcur = tmin;
    while (steps < max_steps) {
      double tn = G.tnx;
      if (G.tny < tn) tn = G.tny;
      if (G.tnz < tn) tn = G.tnz;
      if (__ldg(G.occ + ((int64_t)cx * ncy + cy) * ncz + cz)) {
        if (!run) { run = true; run_t0 = tcur; }
      } else if (run) {
        feed(run_t0, tcur);
        run = false;
      }
      ++steps;
      if (tn >= tmax) break;
      if constexpr (SGN >= 0) {
        constexpr int SX = (SGN & 1) ? 1 : -1, SY = (SGN & 2) ? 1 : -1, SZ = (SGN & 4) ? 1 : -1;
        if (G.tnx == tn) { cx += SX; G.tnx = G.cross(cx, SX, r.ox, r.ix); }
        if (G.tny == tn) { cy += SY; G.tny = G.cross(cy, SY, r.oy, r.iy); }
        if (G.tnz == tn) { cz += SZ; G.tnz = G.cross(cz, SZ, r.oz, r.iz); }
        tcur = tn;
        if ((SX < 0 ? cx < 0 : cx >= G.ncx) || (SY < 0 ? cy < 0 : cy >= ncy) ||
            (SZ < 0 ? cz < 0 : cz >= ncz))
          break;
      } else {
        if (G.tnx == tn) { cx += G.sx; G.tnx = G.cross(cx, G.sx, r.ox, r.ix); }
        if (G.tny == tn) { cy += G.sy; G.tny = G.cross(cy, G.sy, r.oy, r.iy); }
        if (G.tnz == tn) { cz += G.sz; G.tnz = G.cross(cz, G.sz, r.oz, r.iz); }
        tcur = tn;
        if (cx < 0 || cy < 0 || cz < 0 || cx >= G.ncx || cy >= ncy || cz >= ncz) break;
      }
    }
    if (run) feed(run_t0, tmax);
    if (open) emit(ma, mb);
  }
  counts[pix] = n;
  if (flags) atomicOr(flags_out, flags);
}

// k_segments specialised for the k-d tree (_k_kd: _kd_leaves then _sort_merge): one node visit
// per turn, the merge and lattice-range emission inline (same KdWalk / MergeState steps).
__global__ void __launch_bounds__(RENDER_TX* RENDER_TY, VS_SEGMENTS_MINB)
    k_segments_kd(vs_volume_desc vol, vs_index_desc ix, vs_camera_desc cam, vs_rows_desc rows,
                  double dt, int2* __restrict__ segs, int* __restrict__ counts, int cap,
                  int* __restrict__ flags_out) {
  const int i = blockIdx.x * RENDER_TX + threadIdx.x;
  const int l = blockIdx.y * RENDER_TY + threadIdx.y;
  if (i >= cam.width || l >= rows.nrows) return;
  const int64_t pix = (int64_t)l * cam.width + i;
  const int64_t npix = (int64_t)rows.nrows * cam.width;
  Ray r;
  pixel_ray(cam, rows, i, l, r);
  int n = 0, flags = 0;
  double tmin, tmax;
  if (slab(r, 0.0, 0.0, 0.0, (double)vol.nx, (double)vol.ny, (double)vol.nz, tmin, tmax)) {
    KdWalk K;
    K.init(ix, tmin, tmax);
    Integrator L;  // lattice only
    L.entry = tmin;
    L.dt = dt;
    L.inv_dt = 1.0 / dt;
    bool open = false;
    double ma = 0.0, mb = 0.0, last_t0 = -DBL_MAX;
    int kprev = -1;
    auto emit = [&](double a, double b) {
      const int k0 = (int)L.first_k(a), k1 = (int)L.first_k(b);
      if (k1 <= k0) return;
      if (n > 0 && k0 == kprev && n <= cap) {
        segs[(int64_t)(n - 1) * npix + pix].y = k1;
      } else {
        if (n < cap) segs[(int64_t)n * npix + pix] = make_int2(k0, k1);
        ++n;
      }
      kprev = k1;
    };
    while (K.sp > 0) {
      const int nd = K.stk[--K.sp];
      double a, b;
      if (!node_slab(r, K.lo, K.hi, nd, a, b)) continue;
      a = a > tmin ? a : tmin;
      b = b < tmax ? b : tmax;
      if (b <= a) continue;
      const int ax = __ldg(K.axis + nd);
      if (ax < 0) {
        if (a < last_t0) flags |= RF_ORDER;
        last_t0 = a;
        if (open && a <= mb) {
          if (b > mb) mb = b;
        } else {
          if (open) emit(ma, mb);
          ma = a;
          mb = b;
          open = true;
        }
        continue;
      }
      const double pl = (double)__ldg(K.plane + nd);
      bool front_left;
      const bool zero = ax == 0 ? r.zx : (ax == 1 ? r.zy : r.zz);
      if (zero)
        front_left = (ax == 0 ? r.ox : (ax == 1 ? r.oy : r.oz)) < pl;
      else
        front_left = (ax == 0 ? r.ix : (ax == 1 ? r.iy : r.iz)) > 0.0;
      const int lc = __ldg(K.left + nd), rc = __ldg(K.right + nd);
      const int nr = front_left ? lc : rc, fr = front_left ? rc : lc;
      if (K.sp + 2 > STACK_CAP) { flags |= RF_OVERFLOW; break; }
      if (fr >= 0) K.stk[K.sp++] = fr;
      if (nr >= 0) K.stk[K.sp++] = nr;
    }
    if (open) emit(ma, mb);
  }
  counts[pix] = n;
  if (flags) atomicOr(flags_out, flags);
}

// k_segments specialised for the hybrid (_k_hybrid: k-d leaf intervals -> _sort_merge -> for
// each merged leaf interval _dda_runs over the macro grid -> _sort_merge), one flat loop whose
// turn is either one k-d node visit or one grid DDA step; same steps and merges as the
// generic generator stack (KdWalk, MergeState, GridDDA).
template <int SGN>
__global__ void __launch_bounds__(RENDER_TX* RENDER_TY, 6)
    k_segments_hybrid(vs_volume_desc vol, vs_index_desc ix, vs_camera_desc cam, vs_rows_desc rows,
                      double dt, int2* __restrict__ segs, int* __restrict__ counts, int cap,
                      int* __restrict__ flags_out) {
  const int i = blockIdx.x * RENDER_TX + threadIdx.x;
  const int l = blockIdx.y * RENDER_TY + threadIdx.y;
  if (i >= cam.width || l >= rows.nrows) return;
  const int64_t pix = (int64_t)l * cam.width + i;
  const int64_t npix = (int64_t)rows.nrows * cam.width;
  Ray r;
  pixel_ray(cam, rows, i, l, r);
  int n = 0, flags = 0;
  double tmin, tmax;
  if (slab(r, 0.0, 0.0, 0.0, (double)vol.nx, (double)vol.ny, (double)vol.nz, tmin, tmax)) {
    KdWalk K;
    K.init(ix, tmin, tmax);
    Integrator L;  // lattice only
    L.entry = tmin;
    L.dt = dt;
    L.inv_dt = 1.0 / dt;
    // final merge + lattice-range emission
    bool open = false;
    double ma = 0.0, mb = 0.0, last_t0 = -DBL_MAX;
    int kprev = -1;
    auto emit = [&](double a, double b) {
      const int k0 = (int)L.first_k(a), k1 = (int)L.first_k(b);
      if (k1 <= k0) return;
      if (n > 0 && k0 == kprev && n <= cap) {
        segs[(int64_t)(n - 1) * npix + pix].y = k1;
      } else {
        if (n < cap) segs[(int64_t)n * npix + pix] = make_int2(k0, k1);
        ++n;
      }
      kprev = k1;
    };
    auto feed = [&](double a, double b) {
      if (a < last_t0) flags |= RF_ORDER;
      last_t0 = a;
      if (b <= a) return;
      if (open && a <= mb) {
        if (b > mb) mb = b;
        return;
      }
      if (open) emit(ma, mb);
      ma = a;
      mb = b;
      open = true;
    };
    // leaf-interval merge
    bool lopen = false, kd_done = false;
    double la = 0.0, lb = 0.0, llast = -DBL_MAX;
    // grid walk over the current merged leaf interval [g_in, g_out)
    bool gactive = false, run = false;
    GridDDA G;
    int gsteps = 0, gmax = 0;
    double run_t0 = 0.0, tcur = 0.0, g_out = 0.0;
    auto start_grid = [&](double a, double b) {
      G.init(r, ix, a, b);
      gactive = true;
      run = false;
      gsteps = 0;
      gmax = (int)G.max_steps;
      tcur = a;
      g_out = b;
    };
    while (true) {
      if (gactive) {
        // one _dda_runs step (GridDDA::next)
        bool fin = gsteps >= gmax;
        if (!fin) {
          double tn = G.tnx;
          if (G.tny < tn) tn = G.tny;
          if (G.tnz < tn) tn = G.tnz;
          if (__ldg(G.occ + (G.cx * G.ncy + G.cy) * G.ncz + G.cz)) {
            if (!run) { run = true; run_t0 = tcur; }
          } else if (run) {
            feed(run_t0, tcur);
            run = false;
          }
          ++gsteps;
          if (tn >= g_out) {
            fin = true;
          } else if constexpr (SGN >= 0) {  // direction signs known (k_segments_brick)
            constexpr int SX = (SGN & 1) ? 1 : -1, SY = (SGN & 2) ? 1 : -1,
                          SZ = (SGN & 4) ? 1 : -1;
            if (G.tnx == tn) { G.cx += SX; G.tnx = G.cross(G.cx, SX, r.ox, r.ix); }
            if (G.tny == tn) { G.cy += SY; G.tny = G.cross(G.cy, SY, r.oy, r.iy); }
            if (G.tnz == tn) { G.cz += SZ; G.tnz = G.cross(G.cz, SZ, r.oz, r.iz); }
            tcur = tn;
            if ((SX < 0 ? G.cx < 0 : G.cx >= G.ncx) || (SY < 0 ? G.cy < 0 : G.cy >= G.ncy) ||
                (SZ < 0 ? G.cz < 0 : G.cz >= G.ncz))
              fin = true;
          } else {
            if (G.tnx == tn) { G.cx += G.sx; G.tnx = G.cross(G.cx, G.sx, r.ox, r.ix); }
            if (G.tny == tn) { G.cy += G.sy; G.tny = G.cross(G.cy, G.sy, r.oy, r.iy); }
            if (G.tnz == tn) { G.cz += G.sz; G.tnz = G.cross(G.cz, G.sz, r.oz, r.iz); }
            tcur = tn;
            if (G.cx < 0 || G.cy < 0 || G.cz < 0 || G.cx >= G.ncx || G.cy >= G.ncy ||
                G.cz >= G.ncz)
              fin = true;
          }
        }
        if (fin) {
          if (run) feed(run_t0, g_out);
          gactive = false;
        }
        continue;
      }
      if (!kd_done) {
        // one k-d node visit (KdWalk::next)
        if (K.sp == 0) {
          kd_done = true;
          continue;
        }
        const int nd = K.stk[--K.sp];
        double a, b;
        if (!node_slab(r, K.lo, K.hi, nd, a, b)) continue;
        a = a > tmin ? a : tmin;
        b = b < tmax ? b : tmax;
        if (b <= a) continue;
        const int ax = __ldg(K.axis + nd);
        if (ax < 0) {
          // raw leaf interval -> leaf merge (MergeState::feed)
          if (a < llast) flags |= RF_ORDER;
          llast = a;
          if (lopen && a <= lb) {
            if (b > lb) lb = b;
          } else {
            const bool out = lopen;
            const double oa = la, ob = lb;
            la = a;
            lb = b;
            lopen = true;
            if (out) start_grid(oa, ob);
          }
          continue;
        }
        const double pl = (double)__ldg(K.plane + nd);
        bool front_left;
        const bool zero = ax == 0 ? r.zx : (ax == 1 ? r.zy : r.zz);
        if (zero)
          front_left = (ax == 0 ? r.ox : (ax == 1 ? r.oy : r.oz)) < pl;
        else
          front_left = (ax == 0 ? r.ix : (ax == 1 ? r.iy : r.iz)) > 0.0;
        const int lc = __ldg(K.left + nd), rc = __ldg(K.right + nd);
        const int nr = front_left ? lc : rc, fr = front_left ? rc : lc;
        if (K.sp + 2 > STACK_CAP) { flags |= RF_OVERFLOW; kd_done = true; continue; }
        if (fr >= 0) K.stk[K.sp++] = fr;
        if (nr >= 0) K.stk[K.sp++] = nr;
        continue;
      }
      if (lopen) {  // drain the last merged leaf interval
        lopen = false;
        start_grid(la, lb);
        continue;
      }
      break;
    }
    if (open) emit(ma, mb);
  }
  counts[pix] = n;
  if (flags) atomicOr(flags_out, flags);
}

// Output of one integrated ray (render_frame quantisation + optional float RGBA / samples).
__device__ __forceinline__ void write_pixel(const Integrator& I, int64_t pix,
                                            uint8_t* __restrict__ rgba8,
                                            double* __restrict__ rgba64,
                                            int32_t* __restrict__ samples) {
  const double acc[4] = {I.accr, I.accg, I.accb, I.acca};
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const double q = floor(__dadd_rn(__dmul_rn(acc[c], 255.0), 0.5));
    rgba8[4 * pix + c] = (uint8_t)(q < 0.0 ? 0 : (q > 255.0 ? 255 : (int)q));
    if (rgba64) rgba64[4 * pix + c] = acc[c];
  }
  if (samples) samples[pix] = I.taken;
}

__device__ __forceinline__ void load_tables(RenderSmem& sm, const float* __restrict__ lut,
                                            const double* __restrict__ corr, int tid, int nt) {
  for (int k = tid; k < 256; k += nt) {
    sm.lut[k] = make_float4(lut[4 * k], lut[4 * k + 1], lut[4 * k + 2], lut[4 * k + 3]);
    sm.corr[k] = corr[k];
    sm.u8f[k] = (float)((double)k / 255.0);
  }
}

__device__ __forceinline__ void add_total(unsigned long long* total, int64_t taken, int tid) {
  if (total) {
    unsigned long long t = (unsigned long long)taken;
    for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if ((tid & 31) == 0 && t) atomicAdd(total, t);
  }
}

// A ray with more lattice ranges than the buffer holds: traversal and integration fused
// (re-traverses the index).  Out of line, taking only values, so neither the sample loop's
// register budget nor its locals depend on the traversal state.
struct FusedOut {
  double r, g, b, a;
  int taken, flags;
};

template <int KIND, bool ERT>
__device__ __noinline__ FusedOut integrate_fused(vs_volume_desc vol, vs_index_desc ix,
                                                 vs_camera_desc cam, vs_rows_desc rows,
                                                 const RenderSmem* sm, double dt, double ert_a,
                                                 int i, int l) {
  Ray r;
  pixel_ray(cam, rows, i, l, r);
  Integrator I;
  I.r = &r; I.sm = sm; I.bins = vol.bins; I.field = nullptr; I.quads = vol.quads;
  I.idx32 = (int64_t)vol.nx * vol.ny * vol.nz < (1LL << 32); I.use_tab = true;
  I.nx = vol.nx; I.ny = vol.ny; I.nz = vol.nz; I.dt = dt; I.inv_dt = 1.0 / dt;
  I.nearest = false;
  I.ert_a = ERT ? ert_a : 2.0;
  I.accr = I.accg = I.accb = I.acca = 0.0;
  I.taken = 0;
  int flags = 0;
  double tmin, tmax;
  if (slab(r, 0.0, 0.0, 0.0, (double)vol.nx, (double)vol.ny, (double)vol.nz, tmin, tmax)) {
    I.entry = tmin;
    SegmentSource<KIND> src;
    src.init(r, ix, vol.nx, vol.ny, vol.nz, tmin, tmax);
    while (!I.terminated()) {
      int budget = 1 << 30;
      double a, b;
      const int g = src.next(r, ix, a, b, budget, &flags);
      if (g == 0) break;
      I.segment(a, b);
    }
  }
  return FusedOut{I.accr, I.accg, I.accb, I.acca, I.taken, flags};
}

// The hot integration kernel: u8 volumes through the quad gather volume, trilinear (float
// fields and nearest sampling go to k_integrate_fallback).  Rays whose lattice ranges fit the
// segment buffer run the sample-stream loop; the rare overflowing ray calls integrate_fused.
template <int KIND, bool IDX32, bool ERT>
__global__ void __launch_bounds__(RENDER_TX* RENDER_TY, VS_INTEGRATE_MINB)
    k_integrate_segments(vs_volume_desc vol, vs_index_desc ix, vs_camera_desc cam,
                         const float* __restrict__ lut, const double* __restrict__ corr,
                         double dt, vs_rows_desc rows, const int2* __restrict__ segs,
                         const int* __restrict__ counts, int cap, uint8_t* __restrict__ rgba8,
                         double* __restrict__ rgba64, int32_t* __restrict__ samples,
                         unsigned long long* __restrict__ total, int* __restrict__ flags_out,
                         double ert_a) {
  __shared__ RenderSmem sm;
  const int tid = threadIdx.y * RENDER_TX + threadIdx.x;
  load_tables(sm, lut, corr, tid, RENDER_TX * RENDER_TY);
  __syncthreads();
  const int i = blockIdx.x * RENDER_TX + threadIdx.x;
  const int l = blockIdx.y * RENDER_TY + threadIdx.y;
  int64_t taken = 0;
  int flags = 0;
  if (i < cam.width && l < rows.nrows) {
    const int64_t pix = (int64_t)l * cam.width + i;
    const int64_t npix = (int64_t)rows.nrows * cam.width;
    const int n = counts[pix];
    {
      Ray r;
      pixel_ray(cam, rows, i, l, r);
      Integrator I;
      I.r = &r; I.sm = &sm; I.bins = vol.bins; I.field = nullptr; I.quads = vol.quads;
      I.idx32 = IDX32; I.use_tab = true;
      I.nx = vol.nx; I.ny = vol.ny; I.nz = vol.nz; I.dt = dt; I.inv_dt = 1.0 / dt;
      I.nearest = false;
      I.ert_a = ERT ? ert_a : 2.0;
      I.accr = I.accg = I.accb = I.acca = 0.0;
      I.taken = 0;
      double tmin, tmax;
      if (n > cap) {
        const FusedOut f = integrate_fused<KIND, ERT>(vol, ix, cam, rows, &sm, dt, ert_a, i, l);
        I.accr = f.r; I.accg = f.g; I.accb = f.b; I.acca = f.a; I.taken = f.taken;
        flags |= f.flags;
      } else if (n > 0 && slab(r, 0.0, 0.0, 0.0, (double)vol.nx, (double)vol.ny, (double)vol.nz, tmin, tmax)) {
        I.entry = tmin;
        // the ray's lattice ranges as one sample stream (ranges are non-empty): every turn
        // shades one sample, the next range is prefetched one range ahead, and the next
        // sample's gather is issued before the current sample's arithmetic, across range ends
        int q = 0;
        int2 kr = segs[pix];
        int2 krn = n > 1 ? segs[npix + pix] : make_int2(0, 0);
        const uint32_t lut_s = (uint32_t)__cvta_generic_to_shared(sm.lut);
        const uint32_t corr_s = (uint32_t)__cvta_generic_to_shared(sm.corr);
        // the stream cursor: kc = the last lattice index whose gather was issued
        int kc = kr.x;
        auto advance = [&]() -> bool {
          int kn = kc + 1;
          if (kn >= kr.y) {
            if (q + 1 >= n) return false;
            ++q;
            kr = krn;
            kn = kr.x;
            if (q + 1 < n) krn = segs[(int64_t)(q + 1) * npix + pix];
          }
          kc = kn;
          return true;
        };
        auto shade = [&](Integrator::Gather& g) {
          Integrator::settle(g);
          // (render option RO_FP64_BINS sends every ray to k_integrate_fallback instead: all
          // samples through the FP64 path, the check of this filter's exactness)
          int bin = I.bin_fast(g);
          if (bin < 0) bin = Integrator::bin_of(I.interp_t<true>(g));
          // I.shade_bin(bin) on the kernel's shared tables, addressed from 32-bit shared
          // offsets taken once (the generic path re-derives the CTA's window every sample)
          float4 c;
          asm("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
              : "=f"(c.x), "=f"(c.y), "=f"(c.z), "=f"(c.w)
              : "r"(lut_s + 16u * (uint32_t)bin));
          if (c.w > 0.0f) {
            double cr;
            asm("ld.shared.f64 %0, [%1];" : "=d"(cr) : "r"(corr_s + 8u * (uint32_t)bin));
            const double w = __dmul_rn(1.0 - I.acca, cr);
            I.accr = __dadd_rn(I.accr, __dmul_rn(w, (double)c.x));
            I.accg = __dadd_rn(I.accg, __dmul_rn(w, (double)c.y));
            I.accb = __dadd_rn(I.accb, __dmul_rn(w, (double)c.z));
            I.acca = __dadd_rn(I.acca, w);
          }
          ++I.taken;
        };
        auto issue = [&](Integrator::Gather& g) {
          I.gather_t<IDX32, true>(__dadd_rn(I.entry, __dmul_rn((double)kc, dt)), g);
        };
        constexpr int PF = VS_PREFETCH;
        if constexpr (PF >= 2) {
        // gathers issued two samples ahead; the loop is unrolled three times so the three
        // gather slots rotate by role, never by copying (a copy of a loaded register waits on
        // the load like any other use)
        Integrator::Gather g0, g1, g2;
        issue(g0);
        bool h0 = true, h1 = advance(), h2 = false;
        if (h1) issue(g1);
        while (true) {
          h2 = h1 && advance();
          if (h2) issue(g2);
          shade(g0);
          if (!h1 || (ERT && I.terminated())) break;
          h0 = h2 && advance();
          if (h0) issue(g0);
          shade(g1);
          if (!h2 || (ERT && I.terminated())) break;
          h1 = h0 && advance();
          if (h1) issue(g1);
          shade(g2);
          if (!h0 || (ERT && I.terminated())) break;
        }
        } else {
        Integrator::Gather g;
        issue(g);
        while (true) {
          const bool hn = advance();
          Integrator::Gather gn;
          if (hn) issue(gn);
          shade(g);
          if (!hn || (ERT && I.terminated())) break;
          g = gn;
        }
        }
      }
      taken = I.taken;
      write_pixel(I, pix, rgba8, rgba64, samples);
    }
  }
  if (flags) atomicOr(flags_out, flags);
  add_total(total, taken, tid);
}

// Volumes k_integrate_segments does not take: float fields / no quad volume / nearest
// sampling (generic sample path over the stored ranges, fused path for overflowing rays).
template <int KIND, bool ERT>
__global__ void __launch_bounds__(RENDER_TX* RENDER_TY)
    k_integrate_fallback(vs_volume_desc vol, vs_index_desc ix, vs_camera_desc cam,
                         const float* __restrict__ lut, const double* __restrict__ corr, double dt,
                         int nearest, vs_rows_desc rows, const int2* __restrict__ segs,
                         const int* __restrict__ counts, int cap, uint8_t* __restrict__ rgba8,
                         double* __restrict__ rgba64, int32_t* __restrict__ samples,
                         unsigned long long* __restrict__ total, int* __restrict__ flags_out,
                         int render_opts, double ert_a) {
  __shared__ RenderSmem sm;
  const int tid = threadIdx.y * RENDER_TX + threadIdx.x;
  // RO_FP64_BINS (render_opts & 2): every ray here, sampled with the FP64 arithmetic only
  const bool generic = vol.field || !vol.quads || nearest || (render_opts & 2);
  const int i = blockIdx.x * RENDER_TX + threadIdx.x;
  const int l = blockIdx.y * RENDER_TY + threadIdx.y;
  const bool inside = i < cam.width && l < rows.nrows;
  const int64_t pix = (int64_t)l * cam.width + i;
  const int n = inside ? counts[pix] : 0;
  const bool mine = inside && generic;
  if (!__syncthreads_or(mine)) return;  // the common case: nothing to do in this tile
  load_tables(sm, lut, corr, tid, RENDER_TX * RENDER_TY);
  __syncthreads();
  int64_t taken = 0;
  int flags = 0;
  if (mine) {
    const int64_t npix = (int64_t)rows.nrows * cam.width;
    Ray r;
    pixel_ray(cam, rows, i, l, r);
    Integrator I;
    I.r = &r; I.sm = &sm; I.bins = vol.bins; I.field = vol.field;
    I.quads = vol.field ? nullptr : vol.quads;
    I.idx32 = (int64_t)vol.nx * vol.ny * vol.nz < (1LL << 32);
    I.use_tab = (render_opts & 1) != 0;
    I.nx = vol.nx; I.ny = vol.ny; I.nz = vol.nz; I.dt = dt; I.inv_dt = 1.0 / dt;
    I.nearest = nearest != 0;
    I.ert_a = ERT ? ert_a : 2.0;
    I.accr = I.accg = I.accb = I.acca = 0.0;
    I.taken = 0;
    I.active = false;
    double tmin, tmax;
    if (n > 0 && slab(r, 0.0, 0.0, 0.0, (double)vol.nx, (double)vol.ny, (double)vol.nz, tmin, tmax)) {
      I.entry = tmin;
      if (n <= cap) {
        // flat sample loop: each turn either samples or switches to the next lattice range
        int q = 0;
        int2 kr = segs[pix];
        int k = kr.x;
        while (true) {
          if (k < kr.y) {
            I.t = __dadd_rn(I.entry, __dmul_rn((double)k, dt));
            I.sample_at();
            if (ERT && I.terminated()) break;
            ++k;
          } else {
            if (++q >= n) break;
            kr = segs[(int64_t)q * npix + pix];
            k = kr.x;
          }
        }
      } else {  // overflow: fused traversal + integration for this ray
        SegmentSource<KIND> src;
        src.init(r, ix, vol.nx, vol.ny, vol.nz, tmin, tmax);
        while (!I.terminated()) {
          int budget = 1 << 30;
          double a, b;
          const int g = src.next(r, ix, a, b, budget, &flags);
          if (g == 0) break;
          I.segment(a, b);
        }
      }
    }
    taken = I.taken;
    write_pixel(I, pix, rgba8, rgba64, samples);
  }
  if (flags) atomicOr(flags_out, flags);
  add_total(total, taken, tid);
}

// Single-ray traversal (render.py:917-961): the merged interval list of each ray.
template <int KIND>
__device__ void traverse_one(const Ray& r, const vs_index_desc& ix, int nx, int ny, int nz,
                             double tmin, double tmax, double* out, int cap, int& n, int* flags) {
  SegmentSource<KIND> src;
  src.init(r, ix, nx, ny, nz, tmin, tmax);
  while (true) {
    int budget = 1 << 30;
    double a, b;
    const int g = src.next(r, ix, a, b, budget, flags);
    if (g == 0) break;
    if (g == 1) {
      if (n < cap) { out[2 * n] = a; out[2 * n + 1] = b; }
      ++n;
    }
  }
}

__global__ void k_traverse_rays(vs_index_desc ix, int nx, int ny, int nz,
                                const double* __restrict__ origins, const double* __restrict__ dir,
                                int nrays, double* __restrict__ out, int cap,
                                int* __restrict__ counts, int* __restrict__ flags_out) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nrays) return;
  vs_camera_desc c;
  c.dir[0] = dir[0]; c.dir[1] = dir[1]; c.dir[2] = dir[2];
  Ray r;
  ray_setup(r, origins[3 * q], origins[3 * q + 1], origins[3 * q + 2], c);
  int flags = 0, n = 0;
  double* o = out + (int64_t)q * cap * 2;
  double tmin, tmax;
  if (slab(r, 0.0, 0.0, 0.0, (double)nx, (double)ny, (double)nz, tmin, tmax)) {
    switch (ix.kind) {
      case VS_KIND_NAIVE: traverse_one<VS_KIND_NAIVE>(r, ix, nx, ny, nz, tmin, tmax, o, cap, n, &flags); break;
      case VS_KIND_GRID: traverse_one<VS_KIND_GRID>(r, ix, nx, ny, nz, tmin, tmax, o, cap, n, &flags); break;
      case VS_KIND_LBVH:
        if (ix.brick_bits)
          traverse_one<KIND_LBVH_BRICK>(r, ix, nx, ny, nz, tmin, tmax, o, cap, n, &flags);
        else
          traverse_one<VS_KIND_LBVH>(r, ix, nx, ny, nz, tmin, tmax, o, cap, n, &flags);
        break;
      case VS_KIND_KD: traverse_one<VS_KIND_KD>(r, ix, nx, ny, nz, tmin, tmax, o, cap, n, &flags); break;
      default: traverse_one<VS_KIND_HYBRID>(r, ix, nx, ny, nz, tmin, tmax, o, cap, n, &flags); break;
    }
  }
  counts[q] = n;
  if (flags) atomicOr(flags_out, flags);
}

// Single-ray integration over given segments (render.py:964-1015).
__global__ void k_integrate_rays(vs_volume_desc vol, const double* __restrict__ origins,
                                 const double* __restrict__ dir, const double* __restrict__ segs,
                                 const int* __restrict__ counts, int cap, int nrays,
                                 const float* __restrict__ lut, const double* __restrict__ corr,
                                 double dt, int nearest, double* __restrict__ rgba,
                                 long long* __restrict__ samples) {
  const int render_opts = 0;
  __shared__ RenderSmem sm;
  for (int k = threadIdx.x; k < 256; k += blockDim.x) {
    sm.lut[k] = make_float4(lut[4 * k], lut[4 * k + 1], lut[4 * k + 2], lut[4 * k + 3]);
    sm.corr[k] = corr[k];
    sm.u8f[k] = (float)((double)k / 255.0);
  }
  __syncthreads();
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nrays) return;
  vs_camera_desc c;
  c.dir[0] = dir[0]; c.dir[1] = dir[1]; c.dir[2] = dir[2];
  Ray r;
  ray_setup(r, origins[3 * q], origins[3 * q + 1], origins[3 * q + 2], c);
  Integrator I;
  I.r = &r; I.sm = &sm; I.bins = vol.bins; I.field = vol.field;
  I.quads = vol.field ? nullptr : vol.quads;
    I.idx32 = (int64_t)vol.nx * vol.ny * vol.nz < (1LL << 32);
    I.use_tab = (render_opts & 1) != 0;
  I.nx = vol.nx; I.ny = vol.ny; I.nz = vol.nz; I.dt = dt; I.inv_dt = 1.0 / dt; I.nearest = nearest != 0;
  I.ert_a = 2.0;  // single-ray API: the reference integrator, no termination
  I.accr = I.accg = I.accb = I.acca = 0.0;
  I.taken = 0;
  const int m = counts[q];
  double entry, ex;
  if (m > 0 && slab(r, 0.0, 0.0, 0.0, (double)vol.nx, (double)vol.ny, (double)vol.nz, entry, ex)) {
    I.entry = entry;
    for (int s = 0; s < m && s < cap; ++s)
      I.segment(segs[((int64_t)q * cap + s) * 2], segs[((int64_t)q * cap + s) * 2 + 1]);
  }
  rgba[4 * q] = I.accr;
  rgba[4 * q + 1] = I.accg;
  rgba[4 * q + 2] = I.accb;
  rgba[4 * q + 3] = I.acca;
  samples[q] = I.taken;
}

__global__ void k_build_quads(const uint8_t* __restrict__ b, int nx, int ny, int nz,
                              uint32_t* __restrict__ q) {
  const int64_t n = (int64_t)nx * ny * nz;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int z = (int)(i % nz);
  const int y = (int)((i / nz) % ny);
  const int x = (int)(i / ((int64_t)ny * nz));
  const int64_t dz = z + 1 < nz ? 1 : 0, dy = y + 1 < ny ? nz : 0;
  const uint32_t v0 = b[i], v1 = b[i + dz], v2 = b[i + dy], v3 = b[i + dy + dz];
  const QuadGeom qg(nx, ny, nz);
  q[qg.at(x, qg.yz(y, z))] = v0 | (v1 << 8) | (v2 << 16) | (v3 << 24);
}

__global__ void k_brick_grid(const int32_t* __restrict__ coords, const int* __restrict__ n_dev,
                             int64_t n_host, int nby, int nbz, uint32_t* __restrict__ bits) {
  const int64_t n = n_dev ? (int64_t)*n_dev : n_host;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t lin = ((int64_t)coords[3 * i] * nby + coords[3 * i + 1]) * nbz + coords[3 * i + 2];
  atomicOr(bits + (lin >> 5), 1u << (lin & 31));
}

// Direction sign bits of the (orthographic, frame-uniform) camera, -1 if a component is 0.
static int dir_signs(const vs_camera_desc& c) {
  int sgn = 0;
  for (int a = 0; a < 3; ++a) {
    if (c.dir[a] == 0.0) return -1;
    if (c.dir[a] > 0.0) sgn |= 1 << a;
  }
  return sgn;
}

static void launch_segments_grid(dim3 grid, cudaStream_t st, const vs_volume_desc& v,
                                 const vs_index_desc& ix, const vs_camera_desc& c,
                                 const vs_rows_desc& rows, double dt, int2* segs, int* counts,
                                 int cap, int* flags) {
  const dim3 blk(RENDER_TX, RENDER_TY);
  switch (dir_signs(c)) {
#define VS_SEG_GRID(S) \
  case S: k_segments_grid<S><<<grid, blk, 0, st>>>(v, ix, c, rows, dt, segs, counts, cap, flags); break;
    VS_SEG_GRID(0) VS_SEG_GRID(1) VS_SEG_GRID(2) VS_SEG_GRID(3)
    VS_SEG_GRID(4) VS_SEG_GRID(5) VS_SEG_GRID(6) VS_SEG_GRID(7)
#undef VS_SEG_GRID
    default:
      k_segments_grid<-1><<<grid, blk, 0, st>>>(v, ix, c, rows, dt, segs, counts, cap, flags);
  }
}

static void launch_segments_hybrid(dim3 grid, cudaStream_t st, const vs_volume_desc& v,
                                   const vs_index_desc& ix, const vs_camera_desc& c,
                                   const vs_rows_desc& rows, double dt, int2* segs, int* counts,
                                   int cap, int* flags) {
  const dim3 blk(RENDER_TX, RENDER_TY);
  switch (dir_signs(c)) {
#define VS_SEG_HYB(S) \
  case S: k_segments_hybrid<S><<<grid, blk, 0, st>>>(v, ix, c, rows, dt, segs, counts, cap, flags); break;
    VS_SEG_HYB(0) VS_SEG_HYB(1) VS_SEG_HYB(2) VS_SEG_HYB(3)
    VS_SEG_HYB(4) VS_SEG_HYB(5) VS_SEG_HYB(6) VS_SEG_HYB(7)
#undef VS_SEG_HYB
    default:
      k_segments_hybrid<-1><<<grid, blk, 0, st>>>(v, ix, c, rows, dt, segs, counts, cap, flags);
  }
}

// k_segments_brick instantiation for the camera: sign bits when no direction component is 0.
static void launch_segments_brick(dim3 grid, cudaStream_t st, const vs_volume_desc& v,
                                  const vs_index_desc& ix, const vs_camera_desc& c,
                                  const vs_rows_desc& rows, double dt, int2* segs, int* counts,
                                  int cap, int* flags, int exact_runs) {
  const dim3 blk(RENDER_TX, RENDER_TY);
  switch (dir_signs(c)) {
#define VS_SEG_BRICK(S) \
  case S: k_segments_brick<S><<<grid, blk, 0, st>>>(v, ix, c, rows, dt, segs, counts, cap, flags, exact_runs); break;
    VS_SEG_BRICK(0) VS_SEG_BRICK(1) VS_SEG_BRICK(2) VS_SEG_BRICK(3)
    VS_SEG_BRICK(4) VS_SEG_BRICK(5) VS_SEG_BRICK(6) VS_SEG_BRICK(7)
#undef VS_SEG_BRICK
    default:
      k_segments_brick<-1><<<grid, blk, 0, st>>>(v, ix, c, rows, dt, segs, counts, cap, flags,
                                                  exact_runs);
  }
}

template <int K>
static void launch_render(dim3 grid, cudaStream_t st, const vs_volume_desc& v,
                          const vs_index_desc& ix, const vs_camera_desc& c, const float* lut,
                          const double* corr, double dt, int nearest, const vs_rows_desc& rows,
                          uint8_t* rgba8, double* rgba64, int32_t* samples,
                          unsigned long long* total, int* flags, const RenderCfg& cfg) {
  if (cfg.seg_ws && cfg.seg_cap > 0) {
    const int64_t npix = (int64_t)rows.nrows * c.width;
    int2* segs = static_cast<int2*>(cfg.seg_ws);
    int* counts = reinterpret_cast<int*>(segs + (int64_t)cfg.seg_cap * npix);
    if (K == KIND_LBVH_BRICK && !(cfg.opts & 4))
      launch_segments_brick(grid, st, v, ix, c, rows, dt, segs, counts, cfg.seg_cap, flags,
                            (cfg.opts & 16) ? 1 : 0);
    else if (K == VS_KIND_GRID && !(cfg.opts & 4))
      launch_segments_grid(grid, st, v, ix, c, rows, dt, segs, counts, cfg.seg_cap, flags);
    else if (K == VS_KIND_KD && !(cfg.opts & 4))
      k_segments_kd<<<grid, dim3(RENDER_TX, RENDER_TY), 0, st>>>(v, ix, c, rows, dt, segs,
                                                                counts, cfg.seg_cap, flags);
    else if (K == VS_KIND_HYBRID && !(cfg.opts & 4))
      launch_segments_hybrid(grid, st, v, ix, c, rows, dt, segs, counts, cfg.seg_cap, flags);
    else
      k_segments<K><<<grid, dim3(RENDER_TX, RENDER_TY), 0, st>>>(v, ix, c, rows, dt, segs,
                                                                 counts, cfg.seg_cap, flags,
                                                                 cfg.trav_budget);
    const bool idx32 = (int64_t)v.nx * v.ny * v.nz < (1LL << 32), ert = cfg.ert_a <= 1.0;
    // k_integrate_segments' rays exist (RO_FP64_BINS: all rays to the fallback kernel)
    const bool lean = !v.field && v.quads && !nearest && !(cfg.opts & 2);
    if (lean) {
#define VS_INTEGRATE(I32, E)                                                                  \
  k_integrate_segments<K, I32, E><<<grid, dim3(RENDER_TX, RENDER_TY), 0, st>>>(               \
      v, ix, c, lut, corr, dt, rows, segs, counts, cfg.seg_cap, rgba8, rgba64, samples, total,  \
      flags, cfg.ert_a)
      if (idx32) {
        if (ert) VS_INTEGRATE(true, true); else VS_INTEGRATE(true, false);
      } else {
        if (ert) VS_INTEGRATE(false, true); else VS_INTEGRATE(false, false);
      }
#undef VS_INTEGRATE
    }
    else if (ert)
      k_integrate_fallback<K, true><<<grid, dim3(RENDER_TX, RENDER_TY), 0, st>>>(
          v, ix, c, lut, corr, dt, nearest, rows, segs, counts, cfg.seg_cap, rgba8, rgba64,
          samples, total, flags, cfg.opts, cfg.ert_a);
    else
      k_integrate_fallback<K, false><<<grid, dim3(RENDER_TX, RENDER_TY), 0, st>>>(
          v, ix, c, lut, corr, dt, nearest, rows, segs, counts, cfg.seg_cap, rgba8, rgba64,
          samples, total, flags, cfg.opts, cfg.ert_a);
    return;
  }
  k_render<K><<<grid, dim3(RENDER_TX, RENDER_TY), 0, st>>>(v, ix, c, lut, corr, dt, nearest, rows,
                                                          rgba8, rgba64, samples, total, flags,
                                                          cfg.trav_budget, cfg.sample_budget,
                                                          cfg.opts, cfg.ert_a);
}

}  // namespace vs

using namespace vs;

extern "C" {

size_t vs_render_workspace(int64_t npix, int seg_cap) {
  if (npix <= 0 || seg_cap <= 0) return 0;
  return (size_t)npix * seg_cap * 8 + (size_t)npix * 4 + 512;
}

int vs_render(const vs_volume_desc* vol, const vs_index_desc* ix, const vs_camera_desc* cam,
              const float* lut, const double* corr, double dt, int nearest,
              const vs_rows_desc* rows_opt, uint8_t* rgba8, double* rgba64_opt,
              int32_t* samples_opt, unsigned long long* total_opt, int* flags, void* ws,
              size_t ws_bytes, int seg_cap, const vs_render_opts* opts, vs_stream_t stream) {
  if (!vol || !ix || !cam || !lut || !corr || !rgba8 || !flags || !(dt > 0.0))
    return fail_arg("vs_render");
  if (!vol->bins || vol->nx < 1 || vol->ny < 1 || vol->nz < 1) return fail_arg("vs_render: volume");
  if (cam->width < 1 || cam->height < 1) return fail_arg("vs_render: viewport");
  vs_rows_desc rows;
  if (rows_opt) {
    rows = *rows_opt;
  } else {
    rows.nrows = cam->height; rows.stripe = cam->height > 0 ? cam->height : 1;
    rows.nparts = 1; rows.part = 0;
  }
  if (rows.stripe < 1 || rows.nparts < 1 || rows.part < 0 || rows.part >= rows.nparts)
    return fail_arg("vs_render: rows");
  if (rows.nrows <= 0) return 0;
  const int kind = ix->kind;
  if ((kind == VS_KIND_GRID || kind == VS_KIND_HYBRID) && (!ix->occ || ix->cs < 1))
    return fail_arg("vs_render: grid");
  if ((kind == VS_KIND_LBVH || kind == VS_KIND_KD || kind == VS_KIND_HYBRID) &&
      (!ix->lo || !ix->hi || !ix->left || !ix->right))
    return fail_arg("vs_render: tree");
  if ((kind == VS_KIND_KD || kind == VS_KIND_HYBRID) && (!ix->axis || !ix->plane))
    return fail_arg("vs_render: kd");
  dim3 grid((unsigned)cdiv(cam->width, RENDER_TX), (unsigned)cdiv(rows.nrows, RENDER_TY));
  cudaStream_t st = S(stream);
  const int64_t npix = (int64_t)rows.nrows * cam->width;
  RenderCfg cfg = render_cfg(opts);
  if (ws && seg_cap > 0) {
    if (ws_bytes < vs_render_workspace(npix, seg_cap)) return VS_EWORKSPACE;
    if ((reinterpret_cast<uintptr_t>(ws) & 15) != 0) return fail_arg("vs_render: ws alignment");
    cfg.seg_ws = ws;
    cfg.seg_cap = seg_cap;
  }
  switch (kind) {
    case VS_KIND_NAIVE:
      launch_render<VS_KIND_NAIVE>(grid, st, *vol, *ix, *cam, lut, corr, dt, nearest, rows, rgba8,
                                   rgba64_opt, samples_opt, total_opt, flags, cfg);
      break;
    case VS_KIND_GRID:
      launch_render<VS_KIND_GRID>(grid, st, *vol, *ix, *cam, lut, corr, dt, nearest, rows, rgba8,
                                  rgba64_opt, samples_opt, total_opt, flags, cfg);
      break;
    case VS_KIND_LBVH:
      if (ix->brick_bits)
        launch_render<KIND_LBVH_BRICK>(grid, st, *vol, *ix, *cam, lut, corr, dt, nearest, rows,
                                       rgba8, rgba64_opt, samples_opt, total_opt, flags, cfg);
      else
      launch_render<VS_KIND_LBVH>(grid, st, *vol, *ix, *cam, lut, corr, dt, nearest, rows, rgba8,
                                  rgba64_opt, samples_opt, total_opt, flags, cfg);
      break;
    case VS_KIND_KD:
      launch_render<VS_KIND_KD>(grid, st, *vol, *ix, *cam, lut, corr, dt, nearest, rows, rgba8,
                                rgba64_opt, samples_opt, total_opt, flags, cfg);
      break;
    case VS_KIND_HYBRID:
      launch_render<VS_KIND_HYBRID>(grid, st, *vol, *ix, *cam, lut, corr, dt, nearest, rows, rgba8,
                                    rgba64_opt, samples_opt, total_opt, flags, cfg);
      break;
    default:
      return fail_arg("vs_render: kind");
  }
  return check_launch("k_render");
}

int64_t vs_quads_words(int nx, int ny, int nz) {
  if (nx < 1 || ny < 1 || nz < 1) return -1;
  return QuadGeom::words(nx, ny, nz);
}

int vs_build_quads(const uint8_t* bins, int nx, int ny, int nz, uint32_t* quads,
                   vs_stream_t stream) {
  if (!bins || !quads || nx < 1 || ny < 1 || nz < 1) return fail_arg("vs_build_quads");
  if (QuadGeom::words(nx, ny, nz) >= (1LL << 32)) return fail_arg("vs_build_quads: size");
  const int64_t n = (int64_t)nx * ny * nz;
  k_build_quads<<<(unsigned)cdiv(n, 256), 256, 0, S(stream)>>>(bins, nx, ny, nz, quads);
  return check_launch("k_build_quads");
}

int vs_render_segments(const vs_volume_desc* vol, const vs_index_desc* ix,
                       const vs_camera_desc* cam, double dt, const vs_rows_desc* rows_opt,
                       int2_t* segs, int* counts, int cap, int* flags,
                       const vs_render_opts* opts, vs_stream_t stream) {
  if (!vol || !ix || !cam || !segs || !counts || !flags || cap < 1 || !(dt > 0.0))
    return fail_arg("vs_render_segments");
  const RenderCfg cfg = render_cfg(opts);
  vs_rows_desc rows;
  if (rows_opt) rows = *rows_opt;
  else { rows.nrows = cam->height; rows.stripe = cam->height; rows.nparts = 1; rows.part = 0; }
  if (rows.nrows <= 0) return 0;
  dim3 grid((unsigned)cdiv(cam->width, RENDER_TX), (unsigned)cdiv(rows.nrows, RENDER_TY));
  cudaStream_t st = S(stream);
  int2* sg = reinterpret_cast<int2*>(segs);
  switch (ix->kind) {
    case VS_KIND_NAIVE:
      k_segments<VS_KIND_NAIVE><<<grid, dim3(RENDER_TX, RENDER_TY), 0, st>>>(
          *vol, *ix, *cam, rows, dt, sg, counts, cap, flags, cfg.trav_budget);
      break;
    case VS_KIND_GRID:
      if (!(cfg.opts & 4))
        launch_segments_grid(grid, st, *vol, *ix, *cam, rows, dt, sg, counts, cap, flags);
      else
        k_segments<VS_KIND_GRID><<<grid, dim3(RENDER_TX, RENDER_TY), 0, st>>>(
            *vol, *ix, *cam, rows, dt, sg, counts, cap, flags, cfg.trav_budget);
      break;
    case VS_KIND_LBVH:
      if (ix->brick_bits && !(cfg.opts & 4))
        launch_segments_brick(grid, st, *vol, *ix, *cam, rows, dt, sg, counts, cap, flags,
                              (cfg.opts & 16) ? 1 : 0);
      else if (ix->brick_bits)
        k_segments<KIND_LBVH_BRICK><<<grid, dim3(RENDER_TX, RENDER_TY), 0, st>>>(
            *vol, *ix, *cam, rows, dt, sg, counts, cap, flags, cfg.trav_budget);
      else
        k_segments<VS_KIND_LBVH><<<grid, dim3(RENDER_TX, RENDER_TY), 0, st>>>(
            *vol, *ix, *cam, rows, dt, sg, counts, cap, flags, cfg.trav_budget);
      break;
    case VS_KIND_KD:
      if (!(cfg.opts & 4))
        k_segments_kd<<<grid, dim3(RENDER_TX, RENDER_TY), 0, st>>>(*vol, *ix, *cam, rows, dt, sg,
                                                                counts, cap, flags);
      else
        k_segments<VS_KIND_KD><<<grid, dim3(RENDER_TX, RENDER_TY), 0, st>>>(
            *vol, *ix, *cam, rows, dt, sg, counts, cap, flags, cfg.trav_budget);
      break;
    case VS_KIND_HYBRID:
      if (!(cfg.opts & 4))
        launch_segments_hybrid(grid, st, *vol, *ix, *cam, rows, dt, sg, counts, cap, flags);
      else
        k_segments<VS_KIND_HYBRID><<<grid, dim3(RENDER_TX, RENDER_TY), 0, st>>>(
            *vol, *ix, *cam, rows, dt, sg, counts, cap, flags, cfg.trav_budget);
      break;
    default:
      return fail_arg("vs_render_segments: kind");
  }
  return check_launch("k_segments");
}

int vs_lbvh_brick_grid(const int32_t* brick_coords, const int* n_dev, int64_t cap, int nbx,
                       int nby, int nbz, uint32_t* bits, vs_stream_t stream) {
  if (!brick_coords || !bits || nbx < 1 || nby < 1 || nbz < 1 || cap < 0)
    return fail_arg("vs_lbvh_brick_grid");
  const int64_t nwords = ((int64_t)nbx * nby * nbz + 31) / 32;
  VS_CUDA(cudaMemsetAsync(bits, 0, nwords * 4, S(stream)), "memset brick grid");
  if (cap == 0) return 0;
  k_brick_grid<<<(unsigned)cdiv(cap, 256), 256, 0, S(stream)>>>(brick_coords, n_dev, cap, nby,
                                                                 nbz, bits);
  return check_launch("k_brick_grid");
}

int vs_traverse_rays(const vs_index_desc* ix, int nx, int ny, int nz, const double* origins,
                     const double* dir, int nrays, double* out, int cap, int* counts, int* flags,
                     vs_stream_t stream) {
  if (!ix || !origins || !dir || !out || !counts || !flags || nrays < 0 || cap < 1)
    return fail_arg("vs_traverse_rays");
  if (nrays == 0) return 0;
  k_traverse_rays<<<(unsigned)cdiv(nrays, 64), 64, 0, S(stream)>>>(*ix, nx, ny, nz, origins, dir,
                                                                    nrays, out, cap, counts, flags);
  return check_launch("k_traverse_rays");
}

int vs_integrate_rays(const vs_volume_desc* vol, const double* origins, const double* dir,
                      const double* segs, const int* counts, int cap, int nrays, const float* lut,
                      const double* corr, double dt, int nearest, double* rgba,
                      long long* samples, vs_stream_t stream) {
  if (!vol || !origins || !dir || !segs || !counts || !lut || !corr || !rgba || !samples ||
      nrays < 0 || cap < 1 || !(dt > 0.0))
    return fail_arg("vs_integrate_rays");
  if (nrays == 0) return 0;
  k_integrate_rays<<<(unsigned)cdiv(nrays, 64), 64, 0, S(stream)>>>(
      *vol, origins, dir, segs, counts, cap, nrays, lut, corr, dt, nearest, rgba, samples);
  return check_launch("k_integrate_rays");
}

}  // extern "C"
