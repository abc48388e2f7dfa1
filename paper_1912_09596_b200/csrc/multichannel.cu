// Multi-channel volumes (BASELINE.json configs[4]: a 1024^3 volume with 4 channels, one TF per
// channel).  The reference has no multi-channel path (SPEC.md:125 non-goal); the semantics
// here reduce EXACTLY to the reference when every channel but one has zero alpha:
//   classification  visible <=> any channel's TF gives alpha > 0; the 27-bit brick summaries
//                   of the channels are OR'ed (the summary of a union is the OR of summaries),
//                   so one dilated hierarchy serves all channels;
//   compositing     at each lattice sample the channels are composited in channel order with
//                   the reference's update, w = (1 - A) * corr_c, C += w * rgb_c, A += w, for
//                   every channel with alpha > 0 (render.py:750-757 per channel).
// The renderer is the two-phase one: k_segments (shared with single channel) stores each ray's
// lattice ranges; k_integrate_multi<NCH> samples every channel per lattice point from the
// channel-interleaved gather volume (two vector loads per sample for all channels).
#include "common.cuh"

namespace vs {

constexpr int MC_MAX = 4;
// Samples the gathers run ahead of the shading (1 or 2; 2 measured 4-11% faster on the B200).
#ifndef VS_MC_PREFETCH
#define VS_MC_PREFETCH 2
#endif
constexpr int MC_TX = 8, MC_TY = 16;  // warp = 8 x 4 pixels, as the single-channel tiles

__global__ void k_or_words(uint32_t* __restrict__ dst, const uint32_t* __restrict__ src,
                           int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] |= src[i];
}

struct McSmem {
  float4 lut[MC_MAX][256];
  double corr[MC_MAX][256];
  float u8f[256];
};

__device__ __forceinline__ bool mc_slab(double ox, double oy, double oz, double ix, double iy,
                                        double iz, bool zx, bool zy, bool zz, double hx, double hy,
                                        double hz, double& t0, double& t1) {
  double tmin = -1e300, tmax = 1e300;
  const double o[3] = {ox, oy, oz}, inv[3] = {ix, iy, iz}, h[3] = {hx, hy, hz};
  const bool z[3] = {zx, zy, zz};
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    if (z[a]) {
      if (o[a] < 0.0 || o[a] >= h[a]) return false;
    } else {
      double ta = __dmul_rn(0.0 - o[a], inv[a]), tb = __dmul_rn(h[a] - o[a], inv[a]);
      if (ta > tb) { double t = ta; ta = tb; tb = t; }
      if (ta > tmin) tmin = ta;
      if (tb < tmax) tmax = tb;
    }
  }
  if (tmax <= tmin) return false;
  t0 = tmin;
  t1 = tmax;
  return true;
}

// Interleaved trilinear gather volume of all channels: per voxel W words (W = 1, 2 or 4),
// word c = channel c's packed (y,z) 2x2 quad (the vs_build_quads layout).  A multi-channel
// sample then needs two vector loads (x0 and x1 planes) instead of 2 * nch scalar loads.
template <int W>
__global__ void k_build_mquads(const uint8_t* __restrict__ b0, const uint8_t* __restrict__ b1,
                               const uint8_t* __restrict__ b2, const uint8_t* __restrict__ b3,
                               int nch, int nx, int ny, int nz, uint32_t* __restrict__ q) {
  const int64_t n = (int64_t)nx * ny * nz;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int z = (int)(i % nz);
  const int y = (int)((i / nz) % ny);
  const int x = (int)(i / ((int64_t)ny * nz));
  const int64_t dz = z + 1 < nz ? 1 : 0, dy = y + 1 < ny ? nz : 0;
  const uint8_t* bs[4] = {b0, b1, b2, b3};
  const QuadGeom qg(nx, ny, nz);  // the single-channel gather volume's tiling (common.cuh)
  const int64_t o = qg.at(x, qg.yz(y, z));
  uint32_t w[4] = {0, 0, 0, 0};
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    if (c < nch) {
      const uint8_t* b = bs[c];
      w[c] = (uint32_t)b[i] | ((uint32_t)b[i + dz] << 8) | ((uint32_t)b[i + dy] << 16) |
             ((uint32_t)b[i + dy + dz] << 24);
    }
  }
  if (W == 4) reinterpret_cast<uint4*>(q)[o] = make_uint4(w[0], w[1], w[2], w[3]);
  else if (W == 2) reinterpret_cast<uint2*>(q)[o] = make_uint2(w[0], w[1]);
  else q[o] = w[0];
}

// One sample's gathered quads of every channel at the x0 and x1 planes.
template <int NCH>
struct McGather {
  uint32_t w0[NCH], w1[NCH];
  uint32_t fix;  // lazy border fix-ups (bit 0: y0 clamped below, bit 1: z0): mc_settle
  double fx, fy, fz;
};

template <int NCH>
__device__ __forceinline__ void mc_gather(const vs_multi_desc& md, double ox, double oy, double oz,
                                          double dx, double dy, double dz, double t,
                                          McGather<NCH>& g) {
  const int nx = md.nx, ny = md.ny, nz = md.nz;
  const double px = __dadd_rn(ox, __dmul_rn(t, dx));
  const double py = __dadd_rn(oy, __dmul_rn(t, dy));
  const double pz = __dadd_rn(oz, __dmul_rn(t, dz));
  const double qx = px - 0.5, qy = py - 0.5, qz = pz - 0.5;
  const double flx = floor(qx), fly = floor(qy), flz = floor(qz);
  g.fx = qx - flx; g.fy = qy - fly; g.fz = qz - flz;
  const int x0r = (int)flx, y0r = (int)fly, z0r = (int)flz;
  const int x0 = min(max(x0r, 0), nx - 1), x1 = min(max(x0r + 1, 0), nx - 1);
  const int y0 = min(max(y0r, 0), ny - 1), z0 = min(max(z0r, 0), nz - 1);
  const QuadGeom qg(nx, ny, nz);
  const uint32_t yzw = qg.yz(y0, z0);
  const uint32_t o0 = qg.at(x0, yzw), o1 = qg.at(x1, yzw);
  if constexpr (NCH >= 3) {
    const uint4 a = __ldg(reinterpret_cast<const uint4*>(md.mquads) + o0);
    const uint4 b = __ldg(reinterpret_cast<const uint4*>(md.mquads) + o1);
    const uint32_t aw[4] = {a.x, a.y, a.z, a.w}, bw[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
    for (int c = 0; c < NCH; ++c) { g.w0[c] = aw[c]; g.w1[c] = bw[c]; }
  } else if constexpr (NCH == 2) {
    const uint2 a = __ldg(reinterpret_cast<const uint2*>(md.mquads) + o0);
    const uint2 b = __ldg(reinterpret_cast<const uint2*>(md.mquads) + o1);
    g.w0[0] = a.x; g.w0[1] = a.y; g.w1[0] = b.x; g.w1[1] = b.y;
  } else {
    g.w0[0] = __ldg(reinterpret_cast<const uint32_t*>(md.mquads) + o0);
    g.w1[0] = __ldg(reinterpret_cast<const uint32_t*>(md.mquads) + o1);
  }
  g.fix = (y0r < 0 ? 1u : 0u) | (z0r < 0 ? 2u : 0u);
}

// clamped low borders: the +1 neighbour is the voxel itself (applied when the sample is
// consumed, so the gather's loads complete under the previous sample's shading)
template <int NCH>
__device__ __forceinline__ void mc_settle(McGather<NCH>& g) {
#pragma unroll
  for (int c = 0; c < NCH; ++c) {
    if (g.fix & 1u) { g.w0[c] = __byte_perm(g.w0[c], 0, 0x1010); g.w1[c] = __byte_perm(g.w1[c], 0, 0x1010); }
    if (g.fix & 2u) { g.w0[c] = __byte_perm(g.w0[c], 0, 0x2200); g.w1[c] = __byte_perm(g.w1[c], 0, 0x2200); }
  }
}

#ifndef VS_MC_MINB
#define VS_MC_MINB 1
#endif
template <int NCH>
__global__ void __launch_bounds__(MC_TX* MC_TY, VS_MC_MINB)
    k_integrate_multi(vs_multi_desc md, vs_camera_desc cam, double dt, vs_rows_desc rows,
                      const int2* __restrict__ segs, const int* __restrict__ counts, int cap,
                      uint8_t* __restrict__ rgba8, double* __restrict__ rgba64,
                      int32_t* __restrict__ samples, unsigned long long* __restrict__ total,
                      int* __restrict__ flags_out) {
  __shared__ McSmem sm;
  const int tid = threadIdx.y * MC_TX + threadIdx.x;
  for (int k = tid; k < 256; k += MC_TX * MC_TY) {
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
      const float* L = md.lut[c];
      sm.lut[c][k] = make_float4(L[4 * k], L[4 * k + 1], L[4 * k + 2], L[4 * k + 3]);
      sm.corr[c][k] = md.corr[c][k];
    }
    sm.u8f[k] = (float)((double)k / 255.0);
  }
  __syncthreads();
  const int i = blockIdx.x * MC_TX + threadIdx.x;
  const int l = blockIdx.y * MC_TY + threadIdx.y;
  int taken = 0;
  if (i < cam.width && l < rows.nrows) {
    const int64_t pix = (int64_t)l * cam.width + i;
    const int64_t npix = (int64_t)rows.nrows * cam.width;
    const int s = l / rows.stripe, w = l % rows.stripe;
    const int j = (s * rows.nparts + rows.part) * rows.stripe + w;
    const double xs = __dmul_rn(((double)i + 0.5) - (double)cam.width / 2.0, cam.scale);
    const double ys = __dmul_rn(((double)cam.height / 2.0 - (double)j) - 0.5, cam.scale);
    const double ox = __dadd_rn(__dadd_rn(cam.eye[0], __dmul_rn(ys, cam.up[0])), __dmul_rn(xs, cam.right[0]));
    const double oy = __dadd_rn(__dadd_rn(cam.eye[1], __dmul_rn(ys, cam.up[1])), __dmul_rn(xs, cam.right[1]));
    const double oz = __dadd_rn(__dadd_rn(cam.eye[2], __dmul_rn(ys, cam.up[2])), __dmul_rn(xs, cam.right[2]));
    const double dx = cam.dir[0], dy = cam.dir[1], dz = cam.dir[2];
    const bool zx = dx == 0.0, zy = dy == 0.0, zz = dz == 0.0;
    const double ix = zx ? 0.0 : 1.0 / dx, iy = zy ? 0.0 : 1.0 / dy, iz = zz ? 0.0 : 1.0 / dz;
    double accr = 0.0, accg = 0.0, accb = 0.0, acca = 0.0;
    const int n = counts[pix];
    double entry, ex;
    if (n > cap) atomicOr(flags_out, 4);  // caller sizes cap from the counts (no fallback here)
    if (n > 0 && n <= cap &&
        mc_slab(ox, oy, oz, ix, iy, iz, zx, zy, zz, (double)md.nx, (double)md.ny, (double)md.nz,
                entry, ex)) {
      // flat sample loop over the lattice ranges, the next sample's loads issued before the
      // current sample's interpolation and compositing
      // the ranges as one sample stream (see k_integrate_segments): next range prefetched,
      // next sample's gather issued across range ends
      int q = 0;
      int2 kr = segs[pix];
      int2 krn = n > 1 ? segs[npix + pix] : make_int2(0, 0);
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
      auto issue = [&](McGather<NCH>& g) {
        mc_gather<NCH>(md, ox, oy, oz, dx, dy, dz, __dadd_rn(entry, __dmul_rn((double)kc, dt)), g);
      };
      auto shade = [&](McGather<NCH>& g) {
        mc_settle<NCH>(g);
        // every channel's bin by the FP32 filter (common.cuh bin_fast); the rare sample with a
        // channel near a bin edge re-evaluates that channel's reference FP64 lerps
        const float fx32 = __double2float_rn(g.fx), fy32 = __double2float_rn(g.fy),
                    fz32 = __double2float_rn(g.fz);
        int bins[NCH];
        bool sure = true;
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
          bins[c] = bin_fast_bytes(g.w0[c], g.w1[c], fx32, fy32, fz32);
          sure &= bins[c] >= 0;
        }
        if (!sure) {
#pragma unroll
          for (int c = 0; c < NCH; ++c) {
            if (bins[c] >= 0) continue;
            const uint32_t w0 = g.w0[c], w1 = g.w1[c];
            const float* tb = sm.u8f;
            const float c000 = tb[w0 & 0xffu], c001 = tb[(w0 >> 8) & 0xffu];
            const float c010 = tb[(w0 >> 16) & 0xffu], c011 = tb[w0 >> 24];
            const float c100 = tb[w1 & 0xffu], c101 = tb[(w1 >> 8) & 0xffu];
            const float c110 = tb[(w1 >> 16) & 0xffu], c111 = tb[w1 >> 24];
            const float d00 = __fsub_rn(c100, c000), d10 = __fsub_rn(c110, c010);
            const float d01 = __fsub_rn(c101, c001), d11 = __fsub_rn(c111, c011);
            const double c00 = __dadd_rn((double)c000, __dmul_rn((double)d00, g.fx));
            const double c10 = __dadd_rn((double)c010, __dmul_rn((double)d10, g.fx));
            const double c01 = __dadd_rn((double)c001, __dmul_rn((double)d01, g.fx));
            const double c11 = __dadd_rn((double)c011, __dmul_rn((double)d11, g.fx));
            const double c0 = __dadd_rn(c00, __dmul_rn(c10 - c00, g.fy));
            const double c1 = __dadd_rn(c01, __dmul_rn(c11 - c01, g.fy));
            const double value = __dadd_rn(c0, __dmul_rn(c1 - c0, g.fz));
            const int bi = __double2int_rd(__dadd_rn(__dmul_rn(value, 255.0), 0.5));
            bins[c] = bi < 0 ? 0 : (bi > 255 ? 255 : bi);
          }
        }
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
          const float4 col = sm.lut[c][bins[c]];
          if (col.w > 0.0f) {
            const double wgt = __dmul_rn(1.0 - acca, sm.corr[c][bins[c]]);
            accr = __dadd_rn(accr, __dmul_rn(wgt, (double)col.x));
            accg = __dadd_rn(accg, __dmul_rn(wgt, (double)col.y));
            accb = __dadd_rn(accb, __dmul_rn(wgt, (double)col.z));
            acca = __dadd_rn(acca, wgt);
          }
        }
        ++taken;
      };
#if VS_MC_PREFETCH >= 2
      // two samples ahead in three rotating slots (no copies of loaded registers)
      McGather<NCH> g0, g1, g2;
      issue(g0);
      bool h1 = advance(), h2 = false, h0 = true;
      if (h1) issue(g1);
      while (true) {
        h2 = h1 && advance();
        if (h2) issue(g2);
        shade(g0);
        if (!h1) break;
        h0 = h2 && advance();
        if (h0) issue(g0);
        shade(g1);
        if (!h2) break;
        h1 = h0 && advance();
        if (h1) issue(g1);
        shade(g2);
        if (!h0) break;
      }
#else
      // one sample ahead in two rotating slots (no copies of loaded registers)
      McGather<NCH> g0, g1;
      issue(g0);
      while (true) {
        const bool h1 = advance();
        if (h1) issue(g1);
        shade(g0);
        if (!h1) break;
        const bool h0 = advance();
        if (h0) issue(g0);
        shade(g1);
        if (!h0) break;
      }
#endif
    }
    const double acc[4] = {accr, accg, accb, acca};
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const double qq = floor(__dadd_rn(__dmul_rn(acc[c], 255.0), 0.5));
      rgba8[4 * pix + c] = (uint8_t)(qq < 0.0 ? 0 : (qq > 255.0 ? 255 : (int)qq));
      if (rgba64) rgba64[4 * pix + c] = acc[c];
    }
    if (samples) samples[pix] = taken;
  }
  if (total) {
    unsigned long long t = (unsigned long long)taken;
    for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if ((tid & 31) == 0 && t) atomicAdd(total, t);
  }
}

}  // namespace vs

using namespace vs;

extern "C" {

int vs_or_words(uint32_t* dst, const uint32_t* src, int64_t n, vs_stream_t stream) {
  if (!dst || !src || n < 0) return fail_arg("vs_or_words");
  if (n == 0) return 0;
  k_or_words<<<(unsigned)cdiv(n, 256), 256, 0, S(stream)>>>(dst, src, n);
  return check_launch("k_or_words");
}

int vs_render_multi_integrate(const vs_multi_desc* md, const vs_camera_desc* cam, double dt,
                              const vs_rows_desc* rows_opt, const int2_t* segs, const int* counts,
                              int cap, uint8_t* rgba8, double* rgba64_opt, int32_t* samples_opt,
                              unsigned long long* total_opt, int* flags, vs_stream_t stream) {
  if (!md || !cam || !segs || !counts || !rgba8 || !flags || !(dt > 0.0) || md->nch < 1 ||
      md->nch > MC_MAX)
    return fail_arg("vs_render_multi_integrate");
  for (int c = 0; c < md->nch; ++c)
    if (!md->lut[c] || !md->corr[c]) return fail_arg("vs_render_multi: channel");
  if (!md->mquads) return fail_arg("vs_render_multi: interleaved gather volume (vs_build_mquads)");
  if ((int64_t)md->nx * md->ny * md->nz >= (1LL << 32)) return fail_arg("vs_render_multi: size");
  vs_rows_desc rows;
  if (rows_opt) rows = *rows_opt;
  else { rows.nrows = cam->height; rows.stripe = cam->height; rows.nparts = 1; rows.part = 0; }
  if (rows.nrows <= 0) return 0;
  dim3 grid((unsigned)cdiv(cam->width, MC_TX), (unsigned)cdiv(rows.nrows, MC_TY));
  const int2* sg = reinterpret_cast<const int2*>(segs);
  switch (md->nch) {
#define VS_MC_LAUNCH(K)                                                                  \
  case K:                                                                                \
    k_integrate_multi<K><<<grid, dim3(MC_TX, MC_TY), 0, S(stream)>>>(                    \
        *md, *cam, dt, rows, sg, counts, cap, rgba8, rgba64_opt, samples_opt, total_opt, \
        flags);                                                                          \
    break;
    VS_MC_LAUNCH(1)
    VS_MC_LAUNCH(2)
    VS_MC_LAUNCH(3)
    VS_MC_LAUNCH(4)
#undef VS_MC_LAUNCH
  }
  return check_launch("k_integrate_multi");
}

int vs_mquads_words(int nch) { return nch <= 1 ? 1 : (nch == 2 ? 2 : 4); }

int64_t vs_mquads_size(int nch, int nx, int ny, int nz) {
  if (nch < 1 || nch > MC_MAX || nx < 1 || ny < 1 || nz < 1) return -1;
  return QuadGeom::words(nx, ny, nz) * vs_mquads_words(nch);
}

int vs_build_mquads(const uint8_t* const* bins, int nch, int nx, int ny, int nz, uint32_t* out,
                    vs_stream_t stream) {
  if (!bins || !out || nch < 1 || nch > MC_MAX || nx < 1 || ny < 1 || nz < 1)
    return fail_arg("vs_build_mquads");
  if (QuadGeom::words(nx, ny, nz) >= (1LL << 32)) return fail_arg("vs_build_mquads: size");
  for (int c = 0; c < nch; ++c)
    if (!bins[c]) return fail_arg("vs_build_mquads: channel");
  const uint8_t* b[4] = {bins[0], nch > 1 ? bins[1] : nullptr, nch > 2 ? bins[2] : nullptr,
                         nch > 3 ? bins[3] : nullptr};
  const int64_t n = (int64_t)nx * ny * nz;
  const unsigned g = (unsigned)cdiv(n, 256);
  switch (vs_mquads_words(nch)) {
    case 1: k_build_mquads<1><<<g, 256, 0, S(stream)>>>(b[0], b[1], b[2], b[3], nch, nx, ny, nz, out); break;
    case 2: k_build_mquads<2><<<g, 256, 0, S(stream)>>>(b[0], b[1], b[2], b[3], nch, nx, ny, nz, out); break;
    default: k_build_mquads<4><<<g, 256, 0, S(stream)>>>(b[0], b[1], b[2], b[3], nch, nx, ny, nz, out); break;
  }
  return check_launch("k_build_mquads");
}

}  // extern "C"
