// Summed-volume tables and box queries over the packed bit volume.
//
//   build_svt_grid (svt.py:40-57): per brick of edge bs, a zero-bordered (bs+1)^3 uint32 table,
//     T[i][j][k] = number of set flags in the brick-local box [0,i)x[0,j)x[0,k); padded bricks
//     count zeros.  k_svt_build stages one brick's table in shared memory (33^3 words at
//     bs = 32) and runs the three prefix scans there: z via popcount of masked words, then y,
//     then x; the table leaves in one coalesced write.
//   box_count (svt.py:65-90): 8-term inclusion-exclusion per overlapped brick (k_box_count).
//   shrink_to_occupied (svt.py:100-131): the minimal box holding every flag of the box; the
//     binary searches over monotone slab counts find exactly the flags' bounding box, which
//     k_tight_box reads straight from the bits.
#include <algorithm>

#include "common.cuh"

namespace vs {

__global__ void k_svt_build(const uint32_t* __restrict__ bits, int nx, int ny, int nz, int bs,
                            int nbx, int nby, int nbz, uint32_t* __restrict__ tables) {
  extern __shared__ uint32_t T[];
  const int e = bs + 1;
  const int64_t brick = blockIdx.x;
  const int bz = (int)(brick % nbz), by = (int)((brick / nbz) % nby),
            bx = (int)(brick / ((int64_t)nbz * nby));
  const int nzw = (int)nzw_of(nz);
  const int tot = e * e * e;
  for (int q = threadIdx.x; q < tot; q += blockDim.x) T[q] = 0;
  __syncthreads();
  const int z0 = bz * bs;
  // z prefix per (i, j) row
  for (int q = threadIdx.x; q < bs * bs; q += blockDim.x) {
    const int i = q / bs, j = q % bs;
    const int x = bx * bs + i, y = by * bs + j;
    uint32_t* out = T + ((i + 1) * e + (j + 1)) * e;
    if (x >= nx || y >= ny) continue;
    const uint32_t* row = bits + ((int64_t)x * ny + y) * nzw;
    int run = 0;
    for (int k0 = 0; k0 < bs; k0 += 32) {
      const int gz = z0 + k0;
      uint32_t v = 0;
      if (gz < nz) {
        const int gw = gz >> 5, sh = gz & 31;
        v = __ldg(row + gw) >> sh;
        if (sh && gw + 1 < nzw) v |= __ldg(row + gw + 1) << (32 - sh);
        const int rem = nz - gz;
        if (rem < 32) v &= (1u << rem) - 1u;
      }
      const int kn = min(32, bs - k0);
      if (kn < 32) v &= (1u << kn) - 1u;
      for (int k = 0; k < kn; ++k) {
        run += (v >> k) & 1u;
        out[k0 + k + 1] = run;
      }
    }
  }
  __syncthreads();
  // y prefix
  for (int q = threadIdx.x; q < e * e; q += blockDim.x) {
    const int i = q / e, k = q % e;
    uint32_t run = 0;
    for (int j = 0; j < e; ++j) {
      run += T[(i * e + j) * e + k];
      T[(i * e + j) * e + k] = run;
    }
  }
  __syncthreads();
  // x prefix
  for (int q = threadIdx.x; q < e * e; q += blockDim.x) {
    const int j = q / e, k = q % e;
    uint32_t run = 0;
    for (int i = 0; i < e; ++i) {
      run += T[(i * e + j) * e + k];
      T[(i * e + j) * e + k] = run;
    }
  }
  __syncthreads();
  uint32_t* dst = tables + brick * (int64_t)tot;
  for (int q = threadIdx.x; q < tot; q += blockDim.x) dst[q] = T[q];
}

// box_count for a batch of boxes (clipped to dims); one warp per box over its bricks.
__global__ void k_box_count(const uint32_t* __restrict__ tables, int nx, int ny, int nz, int bs,
                            int nby, int nbz, const int32_t* __restrict__ boxes, int nbox,
                            long long* __restrict__ counts) {
  const int lane = threadIdx.x & 31;
  const int q = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (q >= nbox) return;
  int lo[3], hi[3];
  const int dims[3] = {nx, ny, nz};
  bool empty = false;
  for (int a = 0; a < 3; ++a) {
    lo[a] = max(boxes[6 * q + a], 0);
    hi[a] = min(boxes[6 * q + 3 + a], dims[a]);
    empty |= lo[a] >= hi[a];
  }
  long long total = 0;
  if (!empty) {
    const int e = bs + 1;
    const int b0[3] = {lo[0] / bs, lo[1] / bs, lo[2] / bs};
    const int b1[3] = {(hi[0] - 1) / bs, (hi[1] - 1) / bs, (hi[2] - 1) / bs};
    const int n1 = b1[1] - b0[1] + 1, n2 = b1[2] - b0[2] + 1;
    const int64_t nb = (int64_t)(b1[0] - b0[0] + 1) * n1 * n2;
    for (int64_t t = lane; t < nb; t += 32) {
      const int cx = b0[0] + (int)(t / ((int64_t)n1 * n2));
      const int cy = b0[1] + (int)((t / n2) % n1);
      const int cz = b0[2] + (int)(t % n2);
      const int c[3] = {cx, cy, cz};
      int l[3], h[3];
      for (int a = 0; a < 3; ++a) {
        l[a] = min(max(lo[a] - c[a] * bs, 0), bs);
        h[a] = min(max(hi[a] - c[a] * bs, 0), bs);
      }
      const uint32_t* T = tables + (((int64_t)cx * nby + cy) * nbz + cz) * e * e * e;
      auto at = [&](int i, int j, int k) -> long long { return T[((int64_t)i * e + j) * e + k]; };
      total += at(h[0], h[1], h[2]) - at(l[0], h[1], h[2]) - at(h[0], l[1], h[2]) -
               at(h[0], h[1], l[2]) + at(l[0], l[1], h[2]) + at(l[0], h[1], l[2]) +
               at(h[0], l[1], l[2]) - at(l[0], l[1], l[2]);
    }
    for (int o = 16; o; o >>= 1) total += __shfl_xor_sync(0xffffffffu, total, o);
  }
  if (lane == 0) counts[q] = total;
}

// Tight box of the set bits inside one box (shrink_to_occupied), block-wide reduction.
__global__ void k_tight_box(const uint32_t* __restrict__ bits, int nx, int ny, int nz,
                            const int32_t* __restrict__ box, int* __restrict__ out) {
  const int nzw = (int)nzw_of(nz);
  const int x0 = max(box[0], 0), y0 = max(box[1], 0), z0 = max(box[2], 0);
  const int x1 = min(box[3], nx), y1 = min(box[4], ny), z1 = min(box[5], nz);
  if (x0 >= x1 || y0 >= y1 || z0 >= z1) return;
  const int64_t nrows = (int64_t)(x1 - x0) * (y1 - y0);
  int lo[3] = {0x3fffffff, 0x3fffffff, 0x3fffffff}, hi[3] = {-1, -1, -1};
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < nrows;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int x = x0 + (int)(r / (y1 - y0)), y = y0 + (int)(r % (y1 - y0));
    const uint32_t* row = bits + ((int64_t)x * ny + y) * nzw;
    int zf = -1, zl = -1;
    for (int w = z0 >> 5; w <= (z1 - 1) >> 5; ++w) {
      uint32_t v = __ldg(row + w);
      const int wb = 32 * w;
      if (wb < z0) v &= 0xffffffffu << (z0 - wb);
      if (z1 - wb < 32) v &= (1u << (z1 - wb)) - 1u;
      if (v) {
        if (zf < 0) zf = wb + __ffs(v) - 1;
        zl = wb + 31 - __clz(v);
      }
    }
    if (zf >= 0) {
      lo[0] = min(lo[0], x); hi[0] = max(hi[0], x);
      lo[1] = min(lo[1], y); hi[1] = max(hi[1], y);
      lo[2] = min(lo[2], zf); hi[2] = max(hi[2], zl);
    }
  }
  for (int k = 0; k < 3; ++k)
    for (int o = 16; o; o >>= 1) {
      lo[k] = min(lo[k], __shfl_xor_sync(0xffffffffu, lo[k], o));
      hi[k] = max(hi[k], __shfl_xor_sync(0xffffffffu, hi[k], o));
    }
  if ((threadIdx.x & 31) == 0 && hi[0] >= 0)
    for (int k = 0; k < 3; ++k) { atomicMin(out + k, lo[k]); atomicMax(out + 3 + k, hi[k] + 1); }
}

}  // namespace vs

using namespace vs;

extern "C" {

int vs_svt_build(const uint32_t* bits, int nx, int ny, int nz, int bs, uint32_t* tables,
                 vs_stream_t stream) {
  if (!bits || !tables || nx < 1 || ny < 1 || nz < 1 || bs < 2) return fail_arg("vs_svt_build");
  if (bs > 32) return fail_arg("vs_svt_build: brick_size > 32");
  const int nbx = (int)cdiv(nx, bs), nby = (int)cdiv(ny, bs), nbz = (int)cdiv(nz, bs);
  const size_t smem = (size_t)(bs + 1) * (bs + 1) * (bs + 1) * 4;
  VS_CUDA(cudaFuncSetAttribute(k_svt_build, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)smem),
          "smem attr");
  const int64_t nb = (int64_t)nbx * nby * nbz;
  k_svt_build<<<(unsigned)nb, 256, smem, S(stream)>>>(bits, nx, ny, nz, bs, nbx, nby, nbz,
                                                      tables);
  return check_launch("k_svt_build");
}

int vs_box_count(const uint32_t* tables, int nx, int ny, int nz, int bs, const int32_t* boxes,
                 int nbox, long long* counts, vs_stream_t stream) {
  if (!tables || !boxes || !counts || nbox < 0 || bs < 2) return fail_arg("vs_box_count");
  if (nbox == 0) return 0;
  const int nby = (int)cdiv(ny, bs), nbz = (int)cdiv(nz, bs);
  k_box_count<<<(unsigned)cdiv(nbox, 4), 128, 0, S(stream)>>>(tables, nx, ny, nz, bs, nby, nbz,
                                                               boxes, nbox, counts);
  return check_launch("k_box_count");
}

int vs_tight_box(const uint32_t* bits, int nx, int ny, int nz, const int32_t* box, int* out,
                 vs_stream_t stream) {
  if (!bits || !box || !out) return fail_arg("vs_tight_box");
  const int init[6] = {0x3fffffff, 0x3fffffff, 0x3fffffff, -1, -1, -1};
  VS_CUDA(cudaMemcpyAsync(out, init, sizeof init, cudaMemcpyHostToDevice, S(stream)), "init");
  k_tight_box<<<148 * 4, 256, 0, S(stream)>>>(bits, nx, ny, nz, box, out);
  return check_launch("k_tight_box");
}

}  // extern "C"
