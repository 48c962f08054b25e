// K3 volume layout (zero-padded replica + 8^3 brick-max map), the per-thr
// Chebyshev brick-distance map of the exact skip, the 16-bit rescale of
// load_raw, and the K7 phantom input generator.
//
// Reference: volume.py:122-151 (load_raw), grid.py:22-31 (padded_flat),
// volume.py:317-368 + rng.py:24-51 (generate_phantom; inputs only).

#include <cstring>

#include <algorithm>

#include "vx_internal.cuh"

namespace {

// one thread per 8^3 brick; rows of 8 voxels are 8-byte aligned (origin and
// strides are multiples of 16)
__global__ void brick_max_kernel(const uint8_t* __restrict__ origin, int64_t sy, int64_t sz,
                                 int nbx, int nby, int nbz, uint8_t* __restrict__ bmax_origin,
                                 int64_t bsy, int64_t bsz) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nb = (int64_t)nbx * nby * nbz;
  if (b >= nb) return;
  const int bx = (int)(b % nbx);
  const int by = (int)((b / nbx) % nby);
  const int bz = (int)(b / ((int64_t)nbx * nby));
  uint32_t m = 0;
  const uint8_t* p0 = origin + (int64_t)bz * 8 * sz + (int64_t)by * 8 * sy + (int64_t)bx * 8;
#pragma unroll 2
  for (int z = 0; z < 8; ++z) {
#pragma unroll
    for (int y = 0; y < 8; ++y) {
      const uint2 w = __ldg(reinterpret_cast<const uint2*>(p0 + z * sz + y * sy));
      m = __vmaxu4(m, __vmaxu4(w.x, w.y));
    }
  }
  m = max(max(m & 0xffu, (m >> 8) & 0xffu), max((m >> 16) & 0xffu, m >> 24));
  bmax_origin[(int64_t)bz * bsz + (int64_t)by * bsy + bx] = (uint8_t)m;
}

// Chebyshev distance transform on the brick / cell grid, separable min-max
// passes: D(b) = min_o max_i |b_i - o_i| over occupied o = min_oz max(|dz|,
// min_oy max(|dy|, min_ox |dx|)).  Out-of-map cells are unoccupied; capped.
//
// Pass 1 (x, thresholding): the 1D distance to the nearest occupied cell of
// the row, min(cap, forward and backward sweeps) -- O(1) per cell.  Rows of
// the flattened (z, y) index are contiguous, so a block stages 64 whole rows
// with coalesced loads and each thread sweeps one row in shared memory.
// Passes 2-3 (y, z): D(l) = min_a max(v(l +- a), a) over a < cap, by two
// linear sweeps per line (dist_sweep_kernel below).  (One thread per cell on
// global memory took ~0.95 ms per pass on the 258^3 cell map of a 1024^3
// volume.)
constexpr int kRowsPerBlock = 64;

// 256 threads: the 8 warps stage / store the 64 rows (one row per warp at a
// time, lanes along x: coalesced, no per-byte index division), the first 64
// threads sweep one row each
template <int DIR>
__global__ void __launch_bounds__(256) dist_first_x_kernel(
    const uint8_t* __restrict__ src, uint8_t* __restrict__ dst, int mx, int64_t rows, int thr,
    int cap) {
  // DIR 0: two-sided (Chebyshev); +1: distance to the nearest occupied cell
  // at x' >= x (rays moving toward +x); -1: at x' <= x (orthant maps)
  extern __shared__ uint8_t rowbuf[];
  const int pitch = mx | 1;  // odd pitch: threads sweeping rows hit distinct banks
  const int64_t r0 = (int64_t)blockIdx.x * kRowsPerBlock;
  const int nr = (int)min((int64_t)kRowsPerBlock, rows - r0);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint8_t* s = src + r0 * mx;
  for (int r = warp; r < nr; r += 8)
    for (int x = lane; x < mx; x += 32) rowbuf[r * pitch + x] = s[(int64_t)r * mx + x];
  __syncthreads();
  if ((int)threadIdx.x < nr) {
    uint8_t* L = rowbuf + threadIdx.x * pitch;
    if (DIR <= 0) {
      int last = -(1 << 20);
      for (int x = 0; x < mx; ++x) {  // forward: distance to the last occupied cell
        if (L[x] >= thr) last = x;
        L[x] = (uint8_t)min(cap, x - last);
      }
    }
    if (DIR == 0) {
      int next = 1 << 20;
      for (int x = mx - 1; x >= 0; --x) {  // backward, and the minimum of both
        if (L[x] == 0) next = x;
        L[x] = (uint8_t)min((int)L[x], min(cap, next - x));
      }
    } else if (DIR > 0) {
      int next = 1 << 20;
      for (int x = mx - 1; x >= 0; --x) {  // distance to the next occupied cell
        if (L[x] >= thr) next = x;
        L[x] = (uint8_t)min(cap, next - x);
      }
    }
  }
  __syncthreads();
  uint8_t* d = dst + r0 * mx;
  for (int r = warp; r < nr; r += 8)
    for (int x = lane; x < mx; x += 32) d[(int64_t)r * mx + x] = rowbuf[r * pitch + x];
}

// Passes 2-3 as two linear sweeps per line.  Left sweep: L(l) = min over
// y <= l of max(v(y), l - y).  Writing T_w(l) = max(w, l - last[w]) with
// last[w] the latest y <= l holding value w (for a fixed w the latest
// occurrence dominates), L(l) = min_w T_w(l).  From l - 1 to l every T_w
// stays or grows by one, and the new cell adds T_{v(l)} = v(l).  So with
// m = L(l - 1): L(l) = m exactly when the cone of value m is still flat
// (l - last[m] <= m; only w = m can keep the value m), else m + 1 -- then
// min with v(l).  One lookup of last[m] per step, O(n) per line (the outward
// scan of the former kernel was O(cap) per cell: 0.15-0.53 ms per pass at
// 1024^3).  The right sweep mirrors it; D = min(L, R), capped.  A block
// stages 64 x-columns (lines) in shared memory with all 256 threads; 64 of
// them then sweep one line each.
constexpr int kSweepCols = 64;

template <int AXIS, int DIR>
__global__ void __launch_bounds__(4 * kSweepCols) dist_sweep_kernel(const uint8_t* __restrict__ src,
                                                                   uint8_t* __restrict__ dst,
                                                                   int mx, int my, int mz, int cap) {
  // DIR 0: D = min(L, R); DIR +1: R only (cells at l' >= l); DIR -1: L only
  extern __shared__ uint8_t sweep_sm[];
  const int n = AXIS == 1 ? my : mz;
  uint8_t* val = sweep_sm;                                   // [n][64] v, then D
  uint8_t* left = sweep_sm + (size_t)n * kSweepCols;         // [n][64] L
  uint16_t* last = reinterpret_cast<uint16_t*>(sweep_sm + (size_t)2 * n * kSweepCols);  // [cap][64]
  const int64_t stride = AXIS == 1 ? (int64_t)mx : (int64_t)mx * my;
  const int64_t base0 = AXIS == 1 ? (int64_t)blockIdx.y * mx * my : (int64_t)blockIdx.y * mx;
  const int x0 = blockIdx.x * kSweepCols;
  // staging by all 256 threads: 4 lines' rows at a time, lanes along x
  {
    const int c = threadIdx.x & (kSweepCols - 1), r = threadIdx.x / kSweepCols;
    if (x0 + c < mx)
      for (int l = r; l < n; l += 4) val[l * kSweepCols + c] = src[base0 + l * stride + x0 + c];
  }
  __syncthreads();
  const int tx = threadIdx.x;
  if (tx < kSweepCols && x0 + tx < mx) {
    constexpr uint16_t kNone = 0xffffu;
    if (DIR <= 0) {  // left sweep
      for (int w = 0; w < cap; ++w) last[w * kSweepCols + tx] = kNone;
      int m = cap;
      for (int l = 0; l < n; ++l) {
        const int v = val[l * kSweepCols + tx];
        if (v < cap) last[v * kSweepCols + tx] = (uint16_t)l;
        if (m < cap) {
          const int lm = last[m * kSweepCols + tx];
          if (lm == kNone || l - lm > m) m = min(m + 1, cap);
        }
        if (v < m) m = v;
        left[l * kSweepCols + tx] = (uint8_t)m;
      }
    }
    if (DIR < 0) {
      for (int l = 0; l < n; ++l) val[l * kSweepCols + tx] = left[l * kSweepCols + tx];
    } else {
      // right sweep, then D = min(L, R) (or R alone) in place of v (v(l) is
      // not read again)
      for (int w = 0; w < cap; ++w) last[w * kSweepCols + tx] = kNone;
      int m = cap;
      for (int l = n - 1; l >= 0; --l) {
        const int v = val[l * kSweepCols + tx];
        if (v < cap) last[v * kSweepCols + tx] = (uint16_t)l;
        if (m < cap) {
          const int lm = last[m * kSweepCols + tx];
          if (lm == kNone || lm - l > m) m = min(m + 1, cap);
        }
        if (v < m) m = v;
        val[l * kSweepCols + tx] = (uint8_t)(DIR == 0 ? min(m, (int)left[l * kSweepCols + tx]) : m);
      }
    }
  }
  __syncthreads();
  {
    const int c = threadIdx.x & (kSweepCols - 1), r = threadIdx.x / kSweepCols;
    if (x0 + c < mx)
      for (int l = r; l < n; l += 4) dst[base0 + l * stride + x0 + c] = val[l * kSweepCols + c];
  }
}

static int smem_opt_in(const void* fn, size_t smem) {
  if (smem > 48 * 1024)
    VX_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  return VX_OK;
}

// one thread per VX_CELL^3 cell (4^3: 4-byte aligned rows of 4 voxels)
__global__ void cell_max_kernel(const uint8_t* __restrict__ origin, int64_t sy, int64_t sz, int ncx,
                                int ncy, int ncz, uint8_t* __restrict__ cmax_origin, int64_t csy,
                                int64_t csz) {
  static_assert(VX_CELL == 4, "cell_max_kernel assumes 4^3 cells");
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= (int64_t)ncx * ncy * ncz) return;
  const int cx = (int)(c % ncx);
  const int cy = (int)((c / ncx) % ncy);
  const int cz = (int)(c / ((int64_t)ncx * ncy));
  const uint8_t* p = origin + (int64_t)cz * 4 * sz + (int64_t)cy * 4 * sy + (int64_t)cx * 4;
  uint32_t m = 0;
#pragma unroll
  for (int z = 0; z < 4; ++z)
#pragma unroll
    for (int y = 0; y < 4; ++y) m = __vmaxu4(m, __ldg(reinterpret_cast<const uint32_t*>(p + z * sz + y * sy)));
  m = max(max(m & 0xffu, (m >> 8) & 0xffu), max((m >> 16) & 0xffu, m >> 24));
  cmax_origin[(int64_t)cz * csz + (int64_t)cy * csy + cx] = (uint8_t)m;
}

__global__ void u16_to_u8_kernel(const uint16_t* __restrict__ src, uint8_t* __restrict__ dst,
                                 uint64_t n) {
  // (v + 128) / 257 == floor(v * 255 / 65535 + 0.5) for all 65536 v
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    dst[i] = (uint8_t)(((uint32_t)src[i] + 128u) / 257u);
}

// ---- phantom generator (volume.py:317-368) ---------------------------------

__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

struct ShapeD {
  int kind;  // 0 sphere, 1 shell, 2 box
  double cx, cy, cz, radius, thickness, ex, ey, ez;
  int intensity;
  int x0, y0, z0, sx, sy, sz;  // bounding sub-grid
};

__global__ void paint_kernel(uint8_t* __restrict__ dst, int64_t rp, int64_t pp, ShapeD s) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n = (int64_t)s.sx * s.sy * s.sz;
  if (c >= n) return;
  const int x = s.x0 + (int)(c % s.sx);
  const int y = s.y0 + (int)((c / s.sx) % s.sy);
  const int z = s.z0 + (int)(c / ((int64_t)s.sx * s.sy));
  const double dx = __dsub_rn((double)x, s.cx), dy = __dsub_rn((double)y, s.cy),
               dz = __dsub_rn((double)z, s.cz);
  bool inside;
  if (s.kind == 2) {
    inside = fabs(dx) <= s.ex / 2.0 && fabs(dy) <= s.ey / 2.0 && fabs(dz) <= s.ez / 2.0;
  } else {
    const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
    if (s.kind == 0)
      inside = d2 <= __dmul_rn(s.radius, s.radius);
    else
      inside = fabs(__dsub_rn(__dsqrt_rn(d2), s.radius)) <= s.thickness / 2.0;
  }
  if (inside) dst[(int64_t)z * pp + (int64_t)y * rp + x] = (uint8_t)s.intensity;
}

__global__ void noise_kernel(uint8_t* __restrict__ dst, int64_t rp, int64_t pp, int64_t nx,
                             int64_t ny, int64_t nz, double sigma, unsigned long long seed) {
  const int64_t n = nx * ny * nz;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t x = i % nx, y = (i / nx) % ny, z = i / (nx * ny);
    uint8_t* p = dst + z * pp + y * rp + x;
    const double base = (double)*p;
    // draws 2i, 2i+1 of stream(seed): mix64(seed + (j+1)*GOLDEN)  (rng.py:33-51)
    const unsigned long long j0 = 2ull * (unsigned long long)i;
    const unsigned long long b0 = mix64(seed + (j0 + 1ull) * 0x9E3779B97F4A7C15ull);
    const unsigned long long b1 = mix64(seed + (j0 + 2ull) * 0x9E3779B97F4A7C15ull);
    const double u1 = __dmul_rn(__dadd_rn((double)(b0 >> 11), 1.0), 1.1102230246251565e-16);
    const double u2 = __dmul_rn((double)(b1 >> 11), 1.1102230246251565e-16);
    const double g = __dmul_rn(__dsqrt_rn(__dmul_rn(-2.0, log(u1))),
                               cos(__dmul_rn(6.283185307179586, u2)));
    double v = floor(__dadd_rn(__dadd_rn(base, __dmul_rn(sigma, g)), 0.5));
    v = v < 0.0 ? 0.0 : (v > 255.0 ? 255.0 : v);
    *p = (uint8_t)v;
  }
}

__global__ void spot_kernel(uint8_t* __restrict__ dst, int64_t rp, int64_t pp, int64_t nx,
                            int64_t ny, const int64_t* __restrict__ idx, int64_t k, int val) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= k) return;
  const int64_t i = idx[r];
  const int64_t x = i % nx, y = (i / nx) % ny, z = i / (nx * ny);
  dst[z * pp + y * rp + x] = (uint8_t)val;
}

// C4 input: a 16-bit CT file whose load_raw rescale
// (v + 128) / 257 (volume.py:148-150) returns exactly v8 -- u16 =
// clamp(257*v8 + e, 0, 65535) with dither e = (stream(seed)[i] mod 257) - 128
// in [-128, 128]
__global__ void u16_dither_kernel(const uint8_t* __restrict__ v8, uint64_t n, uint64_t i0,
                                  unsigned long long seed, uint16_t* __restrict__ out) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const unsigned long long b = mix64(seed + (i0 + i + 1ull) * 0x9E3779B97F4A7C15ull);
    const int e = (int)(b % 257ull) - 128;
    int v = 257 * (int)v8[i] + e;
    v = v < 0 ? 0 : (v > 65535 ? 65535 : v);
    out[i] = (uint16_t)v;
  }
}

// one thread per 8-voxel brick row (bz, by, bx, z, y): 8 bytes of the
// linear apron layout (X = x + VX_PAD multiple of 8: 8-byte aligned) into
// the brick; bytes beyond the padded grid are zero
__global__ void brickify_kernel(const uint8_t* __restrict__ lin, int64_t sy, int64_t sz,
                                int64_t px, int64_t py, int64_t pz, uint8_t* __restrict__ bricks,
                                int bbx, int bby, int bbz) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nrows = (int64_t)bbx * bby * bbz * 64;
  if (r >= nrows) return;
  const int64_t b = r >> 6;
  const int zy = (int)(r & 63), zi = zy >> 3, yi = zy & 7;
  const int bx = (int)(b % bbx), by = (int)((b / bbx) % bby), bz = (int)(b / ((int64_t)bbx * bby));
  const int64_t X = (int64_t)bx * 8, Y = (int64_t)by * 8 + yi, Z = (int64_t)bz * 8 + zi;
  uint2 w = make_uint2(0u, 0u);
  if (Y < py && Z < pz && X + 8 <= px)
    w = __ldg(reinterpret_cast<const uint2*>(lin + Z * sz + Y * sy + X));
  else if (Y < py && Z < pz)
    for (int k = 0; k < 8 && X + k < px; ++k)
      (k < 4 ? w.x : w.y) |= (uint32_t)lin[Z * sz + Y * sy + X + k] << (8 * (k & 3));
  uint8_t* dst = bricks + (b << 9);
  for (int k = 0; k < 8; ++k)
    dst[vx_in_brick(k, yi, zi)] = (uint8_t)(((k < 4 ? w.x : w.y) >> (8 * (k & 3))) & 0xffu);
}

}  // namespace

int vx_launch_brickify(vx_volume* v, cudaStream_t s) {
  const int64_t nrows = (int64_t)v->bbx * v->bby * v->bbz * 64;
  brickify_kernel<<<(unsigned)((nrows + 255) / 256), 256, 0, s>>>(
      v->alloc, v->sy, v->sz, v->px, v->py, v->pz, v->bricks, v->bbx, v->bby, v->bbz);
  VX_CHECK_LAUNCH();
  return VX_OK;
}

extern "C" int vx_u16_dither_device(const uint8_t* dev_v8, uint64_t n, uint64_t i0, uint64_t seed,
                                    uint16_t* dev_out, void* stream) {
  if ((!dev_v8 || !dev_out) && n) {
    vx_set_error("vx_u16_dither_device: null argument");
    return VX_EINVAL;
  }
  if (!n) return VX_OK;
  const unsigned grid = (unsigned)std::min<uint64_t>((n + 255) / 256, (uint64_t)vx_sm_count() * 16);
  u16_dither_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(dev_v8, n, i0, seed, dev_out);
  VX_CHECK_LAUNCH();
  return VX_OK;
}

int vx_launch_brick_max(vx_volume* v, cudaStream_t s) {
  const int64_t nb = (int64_t)v->nbx * v->nby * v->nbz;
  uint8_t* borigin = v->bmax + v->bsz + v->bsy + 1;
  brick_max_kernel<<<(unsigned)((nb + 127) / 128), 128, 0, s>>>(v->origin, v->sy, v->sz, v->nbx,
                                                                 v->nby, v->nbz, borigin, v->bsy,
                                                                 v->bsz);
  VX_CHECK_LAUNCH();
  return VX_OK;
}

// tmp: an intermediate of mx*my*mz bytes (the volume's build scratch: a
// stream-ordered allocation here grew the pool inside a frame, 1-20 ms)
template <int DX, int DY, int DZ>
static int dist_transform_dir(const uint8_t* maxmap, uint8_t* out, int mx, int my, int mz, int thr,
                              int cap, uint8_t* tmp, cudaStream_t s) {
  const int64_t rows = (int64_t)my * mz;
  const size_t s0 = (size_t)kRowsPerBlock * (mx | 1);
  int rc = smem_opt_in((const void*)dist_first_x_kernel<DX>, s0);
  if (rc) return rc;
  dist_first_x_kernel<DX><<<(unsigned)((rows + kRowsPerBlock - 1) / kRowsPerBlock), 256, s0, s>>>(
      maxmap, out, mx, rows, thr, cap);
  VX_CHECK_LAUNCH();
  const unsigned gx = (unsigned)((mx + kSweepCols - 1) / kSweepCols);
  // values >= cap never enter last[cap] (u8 maps: cap <= 255)
  if (cap > 255) {
    vx_set_error("distance cap %d > 255", cap);
    return VX_EINVAL;
  }
  auto sweep_smem = [cap](int n) {
    return (size_t)2 * n * kSweepCols + (size_t)2 * cap * kSweepCols;
  };
  const size_t s1 = sweep_smem(my), s2 = sweep_smem(mz);
  if ((rc = smem_opt_in((const void*)dist_sweep_kernel<1, DY>, s1))) return rc;
  dist_sweep_kernel<1, DY><<<dim3(gx, (unsigned)mz), 4 * kSweepCols, s1, s>>>(out, tmp, mx, my,
                                                                               mz, cap);
  VX_CHECK_LAUNCH();
  if ((rc = smem_opt_in((const void*)dist_sweep_kernel<2, DZ>, s2))) return rc;
  dist_sweep_kernel<2, DZ><<<dim3(gx, (unsigned)my), 4 * kSweepCols, s2, s>>>(tmp, out, mx, my,
                                                                               mz, cap);
  VX_CHECK_LAUNCH();
  return VX_OK;
}

static int dist_transform(const uint8_t* maxmap, uint8_t* out, int mx, int my, int mz, int thr,
                          int cap, uint8_t* tmp, cudaStream_t s) {
  return dist_transform_dir<0, 0, 0>(maxmap, out, mx, my, mz, thr, cap, tmp, s);
}

// coarse (bricks) then fine (cells) Chebyshev distance maps of thr into `map`
int vx_launch_dist_map(const vx_volume* v, int thr, uint8_t* map, cudaStream_t s) {
  int rc = dist_transform(v->bmax, map, v->nbx + 2, v->nby + 2, v->nbz + 2, thr, VX_DIST_CAP,
                          v->scratch + v->cmap_bytes, s);
  if (rc) return rc;
  return dist_transform(v->cmax, map + v->map_bytes, v->ncx + 2, v->ncy + 2, v->ncz + 2, thr,
                        v->fine_cap, v->scratch + v->cmap_bytes, s);
}

int vx_launch_dist_cells(const vx_volume* v, const uint8_t* occ, uint8_t* out, int thr,
                         cudaStream_t s) {
  return dist_transform(occ, out, v->ncx + 2, v->ncy + 2, v->ncz + 2, thr, v->fine_cap,
                        v->scratch + v->cmap_bytes, s);
}

// Orthant map `oct` (bit a set: rays move toward -axis a): the Chebyshev
// distance to the nearest occupied cell among those a ray of that orthant
// can still reach, D(c) = min over occupied o with s_a (o_a - c_a) >= 0 of
// max_a s_a (o_a - c_a) -- separable like the two-sided map, with one-sided
// sweeps (SURVEY Appendix A skip argument, DESIGN.md §5 "orthant maps").
int vx_launch_dist_cells_oct(const vx_volume* v, const uint8_t* occ, uint8_t* out, int thr, int oct,
                             cudaStream_t s) {
  const int mx = v->ncx + 2, my = v->ncy + 2, mz = v->ncz + 2;
  uint8_t* tmp = v->scratch + v->cmap_bytes;
#define VX_OCT(o, dx, dy, dz) \
  case o: return dist_transform_dir<dx, dy, dz>(occ, out, mx, my, mz, thr, v->fine_cap, tmp, s)
  switch (oct) {
    VX_OCT(0, 1, 1, 1);
    VX_OCT(1, -1, 1, 1);
    VX_OCT(2, 1, -1, 1);
    VX_OCT(3, -1, -1, 1);
    VX_OCT(4, 1, 1, -1);
    VX_OCT(5, -1, 1, -1);
    VX_OCT(6, 1, -1, -1);
    VX_OCT(7, -1, -1, -1);
    default:
      return dist_transform(occ, out, mx, my, mz, thr, v->fine_cap, tmp, s);
  }
#undef VX_OCT
}

int vx_launch_cell_max(vx_volume* v, cudaStream_t s) {
  const int64_t nc = (int64_t)v->ncx * v->ncy * v->ncz;
  uint8_t* corigin = v->cmax + v->csz + v->csy + 1;
  cell_max_kernel<<<(unsigned)((nc + 255) / 256), 256, 0, s>>>(v->origin, v->sy, v->sz, v->ncx,
                                                                v->ncy, v->ncz, corigin, v->csy,
                                                                v->csz);
  VX_CHECK_LAUNCH();
  return VX_OK;
}

int vx_launch_u16_to_u8(const uint16_t* src, uint8_t* dst, uint64_t n, cudaStream_t s) {
  if (!n) return VX_OK;
  uint64_t g = (n + 255) / 256;
  const uint64_t cap = (uint64_t)vx_sm_count() * 16;
  if (g > cap) g = cap;
  u16_to_u8_kernel<<<(unsigned)g, 256, 0, s>>>(src, dst, n);
  VX_CHECK_LAUNCH();
  return VX_OK;
}

int vx_launch_phantom(uint8_t* dst, int64_t rp, int64_t pp, int64_t nx, int64_t ny, int64_t nz,
                      const double* shapes, int64_t n_shapes, double noise_sigma,
                      uint64_t noise_seed, const int64_t* spot_idx, int64_t n_spots,
                      int32_t spot_intensity, cudaStream_t s) {
  // shapes are painted in list order (volume.py:323-352); bounding sub-grid
  // exactly as volume.py:324-335
  for (int64_t k = 0; k < n_shapes; ++k) {
    const double* q = shapes + 10 * k;
    ShapeD sd;
    sd.kind = (int)q[0];
    sd.cx = q[1]; sd.cy = q[2]; sd.cz = q[3];
    sd.intensity = (int)q[4];
    sd.radius = q[5];
    sd.thickness = q[6];
    sd.ex = q[7]; sd.ey = q[8]; sd.ez = q[9];
    double rx, ry, rz;
    if (sd.kind == 2) {
      rx = sd.ex / 2.0; ry = sd.ey / 2.0; rz = sd.ez / 2.0;
    } else {
      rx = ry = rz = sd.radius + (sd.kind == 1 ? sd.thickness / 2.0 : 0.0);
    }
    const long long x0 = std::max(0ll, (long long)ceil(sd.cx - rx));
    const long long x1 = std::min((long long)nx - 1, (long long)floor(sd.cx + rx));
    const long long y0 = std::max(0ll, (long long)ceil(sd.cy - ry));
    const long long y1 = std::min((long long)ny - 1, (long long)floor(sd.cy + ry));
    const long long z0 = std::max(0ll, (long long)ceil(sd.cz - rz));
    const long long z1 = std::min((long long)nz - 1, (long long)floor(sd.cz + rz));
    if (x0 > x1 || y0 > y1 || z0 > z1) continue;
    sd.x0 = (int)x0; sd.y0 = (int)y0; sd.z0 = (int)z0;
    sd.sx = (int)(x1 - x0 + 1); sd.sy = (int)(y1 - y0 + 1); sd.sz = (int)(z1 - z0 + 1);
    const int64_t cnt = (int64_t)sd.sx * sd.sy * sd.sz;
    paint_kernel<<<(unsigned)((cnt + 255) / 256), 256, 0, s>>>(dst, rp, pp, sd);
    VX_CHECK_LAUNCH();
  }
  if (noise_sigma > 0.0) {
    const int64_t n = nx * ny * nz;
    int64_t g = (n + 255) / 256;
    const int64_t cap = (int64_t)vx_sm_count() * 32;
    if (g > cap) g = cap;
    noise_kernel<<<(unsigned)g, 256, 0, s>>>(dst, rp, pp, nx, ny, nz, noise_sigma,
                                             (unsigned long long)noise_seed);
    VX_CHECK_LAUNCH();
  }
  if (n_spots > 0) {
    int64_t* didx = nullptr;
    VX_CUDA(vx_malloc_async(&didx, n_spots * 8, s));
    VX_CUDA(cudaMemcpyAsync(didx, spot_idx, n_spots * 8, cudaMemcpyHostToDevice, s));
    spot_kernel<<<(unsigned)((n_spots + 255) / 256), 256, 0, s>>>(dst, rp, pp, nx, ny, didx,
                                                                   n_spots, spot_intensity);
    VX_CHECK_LAUNCH();
    VX_CUDA(cudaFreeAsync(didx, s));
  }
  return VX_OK;
}
