// K4 first-hit ray caster with fused per-hit filter, Sobel normal, Phong
// shading and image histogram; K5 standalone filter batch; ray setup,
// march_ray, Sobel and Phong batch entry points.
//
// Exact-arithmetic contract (reproduces render.py bit for bit; SURVEY.md
// Appendix A):
//   * ray setup in FP64 with numpy's operation order      render.py:188-230
//   * FP32 march, separate round-to-nearest mul/add (no FMA: this TU is also
//     built with -fmad=false), truncation toward zero, chunked t
//     accumulation: t_k = fl(base + fl(s*k)), base += fl(f32(m)*s)
//                                                            render.py:236-339
//   * integer filter sums, FP64 quotient                     filters.py:165-227
//   * exact-integer Sobel gradient, FP64 normal + Phong       render.py:344-403
//
// Exact empty-space skipping: a sample can only become a
// surface candidate when raw >= thr = ceil(T) (render.py:258,307), and only
// an accepted candidate (f >= T) ends a ray (render.py:311-329).  Per thr
// (and per filter setting) the volume keeps a map of 4^3 cells holding the
// Chebyshev cell distance D (capped per volume at max(dims)/16 clamped to
// [32, 128], vx_fine_cap_for) to the nearest cell with a candidate-level
// voxel (the candidate map) or with an accepted voxel (the accepted-cell
// map, K8); per ray-direction orthant also a one-sided map (DESIGN.md §5:
// only occupied cells on the side the ray moves toward count).  At a sample
// in a cell with D >= skip_min_d (2 for step >= 0.5, else 1), every cell
// within distance D-1 (on that side) is empty, so every later sample whose t
// lies before the ray's exit from that box -- its far faces shrunk by 1/8
// voxel, less a t margin of 1/16 + |t| 2^-19 -- truncates into an empty cell
// (computed positions are monotone in t and their FP32 error is < 2^-7 voxel
// for |p|, |t| < 8192).  Those samples are stepped
// over by index inside a chunk and by the exact FP32 base recurrence across
// chunks, so the t of every sample actually taken is bit-identical to the
// reference's.  Result-neutral by construction; switched off when thr == 0
// (every cell occupied).

#include <atomic>
#include <chrono>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "vx_internal.cuh"

namespace {

// ---------------------------------------------------------------------------
// kernel-argument structs (passed by value)

struct RayCamD {
  double right[3], up[3], fwd[3], origin[3];
  double tan_f, aspect;
  int W, H;
};

// Block = kWarpsPerBlock warps, each an 8x4 pixel slab of an 8x16 tile (warps
// retire independently; 1, 2 and 4 warps per block measured the same on the
// bench frame, r1_config_sweep), 32 resident warps per SM.
#ifndef VX_RAYCAST_WPB
#define VX_RAYCAST_WPB 4
#endif
// resident warps per SM the frame kernel is compiled for (64 registers at 32);
// the no-filter and mean kinds run lighter code and gain from 40 (48
// registers, a few spills: C2 none -3.5 %, mean -4 %; local cluster +9 %,
// entropy +17 % there; profiles/r2/r2_ab_misc.txt)
#ifndef VX_RAYCAST_MIN_WARPS_LIGHT
#define VX_RAYCAST_MIN_WARPS_LIGHT 40
#endif
#ifndef VX_RAYCAST_MIN_WARPS
#define VX_RAYCAST_MIN_WARPS 32
#endif
constexpr int kWarpsPerBlock = VX_RAYCAST_WPB;
constexpr int kBlocksPerTile = 4 / kWarpsPerBlock;
#ifndef VX_SPLIT_RAYS
#define VX_SPLIT_RAYS 1
#endif
constexpr bool kSplitRays = VX_SPLIT_RAYS && kWarpsPerBlock == 4;

// sample-group passes whose loads are issued together (2 or 4; 0 = per
// filter kind, see march())
#ifndef VX_COOP_FIRST
// local cluster: when at most this many lanes of a warp evaluate a first
// candidate, the whole warp splits each one's taps (0 = owner lanes only).
// Measured (bench frame / C2 / C4): 2 -> -3 % / 0 / +0.8 %; 4 -> -3 % /
// +0.9 % / +1.3 %; 8 and 32 slower; two candidates per trip slower
#define VX_COOP_FIRST 2
#endif
#ifndef VX_COOP_MEAN
// the same for the box mean: 4 -> C1 mean -4.5 %, C2 mean 0 (2: +1.6 % on
// C2, 32: +3 %)
#define VX_COOP_MEAN 4
#endif
#ifndef VX_COOP_SIGMA
// the same for sigma: 4 -> C1 -11 %, C2/C3 -3.8 % (2: -11 % / -2.9 %)
#define VX_COOP_SIGMA 4
#endif
#ifndef VX_COOP_ENTROPY
// entropy (M = 3 only: one term per lane): 4 -> C1 -11 %, C3 -4.5 %
#define VX_COOP_ENTROPY 4
#endif
#ifndef VX_GROUP_PIPE
#define VX_GROUP_PIPE 0
#endif
// needy lanes from which each loads its own sample group instead of the
// warp's shuffle-fed passes, in skipping frames (33: never).  Measured
// (profiles/r2/r2_ab_own_group.txt): 8/12/20 cost the skipping frames 6-9 %
// (bench, C3 sigma/entropy) even when rarely taken, so skipping kernels keep
// the passes; the no-skip kernel (SKIP = false) always loads its own groups.
#ifndef VX_OWN_MIN
#define VX_OWN_MIN 33
#endif

struct MarchD {
  float s;        // f32(step)
  float inv_s;    // 1/s (estimates only)
  float sk_last;  // fl(s * (chunk - 1))
  float adv;      // fl(f32(chunk) * s)
  float sk[16];   // fl(s * k), k < chunk
  float xmax, ymax, zmax;
  int chunk;
  int need_clip;
  int explicit_max;  // > 0: exact frame budget; 0: per-ray guard
  int thr;           // ceil(T) in [0, 255]
  int skip;
  int skip_min_d;    // smallest cell distance that takes the box skip (tuning)
  double T;
  double step;       // FP64 step (per-ray guard)
};

struct FiltD {
  int kind;
  int M;        // kernel size
  int d;        // cluster offset
  int pairwise; // entropy sum order (K5, single coordinate)
  double band, okada_t, entropy_t;
};

struct ShadeD {
  double ka, kd, ks, shin;
  double l[3];
  int background;
};

struct OutD {
  uint8_t* pixels;
  int32_t* hit_voxel;
  float* hit_t;
  double* hit_value;
  double* intensity;
  unsigned long long* image_hist;
  unsigned long long* hit_count;
  unsigned long long* samples;
  unsigned long long* diag;
  int32_t* trunc_flag;
  // outputs live in another rank's memory (vx_group): system-scope atomics
  int sys;
};

// counter update of K4's fused outputs (device scope, or system scope when
// several GPUs accumulate into one rank's counters over NVLink)
__device__ __forceinline__ void out_add(unsigned long long* p, unsigned long long v, int sys) {
  if (sys)
    atomicAdd_system(p, v);
  else
    atomicAdd(p, v);
}

struct RenderArgs {
  VolView V;
  RayCamD C;
  MarchD M;
  FiltD F;
  ShadeD S;
  OutD O;
  int rank, world, tiles_x, n_tiles;
  // adaptive tile order (nullable): block b renders owned tile order[b]
  // and records its duration in tile_cost[owned tile] for the next frame
  // order[owned_tiles..+2] holds H8, H4, H2: the first tiles of the order
  // (the heaviest) are rendered by 8, 4 or 2 blocks each with every ray
  // split in as many segments; the launch has owned_tiles + split_max
  // blocks.  A ray is split only with >= split_min_chunks chunks per segment
  // (8; 1 under the tests' split-everything schedule).
  const uint32_t* tile_order;
  uint32_t* tile_cost;
  int owned_tiles, split_max, split_min_chunks;
  // entropy filter LUT in device memory (nullptr for the other filters): a
  // 2 KiB by-value array made the K4 argument block 2.6 KiB, and its launch
  // ~4 us slower
  const double* lut;
  const double* lut_host;  // host copy (map keys; never dereferenced on the device)
};

// Once-per-ray code (FP64 ray setup with its divisions, Sobel, Phong's FP64
// pow) kept out of line, so the march loop's instructions stay resident in
// the instruction cache (ncu: stall_no_instruction ~ as frequent as
// long-scoreboard stalls with everything inlined).
#ifndef VX_NOINLINE_COLD
#define VX_NOINLINE_COLD 0  // measured: noinline costs an 808-byte stack frame and spills
#endif
#if VX_NOINLINE_COLD
#define VX_COLD __device__ __noinline__
#else
#define VX_COLD __device__ __forceinline__
#endif

constexpr int kTileW = 8;
constexpr int kTileH = 16;

// ---------------------------------------------------------------------------
// voxel access

template <bool CHECKED>
__device__ __forceinline__ int rd(const VolView& V, long long x, long long y, long long z) {
  if (CHECKED) {
    if (x < 0 || y < 0 || z < 0 || x >= V.nx || y >= V.ny || z >= V.nz) return 0;
  }
  VX_DCHECK(x >= -VX_PAD && y >= -VX_PAD && z >= -VX_PAD && x < V.nx + VX_PAD &&
                y < V.ny + VX_PAD && z < V.nz + VX_PAD,
            "voxel (%lld, %lld, %lld) outside the apron of (%d, %d, %d)", x, y, z, V.nx, V.ny,
            V.nz);
  VX_DCHECK(V.origin + (z * V.sz + y * V.sy + x) >= V.lo &&
                V.origin + (z * V.sz + y * V.sy + x) < V.hi,
            "voxel (%lld, %lld, %lld) outside the allocation", x, y, z);
#if VX_BRICK_LAYOUT
  {
    const int X = (int)x + VX_PAD, Y = (int)y + VX_PAD, Z = (int)z + VX_PAD;
    const int b = ((Z >> 3) * V.bby + (Y >> 3)) * V.bbx + (X >> 3);
    return __ldg(V.bricks + ((size_t)b << 9) + vx_in_brick(X & 7, Y & 7, Z & 7));
  }
#endif
  return __ldg(V.origin + (z * V.sz + y * V.sy + x));
}

// ---------------------------------------------------------------------------
// filters (filters.py:165-227); integer sums, FP64 quotient

// numpy pairwise_sum (numpy/_core/src/umath/loops_utils.h) over a virtual
// array a(k): n < 8 sequential from 0; n <= 128 eight accumulators; larger n
// splits at n2 = n/2 - (n/2)%8.  Non-recursive (n <= 512: two split levels)
// so the kernels keep a static stack.
template <typename F>
__device__ double pw_block(const F& a, int off, int n) {
  if (n < 8) {
    double r = 0.0;
    for (int i = 0; i < n; ++i) r = __dadd_rn(r, a(off + i));
    return r;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = a(off + j);
  int i = 8;
  for (; i < n - (n % 8); i += 8)
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], a(off + i + j));
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < n; ++i) res = __dadd_rn(res, a(off + i));
  return res;
}

template <typename F>
__device__ double pw_level(const F& a, int off, int n) {  // n <= 256
  if (n <= 128) return pw_block(a, off, n);
  int n2 = n / 2;
  n2 -= n2 % 8;
  return __dadd_rn(pw_block(a, off, n2), pw_block(a, off + n2, n - n2));
}

template <typename F>
__device__ double pairwise_sum(const F& a, int n) {  // n <= 512
  if (n <= 128) return pw_block(a, 0, n);
  int n2 = n / 2;
  n2 -= n2 % 8;
  return __dadd_rn(pw_level(a, 0, n2), pw_level(a, n2, n - n2));
}

// cluster-loop unroll of the local-cluster filter (code size vs loop overhead)
#ifndef VX_LC_UNROLL
#define VX_LC_UNROLL 1
#endif
constexpr int kLcUnroll = VX_LC_UNROLL;
template <bool CHECKED>
__device__ double filter_lc(const VolView& V, const FiltD& F, long long x, long long y,
                            long long z) {
  long long sum = 0;
  const int h = (F.M - 1) >> 1;
#pragma unroll kLcUnroll
  for (int c = 0; c < 9; ++c) {
    long long cx = x, cy = y, cz = z;
    if (c > 0) {
      const int q = c - 1;  // (sx, sy, sz) in {-1,1}^3, filters.py:161
      cx += ((q >> 2) & 1 ? F.d : -F.d);
      cy += ((q >> 1) & 1 ? F.d : -F.d);
      cz += (q & 1 ? F.d : -F.d);
    }
    if (h == 1) {
      // M = 3: arms {c-1, c, c+1} per axis -> centre counted three times
      sum += 3 * rd<CHECKED>(V, cx, cy, cz) + rd<CHECKED>(V, cx - 1, cy, cz) +
             rd<CHECKED>(V, cx + 1, cy, cz) + rd<CHECKED>(V, cx, cy - 1, cz) +
             rd<CHECKED>(V, cx, cy + 1, cz) + rd<CHECKED>(V, cx, cy, cz - 1) +
             rd<CHECKED>(V, cx, cy, cz + 1);
    } else {
      for (int i = -h; i <= h; ++i)
        sum += rd<CHECKED>(V, cx + i, cy, cz) + rd<CHECKED>(V, cx, cy + i, cz) +
               rd<CHECKED>(V, cx, cy, cz + i);
    }
  }
  return __ddiv_rn((double)sum, (double)(27 * F.M));
}

template <bool CHECKED>
__device__ double filter_mean(const VolView& V, const FiltD& F, long long x, long long y,
                              long long z) {
  const int h = (F.M - 1) >> 1;
  long long sum = 0;
  for (int dz = -h; dz <= h; ++dz)
    for (int dy = -h; dy <= h; ++dy)
      for (int dx = -h; dx <= h; ++dx) sum += rd<CHECKED>(V, x + dx, y + dy, z + dz);
  return __ddiv_rn((double)sum, (double)(F.M * F.M * F.M));
}

template <bool CHECKED>
__device__ double filter_sigma(const VolView& V, const FiltD& F, long long x, long long y,
                               long long z) {
  const int h = (F.M - 1) >> 1;
  const int c = rd<CHECKED>(V, x, y, z);
  long long sum = 0;
  long long cnt = 0;
  for (int dz = -h; dz <= h; ++dz)
    for (int dy = -h; dy <= h; ++dy)
      for (int dx = -h; dx <= h; ++dx) {
        const int v = rd<CHECKED>(V, x + dx, y + dy, z + dz);
        const int diff = v > c ? v - c : c - v;
        if ((double)diff <= F.band) {
          sum += v;
          ++cnt;
        }
      }
  return __ddiv_rn((double)sum, (double)cnt);  // centre always qualifies
}

template <bool CHECKED>
__device__ double filter_okada(const VolView& V, const FiltD& F, long long x, long long y,
                               long long z) {
  const int c = rd<CHECKED>(V, x, y, z);
  const int nb[6] = {rd<CHECKED>(V, x - 1, y, z), rd<CHECKED>(V, x + 1, y, z),
                     rd<CHECKED>(V, x, y - 1, z), rd<CHECKED>(V, x, y + 1, z),
                     rd<CHECKED>(V, x, y, z - 1), rd<CHECKED>(V, x, y, z + 1)};
  long long total = 0;
  int n = 0;
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    const int diff = c > nb[k] ? c - nb[k] : nb[k] - c;
    if ((double)diff < F.okada_t) {
      total += nb[k];
      ++n;
    }
  }
  return n > 0 ? __ddiv_rn((double)total, (double)n) : 0.0;
}

template <bool CHECKED, bool PAIRWISE>
__device__ double filter_entropy(const VolView& V, const FiltD& F, const double* lut,
                                 long long x, long long y, long long z) {
  // kernel_offsets order: dx outer, dy, dz inner (filters.py:132-137)
  const int h = (F.M - 1) >> 1;
  double H;
  if (PAIRWISE) {
    // a single-coordinate batch: numpy sums the contiguous (M^3, 1) column
    // with pairwise_sum (SURVEY.md Appendix B exp. 7)
    const int M = F.M;
    auto term = [&](int k) {
      const int dz = k % M - h, dy = (k / M) % M - h, dx = k / (M * M) - h;
      return lut[rd<CHECKED>(V, x + dx, y + dy, z + dz)];
    };
    H = pairwise_sum(term, M * M * M);  // M <= 7 (checked by the host)
  } else {
    // >= 2 coordinates: row-by-row (sequential) reduction over axis 0
    bool first = true;
    H = 0.0;
    for (int dx = -h; dx <= h; ++dx)
      for (int dy = -h; dy <= h; ++dy)
        for (int dz = -h; dz <= h; ++dz) {
          const double t = lut[rd<CHECKED>(V, x + dx, y + dy, z + dz)];
          H = first ? t : __dadd_rn(H, t);
          first = false;
        }
  }
  return H > F.entropy_t ? (double)rd<CHECKED>(V, x, y, z) : 0.0;
}

// axis_cluster_average_batch (filters.py:177-178): the centre cluster alone
template <bool CHECKED>
__device__ double filter_axis(const VolView& V, const FiltD& F, long long x, long long y,
                              long long z) {
  const int h = (F.M - 1) >> 1;
  long long sum = 0;
  for (int i = -h; i <= h; ++i)
    sum += rd<CHECKED>(V, x + i, y, z) + rd<CHECKED>(V, x, y + i, z) + rd<CHECKED>(V, x, y, z + i);
  return __ddiv_rn((double)sum, (double)(3 * F.M));
}

// This lane's share of filter_lc's integer sum at (x, y, z): the 9 clusters'
// 3M-2 distinct taps each (centre weighted 3: the three arms share it),
// dealt round-robin over the warp.  Integer sums are order-free, so the warp
// total equals filter_lc's sum exactly.
template <bool CHECKED>
__device__ __forceinline__ int lc_tap_share(const VolView& V, const FiltD& F, int x, int y,
                                            int z, unsigned lane) {
  const int M = F.M, h = (M - 1) >> 1;
  const int P = 3 * M - 2, T = 9 * P;
  int s = 0;
  for (int t = (int)lane; t < T; t += 32) {
    const int c = (M == 3) ? t / 7 : t / P;
    const int r = t - c * P;
    int cx = x, cy = y, cz = z;
    if (c > 0) {
      const int q = c - 1;
      cx += ((q >> 2) & 1 ? F.d : -F.d);
      cy += ((q >> 1) & 1 ? F.d : -F.d);
      cz += (q & 1 ? F.d : -F.d);
    }
    if (r == 0) {
      s += 3 * rd<CHECKED>(V, cx, cy, cz);
    } else {
      const int a = (M == 3) ? (r - 1) >> 1 : (r - 1) / (M - 1);
      const int idx = (r - 1) - a * (M - 1);
      const int i = idx < h ? idx - h : idx - h + 1;
      s += rd<CHECKED>(V, cx + (a == 0 ? i : 0), cy + (a == 1 ? i : 0), cz + (a == 2 ? i : 0));
    }
  }
  return s;
}

// This lane's share of filter_mean's integer sum (the M^3 box), dealt
// round-robin over the warp.
template <bool CHECKED>
__device__ __forceinline__ int mean_tap_share(const VolView& V, const FiltD& F, int x, int y,
                                              int z, unsigned lane) {
  const int M = F.M, h = (M - 1) >> 1;
  int s = 0;
  for (int t = (int)lane; t < M * M * M; t += 32) {
    const int dz = (M == 3) ? t / 9 : t / (M * M);
    const int r = t - dz * M * M;
    const int dy = (M == 3) ? r / 3 : r / M;
    const int dx = r - dy * M;
    s += rd<CHECKED>(V, x + dx - h, y + dy - h, z + dz - h);
  }
  return s;
}

// This lane's share of filter_sigma's (sum, count) over the M^3 box: voxels
// within the band of the centre value c.
template <bool CHECKED>
__device__ __forceinline__ int sigma_tap_share(const VolView& V, const FiltD& F, int x, int y,
                                               int z, int c, unsigned lane, int& cnt) {
  const int M = F.M, h = (M - 1) >> 1;
  int s = 0;
  cnt = 0;
  for (int t = (int)lane; t < M * M * M; t += 32) {
    const int dz = (M == 3) ? t / 9 : t / (M * M);
    const int r = t - dz * M * M;
    const int dy = (M == 3) ? r / 3 : r / M;
    const int dx = r - dy * M;
    const int v = rd<CHECKED>(V, x + dx - h, y + dy - h, z + dz - h);
    const int diff = v > c ? v - c : c - v;
    if ((double)diff <= F.band) {
      s += v;
      ++cnt;
    }
  }
  return s;
}

constexpr int kAxisCluster = 6;  // K5-only kind

template <int KIND, bool CHECKED, bool PAIRWISE = false>
__device__ __forceinline__ double filter_value(const VolView& V, const FiltD& F, const double* lut,
                                               long long x, long long y, long long z) {
  if (KIND == VX_FILTER_NONE) return (double)rd<CHECKED>(V, x, y, z);
  if (KIND == VX_FILTER_MEAN) return filter_mean<CHECKED>(V, F, x, y, z);
  if (KIND == VX_FILTER_SIGMA) return filter_sigma<CHECKED>(V, F, x, y, z);
  if (KIND == VX_FILTER_OKADA) return filter_okada<CHECKED>(V, F, x, y, z);
  if (KIND == VX_FILTER_ENTROPY) return filter_entropy<CHECKED, PAIRWISE>(V, F, lut, x, y, z);
  if (KIND == kAxisCluster) return filter_axis<CHECKED>(V, F, x, y, z);
  return filter_lc<CHECKED>(V, F, x, y, z);
}

// ---------------------------------------------------------------------------
// ray setup (render.py:188-230)

// u and v of pixel (i, j) (render.py:193-196)
__device__ __forceinline__ double ray_u(const RayCamD& C, int i) {
  return __dmul_rn(
      __dmul_rn(__dsub_rn(__ddiv_rn(__dmul_rn(2.0, __dadd_rn((double)i, 0.5)), (double)C.W), 1.0),
                C.tan_f),
      C.aspect);
}
__device__ __forceinline__ double ray_v(const RayCamD& C, int j) {
  return __dmul_rn(__dsub_rn(1.0, __ddiv_rn(__dmul_rn(2.0, __dadd_rn((double)j, 0.5)), (double)C.H)),
                   C.tan_f);
}

// the normalised direction from u, v (render.py:197-201)
VX_COLD void ray_dir_uv(const RayCamD& C, double u, double v, double d[3]) {
#pragma unroll
  for (int c = 0; c < 3; ++c)
    d[c] = __dadd_rn(__dadd_rn(C.fwd[c], __dmul_rn(u, C.right[c])), __dmul_rn(v, C.up[c]));
  const double nrm = __dsqrt_rn(
      __dadd_rn(__dadd_rn(__dmul_rn(d[0], d[0]), __dmul_rn(d[1], d[1])), __dmul_rn(d[2], d[2])));
#pragma unroll
  for (int c = 0; c < 3; ++c) d[c] = __ddiv_rn(d[c], nrm);
}

VX_COLD void ray_dir(const RayCamD& C, int i, int j, double d[3]) {
  ray_dir_uv(C, ray_u(C, i), ray_v(C, j), d);
}

VX_COLD void ray_span(const double o[3], const double d[3], int nx, int ny,
                                         int nz, double& t_enter, double& t_exit) {
  const double hi[3] = {__dsub_rn((double)nx, 0.5), __dsub_rn((double)ny, 0.5),
                        __dsub_rn((double)nz, 0.5)};
  double tmin = -__longlong_as_double(0x7ff0000000000000ll);
  double tmax = __longlong_as_double(0x7ff0000000000000ll);
  // np.minimum / np.maximum propagate NaN: a NaN anywhere (0 * inf, only for
  // a subnormal direction component) makes both results NaN, so it is
  // tracked once instead of in every min / max
  bool nan = false;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    double near, far;
    if (d[a] == 0.0) {
      const bool inside = (-0.5 <= o[a]) && (o[a] <= hi[a]);
      near = inside ? -__longlong_as_double(0x7ff0000000000000ll)
                    : __longlong_as_double(0x7ff0000000000000ll);
      far = -near;
    } else {
      const double inv = __ddiv_rn(1.0, d[a]);
      const double t1 = __dmul_rn(__dsub_rn(-0.5, o[a]), inv);
      const double t2 = __dmul_rn(__dsub_rn(hi[a], o[a]), inv);
      nan = nan || t1 != t1 || t2 != t2;
      near = t1 < t2 ? t1 : t2;
      far = t1 > t2 ? t1 : t2;
    }
    tmin = tmin > near ? tmin : near;
    tmax = tmax < far ? tmax : far;
  }
  if (nan) {
    t_enter = t_exit = __longlong_as_double(0x7ff8000000000000ll);
    return;
  }
  t_enter = tmin > 0.0 ? tmin : 0.0;
  t_exit = tmax;
}

// ---------------------------------------------------------------------------
// the exact FP32 march (render.py:236-339) with exact skipping

struct RayState {
  float o[3];    // f32(origin + 0.5)
  float d[3];    // f32(dir)
  float inv[3];  // 1/d (skip estimates only; +-inf for +-0)
  float bo[3];   // exit-face offset minus origin: (inv > 0 ? -1/8 : 4 + 1/8) - o
  float base;
  float tend;
  const uint8_t* dmap;  // cell distance map the skips read (orthant or two-sided)
};

// the skip map of this ray: the map of its direction orthant when the frame
// built it (bit a of the orthant = moving toward -axis a, the same test as
// the exit-face choice in R.bo), else the two-sided Chebyshev map
__device__ __forceinline__ void ray_skip_map(RayState& R, const VolView& V) {
  const int oct = (R.inv[0] > 0.0f ? 0 : 1) | (R.inv[1] > 0.0f ? 0 : 2) | (R.inv[2] > 0.0f ? 0 : 4);
  R.dmap = ((V.oct_mask >> oct) & 1) ? V.doct + oct * V.oct_stride : V.dist2;
}

__device__ __forceinline__ void ray_skip_consts(RayState& R) {
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    R.inv[c] = __frcp_rn(R.d[c]);
    R.bo[c] = (R.inv[c] > 0.0f ? -0.125f : (float)VX_CELL + 0.125f) - R.o[c];
  }
}

__device__ __forceinline__ float pos1(float o, float t, float d) {
  return __fadd_rn(o, __fmul_rn(t, d));
}

__device__ __forceinline__ float clip1(float p, float hi) {
  // np.clip(p, 0, hi)
  return p < 0.0f ? 0.0f : (p > hi ? hi : p);
}

// the voxel a sample at t truncates into (render.py:303-306), as the march
// computes it
__device__ __forceinline__ void voxel_at(const RayState& R, const MarchD& M, float t, int& x,
                                         int& y, int& z) {
  float px = pos1(R.o[0], t, R.d[0]), py = pos1(R.o[1], t, R.d[1]), pz = pos1(R.o[2], t, R.d[2]);
  if (M.need_clip) {
    px = clip1(px, M.xmax);
    py = clip1(py, M.ymax);
    pz = clip1(pz, M.zmax);
  }
  x = __float2int_rz(px);
  y = __float2int_rz(py);
  z = __float2int_rz(pz);
}

enum MarchStatus { kMiss = 0, kHit = 1, kExhausted = 2, kRunning = 3 };

// per-warp shared scratch of the cooperative march
struct WarpScratch {
  int wl[32];                // lanes needing samples, by rank
  unsigned char items[256];  // candidate work items: (owner lane << 3) | sample j
  unsigned char pass[256];   // filter value >= T
};

// march statistics (vx_render_out.diag); compiled in only when requested
struct Diag {
  unsigned c[8];
};
enum DiagIndex { dLookup, dInChunk, dChunkLoop, dUnused, dGroup, dFilter, dHit, dIter };
#define VX_DIAG(i) \
  do {             \
    if (DIAG) ++dg.c[i]; \
  } while (0)
#define VX_DIAG_ADD(i, v)      \
  do {                         \
    if (DIAG) dg.c[i] += (v);  \
  } while (0)

constexpr int kGroup = 8;  // samples loaded together in occupied regions
#ifndef VX_CHUNK_UNROLL  // four-chunk trips: -1 never, 0 local cluster only, 1 every kind
#define VX_CHUNK_UNROLL 0
#endif

// t of sample k of the chunk starting at base: fl(base + fl(s * k))
__device__ __forceinline__ float sample_t(float base, float s, int k) {
  return __fadd_rn(base, __fmul_rn(s, (float)k));
}

// J steps of the chunk-base recurrence base <- fl(base + adv) in closed
// form, one binade at a time, in integer ulps.  Inside the binade
// [2^e, 2^(e+1)) of base every float is a multiple of u = ulp(base), so the
// round-to-nearest sum is fl(base + adv) = base + A*u with A = adv/u rounded
// to an integer -- independent of base unless adv/u is a tie (x.5: the
// even-mantissa rule then reads base's last bit), which falls back.  A sum
// reaching 2^(e+1) (mantissa carry into the exponent field) is still exact:
// sums in [2^(e+1) - u/2, 2^(e+1) + u/2) round to 2^(e+1) on either grid.
// So n steps add n*A to base's bit pattern while mant + n*A <= 2^23; a step
// that would leave the binade is taken as one plain add.  Returns the steps
// taken (< J only where it fell back: tie, adv >= ulp(base)*2^23 ... ).
#ifndef VX_CHUNK_JUMP
#define VX_CHUNK_JUMP 0  // 1: integer-ulp jumps; measured slower (profiles/r2/r2_ab_misc.txt)
#endif
__device__ __forceinline__ int chunk_jump_bits(float& base, float adv, int J) {
  const unsigned ab = __float_as_uint(adv);
  const int ea = (int)(ab >> 23);  // adv > 0 (normal): sign bit clear
  const unsigned ma = (ab & 0x7fffffu) | 0x800000u;
  unsigned b = __float_as_uint(base);
  int n_done = 0;
  while (n_done < J) {
    const int eb = (int)(b >> 23);
    const int sh = eb - ea;  // ulp(base) = 2^sh ulp(adv)
    if (sh < 1 || sh > 23 || eb > 253 || ea < 1) break;
    const unsigned half = 1u << (sh - 1);
    if ((ma & (2u * half - 1u)) == half) break;  // tie
    const unsigned A = (ma + half) >> sh;        // >= 1: ma >= 2^23 >= half
    const unsigned room = 0x800000u - (b & 0x7fffffu);
    unsigned n = (unsigned)(J - n_done);
    if ((unsigned long long)n * A > room) n = room / A;
    if (n == 0) {  // this step leaves the binade: the plain add
      b = __float_as_uint(__fadd_rn(__uint_as_float(b), adv));
      ++n_done;
    } else {
      b += n * A;
      n_done += (int)n;
    }
  }
  base = __uint_as_float(b);
  return n_done;
}

// first index in [lo, m] whose sample t exceeds lim (m if none); O(1):
// estimate, then fix up against the exact sample t (monotone in k)
__device__ __forceinline__ int first_beyond(float base, const MarchD& M, float lim, int lo, int m) {
  if (lo >= m) return m;
  const float q = __fmul_rn(__fsub_rn(lim, base), M.inv_s);
  int kn = q < 0.0f ? 0 : (q >= (float)m ? m : (int)q + 1);
  if (kn < lo) kn = lo;
  while (kn < m && sample_t(base, M.s, kn) <= lim) ++kn;
  while (kn > lo && sample_t(base, M.s, kn - 1) > lim) --kn;
  return kn;
}

// March (render.py:236-339), one ray per lane, as a warp-synchronous
// state machine.  Per ray: (done, k, base) = samples before the current
// chunk, next sample index in the chunk, exact FP32 chunk base.  Each
// iteration every running lane takes ONE step:
//   * chunk finished -> exact base recurrence (render.py:331);
//   * otherwise look up the fine Chebyshev cell distance D of the current
//     sample's cell.  D >= 1: the box of cells within D-1 is empty (all
//     max < thr); every sample up to the ray's exit from that box (less
//     margins) is stepped over -- whole chunks by the base recurrence,
//     single samples within a chunk -- and never loaded;
//   * D == 0 (the sample's cell holds a candidate-level voxel): the lane
//     needs its next kGroup samples.  Those are loaded cooperatively by the
//     whole warp (4 rays x 8 samples per pass, ray state by shuffles), so
//     the loads run at full SIMT width however few lanes need them; each
//     owner then resolves its candidates (raw >= thr) in order and runs the
//     filter until one is accepted (render.py:311-329).
// wl: this warp's 32-int shared scratch.  All 32 lanes must call.
// limit = the lane's sample budget.  Returns kHit, kMiss (left the span or
// inactive) or kExhausted (budget ran out while still inside the span).
// RAY_ORIGIN: rays have their own origins (march_ray); false: one camera
// origin for every ray of the frame, so the lanes that load or evaluate for
// another lane's ray use their own copy instead of shuffling it
template <int KIND, bool CHECKED, bool DIAG, bool BUDGET, bool SKIP = true, bool RAY_ORIGIN = false>
__device__ int march(const VolView& V, const MarchD& M, const FiltD& F, const double* lut,
                     const RayState& R, bool active, int limit, int done0, int stop,
                     float& ht, int& hidx, unsigned& nsamp, Diag& dg, WarpScratch* ws) {
  // On a hit only the sample t (ht) and its index (hidx) come back: the hit
  // voxel is trunc(pos(ht)) and its filter value a pure function of it, so
  // the caller recomputes both after the march (hit_voxel_of) instead of
  // keeping six more registers live through it.
  // BUDGET: the budget `limit` caps the march exactly (render.py:293-294).
  // !BUDGET: march unbudgeted; the caller compares the hit index with the
  // ray's own budget (a budget can only turn a hit at index >= limit into a
  // miss: it never changes a miss or an earlier hit).
  int* wl = ws->wl;
  const unsigned lane = (threadIdx.y * blockDim.x + threadIdx.x) & 31u;
  int status = active ? kRunning : kMiss;
  int done = done0;  // samples before R.base (a split ray's second segment)
  int k = 0;
  float base = R.base;
  const float tend = R.tend;
  const int chunk = M.chunk;
  // !BUDGET safety net for degenerate steps (base + adv == base): flag the
  // ray for the exact budgeted re-render instead of looping forever
  // stop > 0 (a split ray's first segment): hand over at sample `stop`
  int guard = BUDGET ? limit : (limit > (1 << 30) ? INT_MAX : limit + (1 << 20));
  if (!BUDGET && stop > 0 && stop < guard) guard = stop;
#ifdef VX_DEBUG_JITTER
  unsigned jit = lane * 2654435761u + blockIdx.x * 40503u;
#endif
  while (__any_sync(0xffffffffu, status == kRunning)) {
#ifdef VX_DEBUG_JITTER
    // checked build: lanes sleep 0-2 us at random before every step, so a
    // shared-scratch access missing its __syncwarp shows as a wrong frame
    jit = jit * 1664525u + 1013904223u;
    if (jit & 0x10000u) __nanosleep((jit >> 21) & 2047u);
#endif
    bool need = false;
    int m = chunk;
    if (status == kRunning) {
      VX_DIAG(dIter);
      if (BUDGET) {
        m = limit - done;
        if (m > chunk) m = chunk;
      }
      if (k >= m) {  // chunk finished: exact base recurrence (render.py:331)
        base = __fadd_rn(base, __fmul_rn((float)m, M.s));
        done += m;
        k = 0;
        if (!(base <= tend))
          status = kMiss;
        else if (done >= guard)
          status = kExhausted;
        if (BUDGET && status == kRunning) {
          m = limit - done;
          if (m > chunk) m = chunk;
        }
      } else if (!BUDGET && done >= guard) {
        // a skip crossed the guard inside a chunk (a split ray's first
        // segment reaching its hand-over sample): every sample before
        // done + k is covered
        status = kExhausted;
      }
      if (status == kRunning) {
        const float tk = sample_t(base, M.s, k);
        if (!(tk <= tend)) {
          // later samples of this chunk are beyond the exit too and the
          // next chunk's base >= t_k: the reference drops the ray
          status = kMiss;
        } else if (SKIP && M.skip) {
          const int vx = __float2int_rz(pos1(R.o[0], tk, R.d[0]));
          const int vy = __float2int_rz(pos1(R.o[1], tk, R.d[1]));
          const int vz = __float2int_rz(pos1(R.o[2], tk, R.d[2]));
          const int cx = vx >> VX_CELL_SHIFT, cy = vy >> VX_CELL_SHIFT, cz = vz >> VX_CELL_SHIFT;
          // in-span samples truncate into [0, n]: inside the map's 1-cell apron
          VX_DIAG(dLookup);
          VX_DCHECK((R.dmap == V.dist2 &&
                     R.dmap + (cz * (int)V.csz + cy * (int)V.csy + cx) >= V.d2lo &&
                     R.dmap + (cz * (int)V.csz + cy * (int)V.csy + cx) < V.d2hi) ||
                        (R.dmap != V.dist2 &&
                         R.dmap + (cz * (int)V.csz + cy * (int)V.csy + cx) >= V.dolo &&
                         R.dmap + (cz * (int)V.csz + cy * (int)V.csy + cx) < V.dohi),
                    "cell (%d, %d, %d) outside the distance map", cx, cy, cz);
          const int D = __ldg(R.dmap + (cz * (int)V.csz + cy * (int)V.csy + cx));
          float lim = -1.0f;
          if (D >= M.skip_min_d) {
            // cells within Chebyshev distance D-1 of this one: the box
            // [4(c-D+1), 4(c+D)) per axis in p = pos + 0.5 coordinates.  The
            // computed positions are monotone in t on each axis, so from
            // this sample (inside cell c) they move toward the box's far
            // faces and cannot pass them (shrunk by 1/8 voxel; FP32 position
            // error < 2^-7 voxel for |p|, |t| < 8192) before t_box (less a t
            // margin): every sample up to lim truncates into an empty cell.
            // Far face per axis: 4(c+D) - 1/8 when d > 0, 4(c-D+1) + 1/8
            // when d < 0 (R.bo folds the offsets).
            const int cc[3] = {cx, cy, cz};
            float tb = 3.0e38f;
#pragma unroll
            for (int a = 0; a < 3; ++a) {
              const int face = VX_CELL * (R.inv[a] > 0.0f ? cc[a] + D : cc[a] - D);
              tb = fminf(tb, __fmul_rn(__fadd_rn((float)face, R.bo[a]), R.inv[a]));  // NaN ignored
            }
            lim = __fsub_rd(tb, __fmaf_ru(fabsf(tb), 1.0f / 524288.0f, 0.0625f));
          }
          if (lim > tk) {
            // step over every sample with t <= lim: the rest of this chunk,
            // whole chunks by the exact base recurrence, then into the chunk
            // holding the first sample beyond lim
            VX_DIAG(dInChunk);
            if (BUDGET) {
              k = first_beyond(base, M, lim, k + 1, m);
              if (k >= m) {
                base = __fadd_rn(base, __fmul_rn((float)m, M.s));
                done += m;
                k = 0;
                // every bound of the budgeted loop (render.py:293, 331-332)
                for (;;) {
                  if (!(base <= tend)) { status = kMiss; break; }
                  if (done >= limit) { status = kExhausted; break; }
                  m = limit - done;
                  if (m > chunk) m = chunk;
                  if (m == chunk && __fadd_rn(base, M.sk_last) <= lim) {
                    VX_DIAG(dChunkLoop);
                    base = __fadd_rn(base, M.adv);
                    done += chunk;
                    continue;
                  }
                  k = first_beyond(base, M, lim, 0, m);
                  if (k < m) break;
                  base = __fadd_rn(base, __fmul_rn((float)m, M.s));
                  done += m;
                  k = 0;
                }
              }
            } else {
              // Unbudgeted: jump to a sample that is certainly <= lim (one
              // step short of the estimate (lim - t_k)/s; FP32 rounding of
              // sample t is far below a step), advancing whole chunks by the
              // exact base recurrence, then walk forward to the first sample
              // beyond lim.  A base past the exit is caught at the next sample
              // (t_k > tend), where the reference drops the ray as well (all
              // skipped samples are non-candidates).
              const float q = __fmul_rn(__fsub_rn(lim, tk), M.inv_s);
              int g = k + (q < 2.0f ? 0 : (q > 1.0e6f ? 1000000 : (int)q - 1));
              // whole chunks in closed form, binade by binade in integer ulps
              // (chunk_jump_bits); what it leaves (a tie) by the sequential
              // recurrence below
              if (VX_CHUNK_JUMP && g >= chunk && done < guard) {
                const int jg = g / chunk;
                const int jd = (guard - done + chunk - 1) / chunk;
                const int J = chunk_jump_bits(base, M.adv, jg < jd ? jg : jd);
                VX_DIAG_ADD(dChunkLoop, J);
                done += J * chunk;
                g -= J * chunk;
              }
              // four chunks per trip (same sequential recurrence, less loop
              // overhead per dependent add).  Measured per filter: local
              // cluster -1.5 % (bench frame) / -6.6 % (C4), the other kinds'
              // instantiations +2-5 % (register allocation), so LC only.
              if ((KIND == VX_FILTER_LOCAL_CLUSTER && VX_CHUNK_UNROLL >= 0) || VX_CHUNK_UNROLL > 0)
              while (g >= 4 * chunk && done + 3 * chunk < guard) {
                VX_DIAG_ADD(dChunkLoop, 4);
                base = __fadd_rn(__fadd_rn(__fadd_rn(__fadd_rn(base, M.adv), M.adv), M.adv), M.adv);
                done += 4 * chunk;
                g -= 4 * chunk;
              }
              while (g >= chunk && done < guard) {
                VX_DIAG(dChunkLoop);
                base = __fadd_rn(base, M.adv);
                done += chunk;
                g -= chunk;
              }
              k = g;
              for (;;) {
                if (k >= chunk) {
                  base = __fadd_rn(base, M.adv);
                  done += chunk;
                  k = 0;
                }
                if (sample_t(base, M.s, k) > lim || done >= guard) break;
                ++k;
              }
            }
          } else {
            need = true;
          }
        } else {
          need = true;
        }
      }
    }
    // ---- cooperative loads of the next kGroup samples of every needy lane ----
    const unsigned gm = __ballot_sync(0xffffffffu, need);
    if (gm) {
      const int nr = __popc(gm);
      const int rank = __popc(gm & ((1u << lane) - 1u));
      unsigned my_c = 0, my_v = 0;
      if (nr >= (SKIP ? VX_OWN_MIN : 0)) {
        // most lanes need samples (dense regions, no-skip frames): each loads
        // its own kGroup samples, all in flight together -- ~3x fewer issue
        // slots per sample than the shuffle-fed passes below, which pay off
        // only when few lanes need samples.  Same samples, same arithmetic.
        if (need) {
          int raws[kGroup];
#pragma unroll
          for (int j = 0; j < kGroup; ++j) {
            const int kk = min(k + j, max(m - 1, 0));
            const float t = sample_t(base, M.s, kk);
            float px = pos1(R.o[0], t, R.d[0]), py = pos1(R.o[1], t, R.d[1]),
                  pz = pos1(R.o[2], t, R.d[2]);
            if (M.need_clip) {
              px = clip1(px, M.xmax);
              py = clip1(py, M.ymax);
              pz = clip1(pz, M.zmax);
            }
            raws[j] = rd<false>(V, __float2int_rz(px), __float2int_rz(py), __float2int_rz(pz));
            if (k + j < m && t <= tend) my_v |= 1u << j;
          }
#pragma unroll
          for (int j = 0; j < kGroup; ++j)
            if (((my_v >> j) & 1u) && raws[j] >= M.thr) my_c |= 1u << j;
        }
      } else {
      if (need) wl[rank] = (int)lane;
      __syncwarp();
      // one pass = 4 rays x 8 samples; two passes are issued back to back so
      // their loads are in flight together
      auto pass_load = [&](int b, int& raw, bool& inr) {
        const int q = b + (int)(lane >> 3);
        const int j = (int)(lane & 7u);
        const int src = wl[q < nr ? q : 0];  // spare slots repeat a real ray: loads stay legal
        const float sb = __shfl_sync(0xffffffffu, base, src);
        const int sk = __shfl_sync(0xffffffffu, k, src);
        // unbudgeted chunks are always full: m == chunk on every lane
        const int sm = BUDGET ? __shfl_sync(0xffffffffu, m, src) : chunk;
        const float st = __shfl_sync(0xffffffffu, tend, src);
        const float o0 = RAY_ORIGIN ? __shfl_sync(0xffffffffu, R.o[0], src) : R.o[0];
        const float o1 = RAY_ORIGIN ? __shfl_sync(0xffffffffu, R.o[1], src) : R.o[1];
        const float o2 = RAY_ORIGIN ? __shfl_sync(0xffffffffu, R.o[2], src) : R.o[2];
        const float d0 = __shfl_sync(0xffffffffu, R.d[0], src);
        const float d1 = __shfl_sync(0xffffffffu, R.d[1], src);
        const float d2 = __shfl_sync(0xffffffffu, R.d[2], src);
        // clamped to the chunk: samples past the exit lie <= chunk*step <= 15
        // voxels outside the box, inside the zero apron (VX_PAD = 16) -- the
        // reference's own argument for unclamped overshoot reads
        // (render.py:283-285, 300-305)
        const int kk = min(sk + j, max(sm - 1, 0));
        const float t = sample_t(sb, M.s, kk);
        float px = pos1(o0, t, d0), py = pos1(o1, t, d1), pz = pos1(o2, t, d2);
        if (M.need_clip) {
          px = clip1(px, M.xmax);
          py = clip1(py, M.ymax);
          pz = clip1(pz, M.zmax);
        }
        raw = rd<false>(V, __float2int_rz(px), __float2int_rz(py), __float2int_rz(pz));
        inr = q < nr && sk + j < sm && t <= st;
      };
      auto pass_take = [&](int b, int raw, bool inr) {
        const unsigned bc = __ballot_sync(0xffffffffu, inr && raw >= M.thr);
        const unsigned bv = __ballot_sync(0xffffffffu, inr);
        if (need && rank >= b && rank < b + 4) {
          const int sh = (rank - b) * 8;
          my_c = (bc >> sh) & 0xffu;
          my_v = (bv >> sh) & 0xffu;
        }
      };
      // passes issued back to back: 4 where rejected candidates are common
      // (sigma, entropy), 2 for local cluster (measured: -3 % on the bench
      // frame with 2, entropy +2.6 %); VX_GROUP_PIPE forces one depth
      // Re-measured with distance-1 cells sampled (skip_min_d 2): 4 for
      // none/mean/okada too (C1 -5 %, C2 mean -3 %, okada -1.5 %), local
      // cluster stays at 2 (4: bench +1.7 %, C2 +3.8 %, C4 +1.3 %)
      // Late round 2, with per-kind occupancy: sigma at 2 too (C2 -3 %, C1
      // unchanged; none / mean / okada / entropy stay at 4: C1 +5 % at 2)
      constexpr int kPipe = VX_GROUP_PIPE ? VX_GROUP_PIPE
                            : (KIND == VX_FILTER_LOCAL_CLUSTER || KIND == VX_FILTER_SIGMA ? 2 : 4);
      if (kPipe == 4) {
      for (int b = 0; b < nr; b += 16) {
        int raw0, raw1 = 0, raw2 = 0, raw3 = 0;
        bool inr0, inr1 = false, inr2 = false, inr3 = false;
        pass_load(b, raw0, inr0);
        if (b + 4 < nr) pass_load(b + 4, raw1, inr1);
        if (b + 8 < nr) pass_load(b + 8, raw2, inr2);
        if (b + 12 < nr) pass_load(b + 12, raw3, inr3);
        pass_take(b, raw0, inr0);
        if (b + 4 < nr) pass_take(b + 4, raw1, inr1);
        if (b + 8 < nr) pass_take(b + 8, raw2, inr2);
        if (b + 12 < nr) pass_take(b + 12, raw3, inr3);
      }
      } else {
      for (int b = 0; b < nr; b += 8) {
        int raw0, raw1 = 0;
        bool inr0, inr1 = false;
        pass_load(b, raw0, inr0);
        if (b + 4 < nr) pass_load(b + 4, raw1, inr1);
        pass_take(b, raw0, inr0);
        if (b + 4 < nr) pass_take(b + 4, raw1, inr1);
      }
      }
      __syncwarp();
      }  // cooperative passes
      // ---- cooperative filter evaluation: every candidate of every needy
      // lane is evaluated by some lane of the warp at once (filter values are
      // pure functions of the voxel), then each owner takes its FIRST passing
      // candidate in sample order -- the reference's sequential resolution
      // (render.py:311-329) without serialising filter-heavy rays ----
      // ---- candidate resolution (render.py:311-329): the first candidate of
      // each needy lane is evaluated by its owner (surface hits usually stop
      // there); the remaining candidates of lanes whose first one failed
      // (noise, filter-rejected interiors) are evaluated cooperatively by the
      // whole warp -- filter values are pure functions of the voxel -- and each
      // owner takes its FIRST passing one in sample order ----
      if (need) {
        VX_DIAG(dGroup);
        nsamp += __popc(my_v);
      }
      unsigned rem = 0;
      bool coop = false;
      constexpr int kCoop = KIND == VX_FILTER_LOCAL_CLUSTER ? VX_COOP_FIRST
                            : KIND == VX_FILTER_MEAN ? VX_COOP_MEAN
                            : KIND == VX_FILTER_SIGMA ? VX_COOP_SIGMA
                            : KIND == VX_FILTER_ENTROPY ? VX_COOP_ENTROPY : 0;
      if (kCoop) {
        const unsigned fm = __ballot_sync(0xffffffffu, need && my_c);
        coop = fm != 0 && __popc(fm) <= kCoop && (KIND != VX_FILTER_ENTROPY || F.M == 3);
        if (coop) {
          int cx = 0, cy = 0, cz = 0;
          const int j = my_c ? __ffs(my_c) - 1 : 0;
          if (need && my_c) {
            const float t = sample_t(base, M.s, k + j);
            float px = pos1(R.o[0], t, R.d[0]);
            float py = pos1(R.o[1], t, R.d[1]);
            float pz = pos1(R.o[2], t, R.d[2]);
            if (M.need_clip) {
              px = clip1(px, M.xmax);
              py = clip1(py, M.ymax);
              pz = clip1(pz, M.zmax);
            }
            cx = __float2int_rz(px);
            cy = __float2int_rz(py);
            cz = __float2int_rz(pz);
          }
          unsigned c = fm;
          while (c) {
            const int src = __ffs(c) - 1;
            c &= c - 1;
            const int sx = __shfl_sync(0xffffffffu, cx, src);
            const int sy = __shfl_sync(0xffffffffu, cy, src);
            const int sz = __shfl_sync(0xffffffffu, cz, src);
            double f;
            if (KIND == VX_FILTER_ENTROPY) {
              // lane i loads term i of the 27 (kernel_offsets order: dx outer,
              // dy, dz inner); the ordered FP64 sum is then formed by every
              // lane from broadcasts, in filter_entropy's sequence
              double term = 0.0;
              if (lane < 27) {
                const int dx = (int)lane / 9 - 1, dy = ((int)lane / 3) % 3 - 1,
                          dz = (int)lane % 3 - 1;
                term = lut[rd<CHECKED>(V, sx + dx, sy + dy, sz + dz)];
              }
              double H = __shfl_sync(0xffffffffu, term, 0);
#pragma unroll
              for (int i = 1; i < 27; ++i) H = __dadd_rn(H, __shfl_sync(0xffffffffu, term, i));
              f = H > F.entropy_t ? (double)rd<CHECKED>(V, sx, sy, sz) : 0.0;
            } else {
              int part, pcnt = 0;
              if (KIND == VX_FILTER_MEAN) {
                part = mean_tap_share<CHECKED>(V, F, sx, sy, sz, lane);
              } else if (KIND == VX_FILTER_SIGMA) {
                // every lane reads the centre itself (one L1-resident byte)
                part = sigma_tap_share<CHECKED>(V, F, sx, sy, sz, rd<CHECKED>(V, sx, sy, sz),
                                                lane, pcnt);
              } else {
                part = lc_tap_share<CHECKED>(V, F, sx, sy, sz, lane);
              }
              const int sum = __reduce_add_sync(0xffffffffu, part);
              const int cnt =
                  KIND == VX_FILTER_SIGMA ? __reduce_add_sync(0xffffffffu, pcnt) : 0;
              const double den = KIND == VX_FILTER_MEAN    ? (double)(F.M * F.M * F.M)
                                 : KIND == VX_FILTER_SIGMA ? (double)cnt  // centre qualifies
                                                           : (double)(27 * F.M);
              f = __ddiv_rn((double)sum, den);
            }
            if ((int)lane == src) {
              VX_DIAG(dFilter);
              if (f >= M.T) {
                VX_DIAG(dHit);
                ht = sample_t(base, M.s, k + j);
                k += j;
                status = kHit;
              } else {
                rem = my_c & (my_c - 1);
              }
            }
          }
        }
      }
      if (!coop && need && my_c) {
        const int j = __ffs(my_c) - 1;
        const float t = sample_t(base, M.s, k + j);
        float px = pos1(R.o[0], t, R.d[0]);
        float py = pos1(R.o[1], t, R.d[1]);
        float pz = pos1(R.o[2], t, R.d[2]);
        if (M.need_clip) {
          px = clip1(px, M.xmax);
          py = clip1(py, M.ymax);
          pz = clip1(pz, M.zmax);
        }
        const int cx = __float2int_rz(px), cy = __float2int_rz(py), cz = __float2int_rz(pz);
        VX_DIAG(dFilter);
        const double f = filter_value<KIND, CHECKED>(V, F, lut, cx, cy, cz);
        if (f >= M.T) {
          VX_DIAG(dHit);
          ht = t;
          k += j;  // hidx = done + k after the loop
          status = kHit;
        } else {
          rem = my_c & (my_c - 1);
        }
      }
      if (__any_sync(0xffffffffu, rem != 0)) {
        const int nc = __popc(rem);
        int incl = nc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int v = __shfl_up_sync(0xffffffffu, incl, o);
          if ((int)lane >= o) incl += v;
        }
        const int off = incl - nc;
        const int total = __shfl_sync(0xffffffffu, incl, 31);
        {
          unsigned c = rem;
          int i = 0;
          while (c) {
            const int j = __ffs(c) - 1;
            c &= c - 1;
            VX_DCHECK(off + i < 256, "candidate item %d outside the warp scratch", off + i);
            ws->items[off + i++] = (unsigned char)((lane << 3) | j);
          }
        }
        __syncwarp();
        for (int w0 = 0; w0 < total; w0 += 32) {
          const int w = w0 + (int)lane;
          const int item = ws->items[w < total ? w : 0];
          const int owner = item >> 3, j = item & 7;
          const float ob = __shfl_sync(0xffffffffu, base, owner);
          const int okk = __shfl_sync(0xffffffffu, k, owner);
          const float o0 = RAY_ORIGIN ? __shfl_sync(0xffffffffu, R.o[0], owner) : R.o[0];
          const float o1 = RAY_ORIGIN ? __shfl_sync(0xffffffffu, R.o[1], owner) : R.o[1];
          const float o2 = RAY_ORIGIN ? __shfl_sync(0xffffffffu, R.o[2], owner) : R.o[2];
          const float d0 = __shfl_sync(0xffffffffu, R.d[0], owner);
          const float d1 = __shfl_sync(0xffffffffu, R.d[1], owner);
          const float d2 = __shfl_sync(0xffffffffu, R.d[2], owner);
          if (w < total) {
            const float t = sample_t(ob, M.s, okk + j);
            float px = pos1(o0, t, d0), py = pos1(o1, t, d1), pz = pos1(o2, t, d2);
            if (M.need_clip) {
              px = clip1(px, M.xmax);
              py = clip1(py, M.ymax);
              pz = clip1(pz, M.zmax);
            }
            VX_DIAG(dFilter);
            const double f = filter_value<KIND, CHECKED>(V, F, lut, __float2int_rz(px),
                                                         __float2int_rz(py), __float2int_rz(pz));
            VX_DCHECK(w < 256, "pass slot %d outside the warp scratch", w);
            ws->pass[w] = f >= M.T ? 1 : 0;
          }
        }
        __syncwarp();
        unsigned c = rem;
        for (int i = 0; i < nc; ++i) {
          const int j = __ffs(c) - 1;
          c &= c - 1;
          if (ws->pass[off + i]) {
            VX_DIAG(dHit);
            ht = sample_t(base, M.s, k + j);
            k += j;  // hidx = done + k after the loop
            status = kHit;
            break;
          }
        }
        __syncwarp();
      }
      if (need && status == kRunning) k += min(kGroup, m - k);
    }
  }
  if (status == kHit) hidx = done + k;
  return status;
}

// ---------------------------------------------------------------------------
// Sobel (render.py:344-377) and Phong (render.py:385-403)

template <bool CHECKED>
VX_COLD void sobel(const VolView& V, long long x, long long y, long long z, const double fb[3],
                      double n[3]) {
  int gx = 0, gy = 0, gz = 0;
#pragma unroll
  for (int dx = -1; dx <= 1; ++dx)
#pragma unroll
    for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
      for (int dz = -1; dz <= 1; ++dz) {
        const int v = rd<CHECKED>(V, x + dx, y + dy, z + dz);
        const int sx = dx == 0 ? 2 : 1, sy = dy == 0 ? 2 : 1, sz = dz == 0 ? 2 : 1;
        gx += dx * sy * sz * v;
        gy += dy * sx * sz * v;
        gz += dz * sx * sy * v;
      }
  const double g0 = gx, g1 = gy, g2 = gz;
  const double nrm =
      __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(g0, g0), __dmul_rn(g1, g1)), __dmul_rn(g2, g2)));
  if (nrm < 1e-12) {
    n[0] = fb[0]; n[1] = fb[1]; n[2] = fb[2];
  } else {
    n[0] = __ddiv_rn(-g0, nrm);
    n[1] = __ddiv_rn(-g1, nrm);
    n[2] = __ddiv_rn(-g2, nrm);
  }
}

// n.l follows the reference host's OpenBLAS dgemv (fma(n2,l2, fma(n0,l0, n1*l1)),
// measured bit-exact on 20k random vectors); r.v follows numpy einsum
// ((r0 v0 + r2 v2) + r1 v1).  See DESIGN.md "shading order".
VX_COLD double phong_intensity(const double n[3], const double v[3],
                                                  const ShadeD& S) {
  const double ndotl = __fma_rn(n[2], S.l[2], __fma_rn(n[0], S.l[0], __dmul_rn(n[1], S.l[1])));
  const double k2 = __dmul_rn(2.0, ndotl);
  const double r0 = __dsub_rn(__dmul_rn(k2, n[0]), S.l[0]);
  const double r1 = __dsub_rn(__dmul_rn(k2, n[1]), S.l[1]);
  const double r2 = __dsub_rn(__dmul_rn(k2, n[2]), S.l[2]);
  const double rdotv = __dadd_rn(__dadd_rn(__dmul_rn(r0, v[0]), __dmul_rn(r2, v[2])), __dmul_rn(r1, v[1]));
  const double dif = ndotl > 0.0 ? ndotl : 0.0;
  const double spe = rdotv > 0.0 ? rdotv : 0.0;
  return __dadd_rn(__dadd_rn(S.ka, __dmul_rn(S.kd, dif)), __dmul_rn(S.ks, pow(spe, S.shin)));
}

__device__ __forceinline__ uint8_t quantise(double I) {
  const double c = I < 0.0 ? 0.0 : (I > 1.0 ? 1.0 : I);
  return (uint8_t)floor(__dadd_rn(__dmul_rn(c, 255.0), 0.5));
}

// per-ray budget guard: max(1, ceil(span/step) + 1) (render.py:469-473)
__device__ __forceinline__ int own_budget(double te, double tx, double step) {
  const double span = __dsub_rn(tx, te);
  const double q = ceil(__ddiv_rn(span, step));
  if (!(q <= 2.0e9)) return INT_MAX;
  int b = (int)q + 1;
  return b < 1 ? 1 : b;
}

// ---------------------------------------------------------------------------
// K4

static_assert(kWarpsPerBlock == 1 || kWarpsPerBlock == 2 || kWarpsPerBlock == 4, "warps per block");

#ifdef VX_WARP_TIMING
// debug build only: per-warp start/end globaltimer and SM of the last frame
__device__ unsigned long long g_warp_t0[1 << 20];
__device__ unsigned long long g_warp_t1[1 << 20];
__device__ unsigned g_warp_sm[1 << 20];
__device__ unsigned g_warp_diag[9 << 20];
#endif

// sigma and okada: 36 (56 registers; C2 sigma -1.5 %, okada -2.2 %)
#ifndef VX_RAYCAST_MIN_WARPS_MID
#define VX_RAYCAST_MIN_WARPS_MID 36
#endif
constexpr int raycast_min_warps(int kind) {
  return kind == VX_FILTER_NONE || kind == VX_FILTER_MEAN    ? VX_RAYCAST_MIN_WARPS_LIGHT
         : kind == VX_FILTER_SIGMA || kind == VX_FILTER_OKADA ? VX_RAYCAST_MIN_WARPS_MID
                                                              : VX_RAYCAST_MIN_WARPS;
}

template <int KIND, bool CHECKED, bool DIAG, bool BUDGET, bool SKIP = true>
__global__ void __launch_bounds__(32 * kWarpsPerBlock, raycast_min_warps(KIND) / kWarpsPerBlock)
    raycast_kernel(const RenderArgs a) {
  __shared__ double lut[KIND == VX_FILTER_ENTROPY ? 256 : 1];
  __shared__ WarpScratch wsc[kWarpsPerBlock];
  __shared__ unsigned long long block_t0;
  const int tid = threadIdx.y * kTileW + threadIdx.x;
  // owned tile of this block: the previous frame's cost order when given
  // (heaviest first, so the longest warps start at once), else the deal.
  // nseg > 1: a split block -- part `part` of the tile (16/nseg rows), each
  // warp 32/nseg rays with lanes l, l+32/nseg, ... marching the nseg
  // consecutive segments of one ray.  The first H8 tiles of the order are
  // split in 8 (eight blocks each), the next H4 in 4, the next H2 in 2, the
  // rest whole.
  int owned, nseg = 1, part = 0;
  if (!BUDGET && kSplitRays && a.tile_order) {
    // capped by this launch's reserve: the order may come from a frame of
    // another filter setting with another split cap
    int H8 = (int)a.tile_order[a.owned_tiles];
    int H4 = (int)a.tile_order[a.owned_tiles + 1];
    int H2 = (int)a.tile_order[a.owned_tiles + 2];
    if (7 * H8 > a.split_max) H8 = a.split_max / 7;
    if (7 * H8 + 3 * H4 > a.split_max) H4 = (a.split_max - 7 * H8) / 3;
    if (7 * H8 + 3 * H4 + H2 > a.split_max) H2 = a.split_max - 7 * H8 - 3 * H4;
    const int b = (int)blockIdx.x;
    const int e8 = 8 * H8, e4 = e8 + 4 * H4, e2 = e4 + 2 * H2;
    if (b < e8) {
      owned = (int)a.tile_order[b >> 3];
      nseg = 8;
      part = b & 7;
    } else if (b < e4) {
      owned = (int)a.tile_order[H8 + ((b - e8) >> 2)];
      nseg = 4;
      part = (b - e8) & 3;
    } else if (b < e2) {
      owned = (int)a.tile_order[H8 + H4 + ((b - e4) >> 1)];
      nseg = 2;
      part = (b - e4) & 1;
    } else if (b - 7 * H8 - 3 * H4 - H2 < a.owned_tiles) {
      owned = (int)a.tile_order[b - 7 * H8 - 3 * H4 - H2];
    } else {
      return;  // spare block (reserve not used up), whole block
    }
  } else {
    owned = a.tile_order ? (int)a.tile_order[blockIdx.x / kBlocksPerTile]
                         : (int)(blockIdx.x / kBlocksPerTile);
  }
  if (KIND == VX_FILTER_ENTROPY)
    for (int i = tid; i < 256; i += 32 * kWarpsPerBlock) lut[i] = a.lut[i];
  if (a.tile_cost && tid == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    block_t0 = t;
  }
  const int tile = a.rank + a.world * owned;
  // tile / tiles_x through an FP32 reciprocal (exact for tile < 2^24 after
  // the +-1 fix-up): a 32-bit integer division is ~25 instructions
  int ty = __float2int_rz(__fmul_rn((float)tile, __frcp_rn((float)a.tiles_x)));
  int tx = tile - ty * a.tiles_x;
  if (tx < 0) {
    --ty;
    tx += a.tiles_x;
  } else if (tx >= a.tiles_x) {
    ++ty;
    tx -= a.tiles_x;
  }
  // the tile's 8 column u and 16 row v (one FP64 division each, render.py:
  // 193-196) once per block instead of per pixel
  __shared__ double su[kTileW], sv[kTileH];
  if (tid < kTileW)
    su[tid] = ray_u(a.C, tx * kTileW + tid);
  else if (tid < kTileW + kTileH)
    sv[tid - kTileW] = ray_v(a.C, ty * kTileH + (tid - kTileW));
  __syncthreads();

#ifdef VX_WARP_TIMING
  unsigned long long wt0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(wt0));
#endif
  const int rpw = 32 / nseg;  // rays per warp
  const int seg = (int)(tid & 31) / rpw;
  const int ray = (int)(tid & 31) % rpw;
  // split: the part's 128/nseg rays, row-major 8 wide, rpw per warp
  const int rp = (tid >> 5) * rpw + ray;
  const int i = tx * kTileW + (nseg > 1 ? (rp & 7) : (ray & 7));
  const int j = nseg > 1 ? ty * kTileH + part * (kTileH / nseg) + (rp >> 3)
                         : ty * kTileH +
                               (int)(blockIdx.x % kBlocksPerTile) * (4 * kWarpsPerBlock) +
                               (int)threadIdx.y;
  bool valid = tile < a.n_tiles && i < a.C.W && j < a.C.H;

  bool hit = false;
  unsigned nsamp = 0;
  uint8_t pix_out = 0;
  Diag dg;
  if (DIAG)
    for (int i = 0; i < 8; ++i) dg.c[i] = 0;
  RayState R;
  bool live = false;
  int limit = 0;
  int hx = -1, hy = -1, hz = -1, hidx = 0;
  float ht = 0.0f;
  double hval = 0.0;
  // the frame's one origin, on every lane (march reads it for other lanes' rays)
#pragma unroll
  for (int c = 0; c < 3; ++c) R.o[c] = __double2float_rn(__dadd_rn(a.C.origin[c], 0.5));
  if (valid) {
    double d[3];
    ray_dir_uv(a.C, su[i - tx * kTileW], sv[j - ty * kTileH], d);
    double te, tx_;
    ray_span(a.C.origin, d, a.V.nx, a.V.ny, a.V.nz, te, tx_);
    hx = hy = hz = -1;
    live = tx_ >= te && a.M.thr <= 255;
    if (live) {
#pragma unroll
      for (int c = 0; c < 3; ++c) R.d[c] = __double2float_rn(d[c]);
      ray_skip_consts(R);
      ray_skip_map(R, a.V);
      R.base = __double2float_rn(te);
      R.tend = __double2float_rn(tx_);
      // Per-ray budget = this ray's own max(1, ceil(span/step) + 1) <= the
      // frame-wide budget of render.py:469-473.  A ray that ends (hit or exit)
      // within it behaves exactly as under the frame budget; one that exhausts
      // it is flagged and the host re-renders with the exact frame budget.
      limit = a.M.explicit_max > 0 ? a.M.explicit_max : own_budget(te, tx_, a.M.step);
    }
  }
  // split ray: segment s marches samples [s*K, (s+1)*K) (the last one to
  // the end), starting from the exact chunk base of sample s*K (the base
  // recurrence applied s*K/chunk times); K chunk-aligned.  A segment may run
  // a little past its end: its first hit is then still the first hit after
  // its start.  The ray's outcome is the first segment's hit, else the last
  // segment's outcome.
  int K = 0, done0 = 0, stop = 0;
  if (nseg > 1 && live) {
    const float nsf = __fmul_rn(__fsub_rn(R.tend, R.base), a.M.inv_s);
    K = nsf < (float)(a.split_min_chunks * a.M.chunk * nseg)
            ? 0
            : ((int)(nsf / nseg) / a.M.chunk) * a.M.chunk;
    if (K == 0) {
      live = seg == 0;  // too short to split: segment 0 marches it all
    } else {
      if (seg < nseg - 1) stop = (seg + 1) * K;
      done0 = seg * K;
      for (int c = 0; c < done0; c += a.M.chunk) R.base = __fadd_rn(R.base, a.M.adv);
    }
  }
  // all lanes of the warp march together (cooperative sample loads)
  {
    int st = march<KIND, CHECKED, DIAG, BUDGET, SKIP>(a.V, a.M, a.F, lut, R, live, limit, done0, stop,
                                                ht, hidx, nsamp, dg, &wsc[tid >> 5]);
    if (nseg > 1) {
      // merge pairwise toward segment 0: an earlier segment's hit wins
      for (int o = rpw; o < 32; o <<= 1) {
        const int st1 = __shfl_down_sync(0xffffffffu, st, o);
        const float ht1 = __shfl_down_sync(0xffffffffu, ht, o);
        const int hidx1 = __shfl_down_sync(0xffffffffu, hidx, o);
        if ((seg & ((2 * o / rpw) - 1)) == 0 && K > 0 && st != kHit) {
          st = st1;
          ht = ht1;
          hidx = hidx1;
        }
      }
      if (seg > 0) {
        st = kMiss;
        valid = false;
      }
    }
    hit = st == kHit;
    if (hit) {
      voxel_at(R, a.M, ht, hx, hy, hz);
      // per-pixel diagnostics live in the DIAG kernel only (keeps a third
      // inline copy of the filter out of the frame kernel's code)
      if (DIAG && a.O.hit_value) hval = filter_value<KIND, CHECKED>(a.V, a.F, lut, hx, hy, hz);
    }
    // unbudgeted march: only a hit at or beyond the ray's own budget can
    // differ from the budgeted reference -> exact re-render by the host
    if (!BUDGET && a.O.trunc_flag && ((hit && hidx >= limit) || st == kExhausted))
      a.O.sys ? atomicOr_system(a.O.trunc_flag, 1) : atomicOr(a.O.trunc_flag, 1);
  }
  if (valid) {
    const size_t p = (size_t)j * a.C.W + i;
    VX_DCHECK(i >= 0 && j >= 0 && i < a.C.W && j < a.C.H, "pixel (%d, %d) outside the frame", i, j);
    uint8_t pix = (uint8_t)a.S.background;
    double I = -1.0;
    if (hit) {
      // the FP64 direction is recomputed (bit-identical) instead of being
      // kept live in registers across the march
      double d[3];
      ray_dir_uv(a.C, su[i - tx * kTileW], sv[j - ty * kTileH], d);
      const double view[3] = {-d[0], -d[1], -d[2]};
      double n[3];
      sobel<CHECKED>(a.V, hx, hy, hz, view, n);
      I = phong_intensity(n, view, a.S);
      pix = quantise(I);
    }
    a.O.pixels[p] = pix;
    if (DIAG) {
      if (a.O.hit_voxel) {
        a.O.hit_voxel[3 * p] = hit ? hx : -1;
        a.O.hit_voxel[3 * p + 1] = hit ? hy : -1;
        a.O.hit_voxel[3 * p + 2] = hit ? hz : -1;
      }
      if (a.O.hit_t) a.O.hit_t[p] = hit ? ht : 0.0f;
      if (a.O.hit_value) a.O.hit_value[p] = hit ? hval : 0.0;
      if (a.O.intensity) a.O.intensity[p] = I;
    }
    pix_out = pix;
  }
  // warp-level aggregation (no block barrier: warps retire independently)
  const unsigned lane = tid & 31u;
  const unsigned hits = __ballot_sync(0xffffffffu, hit);
  if (lane == 0 && a.O.hit_count && hits) out_add(a.O.hit_count, (unsigned long long)__popc(hits), a.O.sys);
  if (a.O.samples) {
    unsigned s = nsamp;
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0 && s) out_add(a.O.samples, (unsigned long long)s, a.O.sys);
  }
  if (DIAG) {
    for (int i = 0; i < 8; ++i) {
      unsigned v = dg.c[i];
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0 && v && a.O.diag) atomicAdd(a.O.diag + i, (unsigned long long)v);
#ifdef VX_WARP_TIMING
      const unsigned w = blockIdx.x * kWarpsPerBlock + (tid >> 5);
      if (lane == 0 && w < (1u << 20)) g_warp_diag[w * 9 + i] = v;
#endif
    }
#ifdef VX_WARP_TIMING
    unsigned mx = dg.c[dIter];
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    const unsigned w = blockIdx.x * kWarpsPerBlock + (tid >> 5);
    if (lane == 0 && w < (1u << 20)) g_warp_diag[w * 9 + 8] = mx;
#endif
  }
#ifdef VX_WARP_TIMING
  {
    unsigned long long wt1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(wt1));
    const unsigned w = blockIdx.x * kWarpsPerBlock + (tid >> 5);
    if (lane == 0 && w < (1u << 20)) {
      g_warp_t0[w] = wt0;
      g_warp_t1[w] = wt1;
      unsigned sm;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
      // sm | nseg << 8 | part << 12 | owned tile << 16
      g_warp_sm[w] = sm | ((unsigned)nseg << 8) | ((unsigned)part << 12) | ((unsigned)owned << 16);
    }
  }
#endif
  if (a.tile_cost && lane == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    // ~microseconds; a split block stands for 1/nseg of its tile's work
    const unsigned long long us = ((t - block_t0) >> 10) * (unsigned)nseg;
    atomicMax(a.tile_cost + owned, (unsigned)min(us, 0xffffffffull));
  }
  if (a.O.image_hist) {
    const unsigned key = valid ? (unsigned)pix_out : 0x100u;
    const unsigned peers = __match_any_sync(0xffffffffu, key);
    if (valid && (__ffs(peers) - 1) == (int)lane)
      out_add(a.O.image_hist + pix_out, (unsigned long long)__popc(peers), a.O.sys);
  }
}

// frame-wide longest span (render.py:469-473), exact fallback budget
__global__ void span_max_kernel(const RayCamD C, int nx, int ny, int nz,
                                unsigned long long* __restrict__ out_bits) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  double span = 0.0;
  if (p < C.W * C.H) {
    double d[3];
    ray_dir(C, p % C.W, p / C.W, d);
    double te, tx;
    ray_span(C.origin, d, nx, ny, nz, te, tx);
    if (tx >= te) span = __dsub_rn(tx, te);
  }
  // non-negative doubles order like their bit patterns
  unsigned long long b = (unsigned long long)__double_as_longlong(span);
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long ob = __shfl_xor_sync(0xffffffffu, b, o);
    b = ob > b ? ob : b;
  }
  if ((threadIdx.x & 31) == 0) atomicMax(out_bits, b);
}

// next frame's tile order from this frame's per-tile costs: heaviest first
// (64 buckets, four per octave, descending; order within a bucket is
// irrelevant, every order renders the same frame).  order[n..n+2] = H8, H4,
// H2: the leading tiles to split next frame in 8, 4 and 2 segments: the tiles
// that would outlast the frame's ideal length (total cost / concurrent tile
// slots) by 4x, 2x and 1x, when the heaviest took >= split_us (split_us == 0:
// tests, see below).  One block; resets the costs.
// split thresholds in eighths of the ideal frame length
#ifndef VX_SPLIT_T2
#define VX_SPLIT_T2 8
#endif
#ifndef VX_SPLIT_T4
#define VX_SPLIT_T4 16
#endif
#ifndef VX_SPLIT_T8
#define VX_SPLIT_T8 32
#endif
__device__ __forceinline__ int cost_bucket(unsigned c) {
  if (c < 4) return (int)c;
  const int e = 31 - __clz(c);
  const int b = 4 * e + (int)((c >> (e - 2)) & 3u) - 4;
  return b > 63 ? 63 : b;
}

// A moving camera (rx, ry > 0: the image-space motion between the frames
// whose costs are used, in tiles) orders and splits by the costs dilated
// over that neighbourhood (max filter), so a heavy region that moved one or
// two tiles is still started first and split; the frame-length estimate
// (total) stays the undilated sum.  dil: n words of scratch.
__global__ void __launch_bounds__(1024) tile_order_kernel(uint32_t* __restrict__ cost,
                                                          uint32_t* __restrict__ order, int n,
                                                          int split_us, int slots, int tiles_x,
                                                          int rx, int ry,
                                                          uint32_t* __restrict__ dil) {
  __shared__ unsigned cnt[64];
  __shared__ unsigned long long total;
  __shared__ unsigned top;
  const int tid = threadIdx.x;
  if (tid < 64) cnt[tid] = 0;
  if (tid == 0) {
    total = 0;
    top = 0;
  }
  unsigned long long raw_total = 0;
  const uint32_t* cc = cost;
  if (rx > 0 || ry > 0) {
    const int tiles_y = (n + tiles_x - 1) / tiles_x;
    for (int i = tid; i < n; i += blockDim.x) {
      const int tx = i % tiles_x, ty = i / tiles_x;
      unsigned m = 0;
      for (int dy = -ry; dy <= ry; ++dy) {
        const int y = ty + dy;
        if (y < 0 || y >= tiles_y) continue;
        for (int dx = -rx; dx <= rx; ++dx) {
          const int x = tx + dx;
          const int j = y * tiles_x + x;
          if (x >= 0 && x < tiles_x && j < n) m = max(m, cost[j]);
        }
      }
      dil[i] = m;
      raw_total += cost[i];
    }
    cc = dil;
  }
  __syncthreads();
  const bool dilated = cc != cost;
  unsigned long long my_total = raw_total;  // the frame-length estimate: undilated
  unsigned my_top = 0;
  for (int i = tid; i < n; i += blockDim.x) {
    const unsigned c = cc[i];
    atomicAdd(&cnt[cost_bucket(c)], 1u);
    if (!dilated) my_total += c;
    my_top = max(my_top, c);
  }
  for (int o = 16; o > 0; o >>= 1) {
    my_total += __shfl_xor_sync(0xffffffffu, my_total, o);
    my_top = max(my_top, __shfl_xor_sync(0xffffffffu, my_top, o));
  }
  if ((tid & 31) == 0) {
    atomicAdd(&total, my_total);
    atomicMax(&top, my_top);
  }
  __syncthreads();
  if (tid == 0) {
    // H8: tiles >= 4x the ideal length (split in 8), H4: >= 2x (in 4), H2:
    // >= the ideal (in 2); extra blocks 7*H8 + 3*H4 + H2 within the launch's
    // reserve
    unsigned h8 = 0, h4 = 0, h2 = 0;
    if (split_us == 0) {  // tests: 1/16 of the tiles in 8, 1/8 in 4, 1/8 in 2
      h8 = (unsigned)n / 16;  // (15/16 n extra blocks: fits a reserve of n)
      h4 = (unsigned)n / 8;
      h2 = (unsigned)n / 8;
    } else if (top >= (unsigned)split_us) {
      const unsigned long long ideal = total / (unsigned long long)(slots > 0 ? slots : 1);
      const int b2 = cost_bucket((unsigned)min(ideal * VX_SPLIT_T2 / 8, 0xffffffffull));
      const int b4 = cost_bucket((unsigned)min(ideal * VX_SPLIT_T4 / 8, 0xffffffffull));
      const int b8 = cost_bucket((unsigned)min(ideal * VX_SPLIT_T8 / 8, 0xffffffffull));
      for (int b = 63; b >= b2; --b) (b >= b8 ? h8 : (b >= b4 ? h4 : h2)) += cnt[b];
    }
    // uncapped demand: the launch caps it to its reserve, and the host sizes
    // the next reserve from it
    order[n] = h8;
    order[n + 1] = h4;
    order[n + 2] = h2;
    unsigned run = 0;
    for (int b = 63; b >= 0; --b) {
      const unsigned c = cnt[b];
      cnt[b] = run;
      run += c;
    }
  }
  __syncthreads();
  for (int i = tid; i < n; i += blockDim.x) {
    order[atomicAdd(&cnt[cost_bucket(cc[i])], 1u)] = (uint32_t)i;
    cost[i] = 0;
  }
}

// ---------------------------------------------------------------------------
// march_ray (render.py:426-464) for arbitrary rays

template <int KIND, bool CHECKED>
__global__ void march_rays_kernel(VolView V, MarchD M, FiltD F, const double* __restrict__ lut_g,
                                  const double* __restrict__ origins, const double* __restrict__ dirs,
                                  const double* __restrict__ t_enter, const double* __restrict__ t_exit,
                                  const int32_t* __restrict__ max_steps, int64_t n,
                                  uint8_t* hit_out, int32_t* voxel_out, float* t_out,
                                  double* value_out) {
  __shared__ WarpScratch wsc[4];  // blockDim.x == 128
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = r < n;
  int hx = -1, hy = -1, hz = -1, hidx = 0;
  float ht = 0.0f;
  double hval = 0.0;
  unsigned nsamp = 0;
  RayState R;
  bool live = false;
  int limit = 0;
  if (valid) {
    const double te = t_enter[r], tx = t_exit[r];
    live = tx >= te && M.thr <= 255;
    if (live) {
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        R.o[c] = __double2float_rn(__dadd_rn(origins[3 * r + c], 0.5));
        R.d[c] = __double2float_rn(dirs[3 * r + c]);
      }
      ray_skip_consts(R);
      ray_skip_map(R, V);
      R.base = __double2float_rn(te);
      R.tend = __double2float_rn(tx);
      limit = max_steps[r];
    }
  }
  Diag dg;
  const bool hit = march<KIND, CHECKED, false, true, true, true>(V, M, F, lut_g, R, live, limit, 0, 0, ht,
                                                     hidx, nsamp, dg, &wsc[threadIdx.x >> 5]) == kHit;
  if (hit) {
    voxel_at(R, M, ht, hx, hy, hz);
    hval = filter_value<KIND, CHECKED>(V, F, lut_g, hx, hy, hz);
  }
  if (!valid) return;
  hit_out[r] = hit ? 1 : 0;
  voxel_out[3 * r] = hx;
  voxel_out[3 * r + 1] = hy;
  voxel_out[3 * r + 2] = hz;
  t_out[r] = ht;
  value_out[r] = hval;
}

// K5 apply_filter_batch (filters.py:230-266)
template <int KIND>
__global__ void filter_batch_kernel(VolView V, FiltD F, const double* __restrict__ lut,
                                    const int64_t* __restrict__ xs, const int64_t* __restrict__ ys,
                                    const int64_t* __restrict__ zs, int64_t n, double* out) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  out[r] = F.pairwise ? filter_value<KIND, true, true>(V, F, lut, xs[r], ys[r], zs[r])
                     : filter_value<KIND, true, false>(V, F, lut, xs[r], ys[r], zs[r]);
}

__global__ void sobel_batch_kernel(VolView V, const int64_t* __restrict__ xs,
                                   const int64_t* __restrict__ ys, const int64_t* __restrict__ zs,
                                   int64_t n, const double* __restrict__ fb, double* out) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const double f[3] = {fb[3 * r], fb[3 * r + 1], fb[3 * r + 2]};
  double nn[3];
  sobel<true>(V, xs[r], ys[r], zs[r], f, nn);
  out[3 * r] = nn[0];
  out[3 * r + 1] = nn[1];
  out[3 * r + 2] = nn[2];
}

__global__ void phong_batch_kernel(const double* __restrict__ normals, const double* __restrict__ views,
                                   int64_t n, ShadeD S, uint8_t* out) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const double nn[3] = {normals[3 * r], normals[3 * r + 1], normals[3 * r + 2]};
  const double v[3] = {views[3 * r], views[3 * r + 1], views[3 * r + 2]};
  out[r] = quantise(phong_intensity(nn, v, S));
}

__global__ void ray_dirs_kernel(RayCamD C, double* out) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= (int64_t)C.W * C.H) return;
  double d[3];
  ray_dir(C, (int)(p % C.W), (int)(p / C.W), d);
  out[3 * p] = d[0];
  out[3 * p + 1] = d[1];
  out[3 * p + 2] = d[2];
}

__global__ void ray_spans_kernel(double o0, double o1, double o2, const double* __restrict__ dirs,
                                 int64_t n, int nx, int ny, int nz, double* te, double* tx) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const double o[3] = {o0, o1, o2};
  const double d[3] = {dirs[3 * r], dirs[3 * r + 1], dirs[3 * r + 2]};
  ray_span(o, d, nx, ny, nz, te[r], tx[r]);
}

// ---------------------------------------------------------------------------
// host-side helpers

RayCamD make_cam(const vx_ray_setup* rs) {
  RayCamD C;
  for (int c = 0; c < 3; ++c) {
    C.right[c] = rs->right[c];
    C.up[c] = rs->up[c];
    C.fwd[c] = rs->fwd[c];
    C.origin[c] = rs->origin[c];
  }
  C.tan_f = rs->tan_f;
  C.aspect = rs->aspect;
  C.W = rs->width;
  C.H = rs->height;
  return C;
}

int make_march(const vx_volume* v, const vx_render_params* rp, const vx_filter_config* fc,
               MarchD& M) {
  if (!(rp->step_size > 0.0)) {
    vx_set_error("step_size must be > 0, got %g", rp->step_size);
    return VX_EINVAL;
  }
  if (rp->chunk < 1 || rp->chunk > 16) {
    vx_set_error("chunk must be in [1, 16], got %d", rp->chunk);
    return VX_EINVAL;
  }
  M.s = (float)rp->step_size;  // np.float32(step): round to nearest
  M.inv_s = 1.0f / M.s;
  M.sk_last = M.s * (float)(rp->chunk - 1);
  for (int k = 0; k < 16; ++k) M.sk[k] = M.s * (float)k;
  M.adv = (float)rp->chunk * M.s;
  M.xmax = (float)v->nx;
  M.ymax = (float)v->ny;
  M.zmax = (float)v->nz;
  M.chunk = rp->chunk;
  M.need_clip = rp->need_clip;
  M.explicit_max = rp->max_steps > 0 ? rp->max_steps : 0;
  double T = fc->threshold;
  double c = ceil(T);
  int thr = c < 0.0 ? 0 : (c > 256.0 ? 256 : (int)c);  // max(0, ceil(T)); >255 = no hits
  M.thr = thr;
  M.T = T;
  M.step = rp->step_size;
  M.skip = rp->skip && thr > 0 && thr <= 255;
  {
    // D = 1 (the empty cell itself, at most 4 voxels of the ray): one
    // sample group (8 samples) covers it when step >= 0.5, cheaper than a
    // lookup + skip + re-lookup.  Measured at step 0.5: 2 vs 1 -> bench
    // frame -4 %, C2 LC -7 %, C1 -8..-13 %, C4 -4 %; 3 is slower everywhere
    const char* e = getenv("VOXB200_SKIP_MIN_D");
    M.skip_min_d = e ? atoi(e) : (rp->step_size >= 0.5 ? 2 : 1);
    if (M.skip_min_d < 1) M.skip_min_d = 1;
  }
  return VX_OK;
}

int make_filter(const vx_filter_config* fc, FiltD& F, bool batch_api = false) {
  if (fc->kind < 0 || fc->kind > (batch_api ? kAxisCluster : 5)) {
    vx_set_error("unhandled filter kind %d", fc->kind);
    return VX_EINVAL;
  }
  if (fc->kernel_size < 3 || (fc->kernel_size & 1) == 0) {
    vx_set_error("kernel_size must be odd and >= 3, got %d", fc->kernel_size);
    return VX_EINVAL;
  }
  if (fc->cluster_offset < 1) {
    vx_set_error("cluster_offset must be >= 1, got %d", fc->cluster_offset);
    return VX_EINVAL;
  }
  F.kind = fc->kind;
  F.M = fc->kernel_size;
  F.d = fc->cluster_offset;
  F.pairwise = fc->entropy_pairwise;
  F.band = fc->sigma_band;
  F.okada_t = fc->okada_threshold;
  F.entropy_t = fc->entropy_threshold;
  if (F.pairwise && F.M > 7) {
    vx_set_error("pairwise entropy order supports kernel_size <= 7");
    return VX_EINVAL;
  }
  return VX_OK;
}

int filter_reach(const FiltD& F) {
  const int h = (F.M - 1) / 2;
  if (F.kind == VX_FILTER_LOCAL_CLUSTER) return h + F.d;
  if (F.kind == VX_FILTER_OKADA) return 1;
  if (F.kind == VX_FILTER_NONE) return 0;
  return h;
}

ShadeD make_shade(const vx_render_params* rp) {
  ShadeD S;
  S.ka = rp->ambient;
  S.kd = rp->diffuse;
  S.ks = rp->specular;
  S.shin = rp->shininess;
  for (int c = 0; c < 3; ++c) S.l[c] = rp->light[c];
  S.background = rp->background;
  return S;
}

template <int KIND, bool CHECKED>
void launch_raycast(const RenderArgs& a, int grid, cudaStream_t s) {
  const dim3 blk(kTileW, 4 * kWarpsPerBlock);
  grid *= kBlocksPerTile;
  // unbudgeted launches reserve split_max extra blocks for split tiles
  const int grid_u = grid + (kSplitRays && a.tile_order ? a.split_max : 0);
  // per-pixel diagnostics (hit voxel / t / value / intensity, march counters)
  // are written by the DIAG kernels only
  const bool diag = a.O.diag || a.O.hit_voxel || a.O.hit_t || a.O.hit_value || a.O.intensity;
  if (a.M.explicit_max > 0 && diag)  // exact budget: user max_steps or the re-render
    raycast_kernel<KIND, CHECKED, true, true><<<grid, blk, 0, s>>>(a);
  else if (a.M.explicit_max > 0)
    raycast_kernel<KIND, CHECKED, false, true><<<grid, blk, 0, s>>>(a);
  else if (diag)
    raycast_kernel<KIND, CHECKED, true, false><<<grid_u, blk, 0, s>>>(a);
  else if (!a.M.skip)  // full traversal (skipping off, or thr == 0): lean own-group loads
    raycast_kernel<KIND, CHECKED, false, false, false><<<grid_u, blk, 0, s>>>(a);
  else
    raycast_kernel<KIND, CHECKED, false, false><<<grid_u, blk, 0, s>>>(a);
}

template <bool CHECKED>
void dispatch_raycast(const RenderArgs& a, int grid, cudaStream_t s) {
  switch (a.F.kind) {
    case VX_FILTER_NONE: launch_raycast<VX_FILTER_NONE, CHECKED>(a, grid, s); break;
    case VX_FILTER_MEAN: launch_raycast<VX_FILTER_MEAN, CHECKED>(a, grid, s); break;
    case VX_FILTER_SIGMA: launch_raycast<VX_FILTER_SIGMA, CHECKED>(a, grid, s); break;
    case VX_FILTER_OKADA: launch_raycast<VX_FILTER_OKADA, CHECKED>(a, grid, s); break;
    case VX_FILTER_ENTROPY: launch_raycast<VX_FILTER_ENTROPY, CHECKED>(a, grid, s); break;
    default: launch_raycast<VX_FILTER_LOCAL_CLUSTER, CHECKED>(a, grid, s); break;
  }
}

template <bool CHECKED>
void dispatch_march(const VolView& V, const MarchD& M, const FiltD& F, const double* lut,
                    const double* o, const double* d, const double* te, const double* tx,
                    const int32_t* ms, int64_t n, uint8_t* h, int32_t* vox, float* t, double* val,
                    cudaStream_t s) {
  const int bs = 128;
  const unsigned g = (unsigned)((n + bs - 1) / bs);
#define VX_MR(K) march_rays_kernel<K, CHECKED><<<g, bs, 0, s>>>(V, M, F, lut, o, d, te, tx, ms, n, h, vox, t, val)
  switch (F.kind) {
    case VX_FILTER_NONE: VX_MR(VX_FILTER_NONE); break;
    case VX_FILTER_MEAN: VX_MR(VX_FILTER_MEAN); break;
    case VX_FILTER_SIGMA: VX_MR(VX_FILTER_SIGMA); break;
    case VX_FILTER_OKADA: VX_MR(VX_FILTER_OKADA); break;
    case VX_FILTER_ENTROPY: VX_MR(VX_FILTER_ENTROPY); break;
    default: VX_MR(VX_FILTER_LOCAL_CLUSTER); break;
  }
#undef VX_MR
}

// ---------------------------------------------------------------------------
// accepted-cell occupancy (the filter-aware skip structure)
//
// A sample can end a ray only at a voxel v with raw(v) >= thr AND
// filter(v) >= T (render.py:307-317): a rejected candidate is stepped over
// exactly like an empty sample.  So the set the distance map must guard is
// A = {v : raw >= thr, f(v) >= T}, not every candidate: isolated spots and
// speckle that the filter rejects stop costing samples and filter
// evaluations.  The filter is the march's own filter_value at the same
// template arguments, so membership is bit-identical to what the march
// would decide.  One warp per 32 cells: the lanes vote which cells hold a
// candidate (cell max >= thr), then the warp tests such a cell's 64 voxels,
// 32 at a time, and stops at the first accepted one.

struct LutArg {
  double v[256];
};

struct AccArgs {
  const uint8_t* cmax;  // cell max map at cell (0,0,0)
  uint8_t* occ;         // out: 255 where the cell holds an accepted voxel
  int ncx, ncy, ncz;
  int64_t csy, csz;
  int thr;
  double T;
};

template <int KIND, bool CHECKED>
__global__ void __launch_bounds__(256) accept_cells_kernel(VolView V, FiltD F, AccArgs A,
                                                           LutArg L) {
  __shared__ double lut[KIND == VX_FILTER_ENTROPY ? 256 : 1];
  if (KIND == VX_FILTER_ENTROPY) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) lut[i] = L.v[i];
    __syncthreads();
  }
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const long long nc = (long long)A.ncx * A.ncy * A.ncz;
  const long long ci = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  int cx = 0, cy = 0, cz = 0;
  bool cand = false;
  if (ci < nc) {
    cx = (int)(ci % A.ncx);
    cy = (int)((ci / A.ncx) % A.ncy);
    cz = (int)(ci / ((long long)A.ncx * A.ncy));
    cand = __ldg(A.cmax + (cz * A.csz + cy * A.csy + cx)) >= A.thr;
  }
  // Round 1, one cell per lane: the filter at the cell's first voxel (in
  // the 64-voxel order below) that reaches thr.  Interior cells of an object
  // are accepted here with one evaluation per cell, all lanes in parallel.
  bool unresolved = false;
  if (cand) {
    const int x0 = cx * VX_CELL, y0 = cy * VX_CELL, z0 = cz * VX_CELL;
    int fq = -1;
    for (int q = 0; q < 16 && fq < 0; ++q) {
      const int y = y0 + (q & 3), z = z0 + (q >> 2);
      if (y >= V.ny || z >= V.nz) continue;
      // 4-voxel rows are 4-byte aligned (origin and pitches are multiples of 16)
      const uint32_t w = __ldg(reinterpret_cast<const uint32_t*>(V.origin + z * V.sz + y * V.sy + x0));
      for (int xx = 0; xx < 4; ++xx)
        if (x0 + xx < V.nx && (int)((w >> (8 * xx)) & 0xffu) >= A.thr) {
          fq = 4 * q + xx;
          break;
        }
    }
    if (fq >= 0) {
      if (filter_value<KIND, CHECKED>(V, F, lut, x0 + (fq & 3), y0 + ((fq >> 2) & 3), z0 + (fq >> 4)) >=
          A.T)
        A.occ[(int64_t)cz * A.csz + (int64_t)cy * A.csy + cx] = 255;
      else
        unresolved = true;  // another voxel of the cell may still pass
    }
  }
  // Round 2: cells whose first voxel failed, 32 voxels at a time by the warp
  unsigned todo = __ballot_sync(full, unresolved);
  while (todo) {
    const int src = __ffs(todo) - 1;
    todo &= todo - 1;
    const int x0 = __shfl_sync(full, cx, src) * VX_CELL;
    const int y0 = __shfl_sync(full, cy, src) * VX_CELL;
    const int z0 = __shfl_sync(full, cz, src) * VX_CELL;
    bool acc = false;
    for (int r = 0; r < 2 && !acc; ++r) {
      const int q = r * 32 + lane;
      const int x = x0 + (q & 3), y = y0 + ((q >> 2) & 3), z = z0 + (q >> 4);
      bool pass = false;
      if (x < V.nx && y < V.ny && z < V.nz && rd<false>(V, x, y, z) >= A.thr)
        pass = filter_value<KIND, CHECKED>(V, F, lut, x, y, z) >= A.T;
      acc = __any_sync(full, pass);
    }
    if (acc && lane == 0)
      A.occ[(int64_t)(z0 >> VX_CELL_SHIFT) * A.csz + (int64_t)(y0 >> VX_CELL_SHIFT) * A.csy +
            (x0 >> VX_CELL_SHIFT)] = 255;
  }
}

template <bool CHECKED>
void dispatch_accept(const VolView& V, const FiltD& F, const AccArgs& A, const LutArg& L,
                     unsigned grid, cudaStream_t s) {
#define VX_AC(K) accept_cells_kernel<K, CHECKED><<<grid, 256, 0, s>>>(V, F, A, L)
  switch (F.kind) {
    case VX_FILTER_MEAN: VX_AC(VX_FILTER_MEAN); break;
    case VX_FILTER_SIGMA: VX_AC(VX_FILTER_SIGMA); break;
    case VX_FILTER_OKADA: VX_AC(VX_FILTER_OKADA); break;
    case VX_FILTER_ENTROPY: VX_AC(VX_FILTER_ENTROPY); break;
    default: VX_AC(VX_FILTER_LOCAL_CLUSTER); break;
  }
#undef VX_AC
}

// scratch buffer freed on scope exit (stream ordered)
struct Scratch {
  void* p = nullptr;
  cudaStream_t s;
  explicit Scratch(cudaStream_t st) : s(st) {}
  ~Scratch() {
    if (p) cudaFreeAsync(p, s);
  }
  template <typename T>
  T* get() { return reinterpret_cast<T*>(p); }
};

}  // namespace

// Force the lazy module loader to bring in the frame kernels of the paper's
// filter (and the unfiltered one) now, at volume creation, instead of inside
// the first frame (cudaFuncGetAttributes loads the function).
static int demand_arena_init();

int vx_preload_render_kernels() {
  cudaFuncAttributes fa;
  VX_CUDA(cudaFuncGetAttributes(&fa, raycast_kernel<VX_FILTER_LOCAL_CLUSTER, false, false, false>));
  VX_CUDA(cudaFuncGetAttributes(&fa, raycast_kernel<VX_FILTER_NONE, false, false, false>));
  VX_CUDA(cudaFuncGetAttributes(&fa, tile_order_kernel));
  VX_CUDA(cudaFuncGetAttributes(&fa, accept_cells_kernel<VX_FILTER_LOCAL_CLUSTER, false>));
  return demand_arena_init();
}

// VOXB200_TRACE=1: host wall-clock phases of vx_render on stderr (cold-path
// diagnosis: map builds, allocations, copies)
static bool trace_on() {
  static const bool on = [] {
    const char* e = getenv("VOXB200_TRACE");
    return e && atoi(e) != 0;
  }();
  return on;
}
static double trace_us() {
  return std::chrono::duration<double, std::micro>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}
#define VX_TRACE(label, t0)                                                       \
  do {                                                                            \
    if (trace_on()) {                                                             \
      const double _t = trace_us();                                               \
      fprintf(stderr, "[vx_trace] %-18s %9.1f us\n", label, _t - (t0));          \
      t0 = _t;                                                                    \
    }                                                                             \
  } while (0)

#ifndef VX_ORDER_FRESH
#define VX_ORDER_FRESH 1
#endif

// Cost dilation of the tile order for a moving camera (VOXB200_DILATE=1).
// Measured (scripts/orbit_probe.py, 1 degree per frame): device p50 0.194
// ms dilated vs 0.159 ms on the plain k-2 costs -- the max filter turns the
// heavy region into a plateau that over-splits and loses the order -- so it
// is off by default.
static bool dilate_moving() {
  static const bool on = [] {
    const char* e = getenv("VOXB200_DILATE");
    return e && atoi(e) != 0;
  }();
  return on;
}

// Orthant skip maps: VOXB200_ORTHANT=0 renders on the
// two-sided Chebyshev maps only
static bool orthant_maps_on() {
  static const bool on = [] {
    const char* e = getenv("VOXB200_ORTHANT");
    return !e || atoi(e) != 0;
  }();
  return on;
}

// The direction orthants of a frame's primary rays.  d = (fwd + u right) +
// v up before normalisation (which keeps signs) is affine in the pixel's
// (u, v), so per axis its range over the image is spanned by the four
// corner pixels; an axis whose range reaches within 1e-9 of zero may be
// either sign.  A ray whose orthant is not in the set falls back to the
// two-sided map on the device, so this only decides what gets built.
static unsigned frame_octants(const vx_ray_setup* rs) {
  const double W = rs->width, H = rs->height;
  const double us[2] = {((2.0 * 0.5) / W - 1.0) * rs->tan_f * rs->aspect,
                        ((2.0 * (W - 0.5)) / W - 1.0) * rs->tan_f * rs->aspect};
  const double vs[2] = {(1.0 - (2.0 * 0.5) / H) * rs->tan_f, (1.0 - (2.0 * (H - 0.5)) / H) * rs->tan_f};
  unsigned can_pos = 0, can_neg = 0;
  for (int a = 0; a < 3; ++a) {
    double lo = 1e300, hi = -1e300;
    for (double u : us)
      for (double v : vs) {
        const double d = (rs->fwd[a] + u * rs->right[a]) + v * rs->up[a];
        lo = d < lo ? d : lo;
        hi = d > hi ? d : hi;
      }
    if (hi > -1e-9) can_pos |= 1u << a;
    if (lo < 1e-9) can_neg |= 1u << a;
  }
  unsigned mask = 0;
  for (int o = 0; o < 8; ++o) {
    bool ok = true;
    for (int a = 0; a < 3; ++a) ok = ok && (((o >> a) & 1) ? (can_neg >> a) & 1 : (can_pos >> a) & 1);
    if (ok) mask |= 1u << o;
  }
  return mask;
}

// Accepted-cell distance map for the render's filter setting (nullptr: use
// the raw candidate map).  Policy: a setting seen for the first time renders
// on the raw map (one-shot frames such as a filter comparison pay nothing);
// from its second frame on the map is built once (~1 ms at 1024^3) and kept
// in a small LRU on the volume.  VOXB200_ACCEPT_MAP=0 disables it, =eager
// builds on first sight.
static int get_accept_map(vx_volume* v, const RenderArgs& a, bool checked, const uint8_t** out,
                          MapSlot** slot_out, cudaStream_t s) {
  *out = nullptr;
  *slot_out = nullptr;
  static const int mode = [] {
    const char* e = getenv("VOXB200_ACCEPT_MAP");
    if (!e) return 1;
    if (!strcmp(e, "eager")) return 2;
    return atoi(e) ? 1 : 0;
  }();
  if (!mode || a.F.kind == VX_FILTER_NONE || !a.M.skip) return VX_OK;
  struct Key {
    int32_t kind, M, d, thr;
    double T, band, okada_t, entropy_t;
    double lut[256];
  } key;
  static_assert(sizeof(Key) == VX_ACC_KEY_BYTES, "accept key layout");
  memset(&key, 0, sizeof(key));
  key.kind = a.F.kind;
  key.M = a.F.M;
  key.d = a.F.kind == VX_FILTER_LOCAL_CLUSTER ? a.F.d : 0;
  key.thr = a.M.thr;
  key.T = a.M.T;
  if (a.F.kind == VX_FILTER_SIGMA) key.band = a.F.band;
  if (a.F.kind == VX_FILTER_OKADA) key.okada_t = a.F.okada_t;
  if (a.F.kind == VX_FILTER_ENTROPY) {
    key.entropy_t = a.F.entropy_t;
    memcpy(key.lut, a.lut_host, sizeof(key.lut));
  }
  std::lock_guard<std::mutex> lock(v->mu);
  ++v->stamp;
  AccEntry* e = nullptr;
  for (auto& c : v->acc)
    if (c.valid && !memcmp(c.key, &key, sizeof(key))) e = &c;
  if (e && e->built) {
    e->stamp = v->stamp;
    int rc = vx_map_pin(e, s);
    if (rc) return rc;
    *out = e->map;
    *slot_out = e;
    return VX_OK;
  }
  if (!e) {
    for (auto& c : v->acc) {
      if (c.pins) continue;  // a render between lookup and launch still reads it
      if (!c.valid) {
        e = &c;
        break;
      }
      if (!e || c.stamp < e->stamp) e = &c;
    }
    if (!e) return VX_OK;  // every slot in flight: the raw candidate map
    // the slot's old map is overwritten only after its last readers
    // (vx_map_claim below orders the build after their use events)
    e->valid = true;
    e->built = false;
    memcpy(e->key, &key, sizeof(key));
    e->stamp = v->stamp;
    if (mode == 1) return VX_OK;  // first sight: raw map
  }
  double tt = trace_on() ? trace_us() : 0.0;
  e->valid = false;  // until built
  int rc = vx_map_claim(v, e, s);
  if (rc) return rc;
  // the occupancy stays with the slot: the orthant maps are built from it
  if (!e->occ) VX_CUDA(cudaMalloc(&e->occ, v->cmap_bytes));
  uint8_t* occ = e->occ;
  VX_CUDA(cudaMemsetAsync(occ, 0, v->cmap_bytes, s));
  VX_CUDA(cudaMemsetAsync(e->map, 0, v->map_bytes, s));  // coarse level unused: no skip
  VX_TRACE("  acc scratch", tt);
  AccArgs A;
  A.cmax = v->cmax + v->csz + v->csy + 1;
  A.occ = occ + v->csz + v->csy + 1;
  A.ncx = v->ncx;
  A.ncy = v->ncy;
  A.ncz = v->ncz;
  A.csy = v->csy;
  A.csz = v->csz;
  A.thr = a.M.thr;
  A.T = a.M.T;
  LutArg L;
  memcpy(L.v, a.lut_host, sizeof(L.v));
  const int64_t nc = (int64_t)v->ncx * v->ncy * v->ncz;
  const unsigned grid = (unsigned)((nc + 255) / 256);
  if (checked)
    dispatch_accept<true>(a.V, a.F, A, L, grid, s);
  else
    dispatch_accept<false>(a.V, a.F, A, L, grid, s);
  VX_CHECK_LAUNCH();
  rc = vx_launch_dist_cells(v, occ, e->map + v->map_bytes, 1, s);
  if (rc) return rc;
  e->occ_src = occ;
  e->occ_thr = 1;
  VX_TRACE("  acc launches", tt);
  // other streams wait on the slot's ready event (no host sync under mu)
  if ((rc = vx_map_publish(v, e, s))) return rc;
  if ((rc = vx_map_pin(e, s))) return rc;
  e->valid = true;
  e->built = true;
  e->stamp = v->stamp;
  *out = e->map;
  *slot_out = e;
  return VX_OK;
}

// unpins a cached map slot when the render that looked it up returns (its
// K4 is enqueued by then, or it failed)
struct SlotPin {
  vx_volume* v;
  cudaStream_t s;
  MapSlot* m = nullptr;
  SlotPin(vx_volume* vol, cudaStream_t st) : v(vol), s(st) {}
  ~SlotPin() { vx_map_release(v, m, s); }
};

// ===========================================================================
// exported entry points

// Adaptive tile order: K4 records each tile's duration; a one-block kernel
// turns them into the next frame's order, heaviest first, so the longest
// warps (rays threading cluttered free space) start at once instead of
// setting the frame's tail.  Any order renders the same frame (tiles are
// independent), so stale costs only cost time.  Per calling thread, keyed by
// (volume, frame size, partition, stream); VOXB200_TILE_ORDER=0 disables.
//
// Double-buffered off the frame's critical path: frame k (parity p = k & 1)
// renders in the order computed from frame k-2's costs (buf[p]) and records
// its own costs into buf[p]; the ordering kernel for them then runs on a side
// stream, concurrently with frame k+1 (which uses buf[p ^ 1]).  In-stream it
// cost ~13 us of a ~160 us frame (one latency-bound block).
constexpr int kSchedHdr = 4;  // u32 slots between order[] and cost[]
struct TileSched {
  const void* vol = nullptr;
  int w = 0, h = 0, rank = 0, world = 0, grid = 0;
  cudaStream_t stream = nullptr;
  uint32_t* buf[2] = {nullptr, nullptr};     // order[grid], H8, H4, H2, pad, then cost[grid]
  uint32_t* demand[2] = {nullptr, nullptr};  // pinned host copies of H8, H4, H2, pad
  bool valid[2] = {false, false};
  int parity = 0;
  cudaStream_t side = nullptr;  // ordering kernels
  cudaEvent_t costs_done[2] = {nullptr, nullptr}, order_done[2] = {nullptr, nullptr};
  int device = -1;
  vx_ray_setup last_rs[2];  // camera of the frame that recorded costs into buf[p]
  bool have_rs[2] = {false, false};
  vx_ray_setup prev_rs;  // camera of the previous frame on this schedule
  bool have_prev = false;
};
// a thread's schedules, one per (volume, frame size, partition, stream):
// a thread alternating between frames of several kinds -- or enqueueing
// every device's tiles of a multi-device frame (vx_multi.cu) -- keeps each
// schedule instead of rebuilding one (LRU of 8)
constexpr int kSchedSlots = 8;
static thread_local TileSched tl_sched[kSchedSlots];
static thread_local uint64_t tl_sched_use[kSchedSlots];
static thread_local uint64_t tl_sched_clock = 0;

// scheduling knobs (vx_set_schedule): order on/off, smallest grid (in tiles,
// -1 = 4 waves of SMs) that gets an order, split threshold (us), split cap
// (tiles = grid / div)
static std::atomic<int> g_sched_order{-1}, g_sched_min_grid{-1}, g_sched_split_us{16},
    g_sched_split_div{4};

extern "C" int vx_set_schedule(int32_t tile_order, int32_t min_grid_tiles, int32_t split_min_us,
                               int32_t split_max_div) {
  if (split_max_div < 1 || split_min_us < 0) {
    vx_set_error("vx_set_schedule: split_max_div must be >= 1 and split_min_us >= 0");
    return VX_EINVAL;
  }
  g_sched_order = tile_order;
  g_sched_min_grid = min_grid_tiles;
  g_sched_split_us = split_min_us;
  g_sched_split_div = split_max_div;
  return VX_OK;
}

// page-locked split-demand slots for the per-thread schedules, carved from one
// arena allocated with the frame kernels' preload (a cudaHostAlloc inside the
// first frame measured ~1-3 ms)
static std::mutex g_demand_mu;
static uint32_t* g_demand_arena = nullptr;
static int g_demand_used = 0;
constexpr int kDemandSlots = 256;

static int demand_arena_init() {
  std::lock_guard<std::mutex> lk(g_demand_mu);
  if (!g_demand_arena)
    VX_CUDA(cudaHostAlloc(&g_demand_arena, 4 * kSchedHdr * kDemandSlots, cudaHostAllocDefault));
  return VX_OK;
}

static uint32_t* demand_slot() {
  std::lock_guard<std::mutex> lk(g_demand_mu);
  if (!g_demand_arena || g_demand_used >= kDemandSlots) return nullptr;
  return g_demand_arena + kSchedHdr * g_demand_used++;
}

static int tile_sched(vx_volume* vol, const vx_ray_setup* rs, int rank, int world, int grid,
                      cudaStream_t s, TileSched** out) {
  static const bool env_on = [] {
    const char* e = getenv("VOXB200_TILE_ORDER");
    return !e || atoi(e) != 0;
  }();
  *out = nullptr;
  const int order = g_sched_order.load();
  const bool enabled = order < 0 ? env_on : order != 0;
  // small frames fit in one wave of blocks: nothing to reorder
  const int min_grid = g_sched_min_grid.load() < 0 ? 4 * vx_sm_count() : g_sched_min_grid.load();
  if (!enabled || grid < min_grid) return VX_OK;
  int cur_dev = 0;
  VX_CUDA(cudaGetDevice(&cur_dev));
  int pick = -1;
  for (int i = 0; i < kSchedSlots && pick < 0; ++i) {
    const TileSched& c = tl_sched[i];
    if (c.vol == vol && c.w == rs->width && c.h == rs->height && c.rank == rank &&
        c.world == world && c.grid == grid && c.stream == s && c.device == cur_dev && c.buf[0])
      pick = i;
  }
  if (pick < 0) {  // least recently used slot (an empty one first)
    pick = 0;
    for (int i = 1; i < kSchedSlots; ++i)
      if (tl_sched_use[i] < tl_sched_use[pick]) pick = i;
  }
  tl_sched_use[pick] = ++tl_sched_clock;
  TileSched& t = tl_sched[pick];
  int dev = 0;
  VX_CUDA(cudaGetDevice(&dev));
  if (t.device != dev) {  // per-thread side stream and events of this device
    if (t.side) {  // the slot served another device: release its resources there
      VX_CUDA(cudaSetDevice(t.device));
      VX_CUDA(cudaStreamSynchronize(t.side));
      if (t.stream) VX_CUDA(cudaStreamSynchronize(t.stream));
      for (int p = 0; p < 2; ++p) {
        if (t.buf[p]) VX_CUDA(cudaFree(t.buf[p]));
        VX_CUDA(cudaEventDestroy(t.costs_done[p]));
        VX_CUDA(cudaEventDestroy(t.order_done[p]));
        t.valid[p] = false;
      }
      VX_CUDA(cudaStreamDestroy(t.side));
      VX_CUDA(cudaSetDevice(dev));
      t.vol = nullptr;  // rebuilt below
    }
    VX_CUDA(cudaStreamCreateWithFlags(&t.side, cudaStreamNonBlocking));
    for (int p = 0; p < 2; ++p) {
      VX_CUDA(cudaEventCreateWithFlags(&t.costs_done[p], cudaEventDisableTiming));
      VX_CUDA(cudaEventCreateWithFlags(&t.order_done[p], cudaEventDisableTiming));
    }
    t.device = dev;
    t.buf[0] = t.buf[1] = nullptr;
  }
  if (t.vol != vol || t.w != rs->width || t.h != rs->height || t.rank != rank ||
      t.world != world || t.grid != grid || t.stream != s || !t.buf[0]) {
    VX_CUDA(cudaStreamSynchronize(t.side));
    for (int p = 0; p < 2; ++p) {
      if (t.buf[p]) {
        VX_CUDA(cudaStreamSynchronize(t.stream));
        VX_CUDA(cudaFreeAsync(t.buf[p], t.stream));
        t.buf[p] = nullptr;
      }
      // stream-ordered pool (no device-wide cudaMalloc inside a frame)
      // order[grid], header, cost[grid], dilated cost[grid]
      VX_CUDA(vx_malloc_async(&t.buf[p], (size_t)grid * 12 + 4 * kSchedHdr, s));
      if (!t.demand[p]) t.demand[p] = demand_slot();
      if (!t.demand[p]) VX_CUDA(cudaHostAlloc(&t.demand[p], 4 * kSchedHdr, cudaHostAllocDefault));
      for (int k = 0; k < kSchedHdr; ++k) t.demand[p][k] = 0;
      VX_CUDA(cudaMemsetAsync(t.buf[p] + grid + kSchedHdr, 0, (size_t)grid * 4, s));
      t.valid[p] = false;
      t.have_rs[p] = false;
      t.have_prev = false;
    }
    t.vol = vol;
    t.w = rs->width;
    t.h = rs->height;
    t.rank = rank;
    t.world = world;
    t.grid = grid;
    t.stream = s;
    t.parity = 0;
  }
  *out = &t;
  return VX_OK;
}

// the order of frame k + 2 from frame k's costs (tile_order_kernel + the
// split-demand read back), on the side stream behind this frame's K4
struct OrderJob {
  TileSched* ts = nullptr;
  int grid = 0;
  int tiles_x = 0, rx = 0, ry = 0;  // camera motion in tiles (dilation radius)
  int min_warps = VX_RAYCAST_MIN_WARPS;  // resident warps per SM of the frame kernel
};

// Image-space motion of the volume between two cameras, in tiles: the
// largest displacement of the box corners and centre, per axis (capped at 4;
// 4 when a point lies behind either camera).  Drives the cost dilation of
// the tile order for a moving camera (0 for a static one).
static void camera_motion_tiles(const vx_ray_setup* a, const vx_ray_setup* b, const vx_volume* v,
                                int* rx, int* ry) {
  *rx = *ry = 0;
  if (!memcmp(a, b, sizeof(vx_ray_setup))) return;
  const double lo = -0.5, hi[3] = {v->nx - 0.5, v->ny - 0.5, v->nz - 0.5};
  double dxm = 0.0, dym = 0.0;
  for (int k = 0; k < 9; ++k) {
    double P[3];
    for (int c = 0; c < 3; ++c)
      P[c] = k == 8 ? 0.5 * (lo + hi[c]) : (((k >> c) & 1) ? hi[c] : lo);
    double px[2], py[2];
    const vx_ray_setup* cs[2] = {a, b};
    for (int i = 0; i < 2; ++i) {
      const vx_ray_setup* r = cs[i];
      double q[3], z = 0.0, u = 0.0, w = 0.0;
      for (int c = 0; c < 3; ++c) q[c] = P[c] - r->origin[c];
      for (int c = 0; c < 3; ++c) {
        z += q[c] * r->fwd[c];
        u += q[c] * r->right[c];
        w += q[c] * r->up[c];
      }
      if (z <= 1e-6) {
        *rx = *ry = 4;
        return;
      }
      px[i] = (u / z / (r->tan_f * r->aspect) + 1.0) * 0.5 * r->width;
      py[i] = (1.0 - w / z / r->tan_f) * 0.5 * r->height;
    }
    dxm = fmax(dxm, fabs(px[1] - px[0]));
    dym = fmax(dym, fabs(py[1] - py[0]));
  }
  *rx = (int)fmin(4.0, ceil(dxm / kTileW));
  *ry = (int)fmin(4.0, ceil(dym / kTileH));
}

static int order_tiles(const OrderJob& j, cudaStream_t s) {
  if (!j.ts) return VX_OK;
  TileSched* ts = j.ts;
  const int p = ts->parity;
  uint32_t* b = ts->buf[p];
  VX_CUDA(cudaEventRecord(ts->costs_done[p], s));
  VX_CUDA(cudaStreamWaitEvent(ts->side, ts->costs_done[p], 0));
  tile_order_kernel<<<1, 1024, 0, ts->side>>>(b + j.grid + kSchedHdr, b, j.grid,
                                              g_sched_split_us.load(),
                                              vx_sm_count() * (j.min_warps / kWarpsPerBlock),
                                              j.tiles_x, j.rx, j.ry,
                                              b + 2 * j.grid + kSchedHdr);
  VX_CHECK_LAUNCH();
  // the split demand, read back without a sync: it sizes a later frame's
  // reserve of extra blocks (a stale value only costs time)
  VX_CUDA(cudaMemcpyAsync(ts->demand[p], b + j.grid, 4 * kSchedHdr, cudaMemcpyDeviceToHost,
                          ts->side));
  VX_CUDA(cudaEventRecord(ts->order_done[p], ts->side));
  ts->valid[p] = true;
  ts->parity = p ^ 1;
  return VX_OK;
}

static int render_impl(vx_volume* vol, const vx_ray_setup* rs, const vx_render_params* rp,
                       const vx_filter_config* fc, const vx_partition* part, vx_render_out* o,
                       cudaStream_t s, int explicit_budget_override, OrderJob* defer = nullptr,
                       bool sys_atomics = false) {
  if (!vol || !rs || !rp || !fc || !o || !o->pixels) {
    vx_set_error("vx_render: null argument");
    return VX_EINVAL;
  }
  if (rs->width < 1 || rs->height < 1) {
    vx_set_error("image size must be >= 1x1, got %dx%d", rs->width, rs->height);
    return VX_EINVAL;
  }
  RenderArgs a;
  a.C = make_cam(rs);
  int rc = make_march(vol, rp, fc, a.M);
  if (rc) return rc;
  if (explicit_budget_override > 0) a.M.explicit_max = explicit_budget_override;
  rc = make_filter(fc, a.F);
  if (rc) return rc;
  a.S = make_shade(rp);
  a.lut_host = fc->entropy_lut;
  a.lut = nullptr;
  // released (stream-ordered) when this function returns, behind the launch
  Scratch lut_dev(s);
  if (a.F.kind == VX_FILTER_ENTROPY) {
    VX_CUDA(vx_malloc_async(reinterpret_cast<double**>(&lut_dev.p), sizeof(fc->entropy_lut), s));
    VX_CUDA(cudaMemcpyAsync(lut_dev.p, fc->entropy_lut, sizeof(fc->entropy_lut),
                            cudaMemcpyHostToDevice, s));
    a.lut = lut_dev.get<double>();
  }
  const bool checked = filter_reach(a.F) > VX_PAD - 1;
  const uint8_t* dist = nullptr;
  double tt = trace_on() ? trace_us() : 0.0;
  SlotPin pin(vol, s);  // released when this function returns (after the K4 launch)
  if (a.M.skip) {
    a.V = vx_view(vol, nullptr);
    rc = get_accept_map(vol, a, checked, &dist, &pin.m, s);
    if (rc) return rc;
    VX_TRACE("accept_map", tt);
    if (!dist) rc = vx_get_dist_map(vol, a.M.thr, &dist, &pin.m, s);
    if (rc) return rc;
    VX_TRACE("dist_map", tt);
    // every map slot in flight (more concurrent settings than slots): no
    // skipping for this frame (exact either way)
    if (!dist) a.M.skip = 0;
  }
  a.V = vx_view(vol, dist);
  if (dist && pin.m && orthant_maps_on()) {
    // the orthant maps of the directions this frame's rays take
    unsigned built = 0;
    {
      std::lock_guard<std::mutex> lock(vol->mu);
      rc = vx_map_octants(vol, pin.m, frame_octants(rs), &built, s);
    }
    if (rc) return rc;
    VX_TRACE("orthant_maps", tt);
    if (built) {
      a.V.doct = pin.m->oct + vol->csz + vol->csy + 1;
      a.V.oct_stride = (int64_t)vol->cmap_bytes;
      a.V.oct_mask = (int)built;
#ifdef VX_DEBUG_CHECKS
      a.V.dolo = pin.m->oct;
      a.V.dohi = pin.m->oct + 8 * vol->cmap_bytes;
#endif
    }
  }
  a.O.pixels = o->pixels;
  a.O.hit_voxel = o->hit_voxel;
  a.O.hit_t = o->hit_t;
  a.O.hit_value = o->hit_value;
  a.O.intensity = o->intensity;
  a.O.image_hist = reinterpret_cast<unsigned long long*>(o->image_hist);
  a.O.hit_count = reinterpret_cast<unsigned long long*>(o->hit_count);
  a.O.samples = reinterpret_cast<unsigned long long*>(o->samples);
  a.O.diag = reinterpret_cast<unsigned long long*>(o->diag);
  a.O.trunc_flag = o->trunc_flag;
  a.O.sys = sys_atomics ? 1 : 0;
  a.world = part ? part->world : 1;
  a.rank = part ? part->rank : 0;
  if (a.world < 1 || a.rank < 0 || a.rank >= a.world) {
    vx_set_error("bad partition rank %d of %d", a.rank, a.world);
    return VX_EINVAL;
  }
  a.tiles_x = (rs->width + kTileW - 1) / kTileW;
  const int tiles_y = (rs->height + kTileH - 1) / kTileH;
  a.n_tiles = a.tiles_x * tiles_y;
  const int grid = (a.n_tiles - a.rank + a.world - 1) / a.world;
  if (grid <= 0) return VX_OK;
  TileSched* ts = nullptr;
  a.tile_order = nullptr;
  a.tile_cost = nullptr;
  rc = tile_sched(vol, rs, a.rank, a.world, grid, s, &ts);
  if (rc) return rc;
  a.owned_tiles = grid;
  // ray splitting pays where heavy tiles are bound by the dependent lookup
  // chain; the entropy filter's heavy tiles are bound by filter evaluations
  // of rejected candidates, which a second segment only multiplies
  // (C3 entropy 0.245 -> 0.345 ms measured), so it is not split.  The
  // reserve of extra blocks follows the last known demand (spare blocks
  // still cost a launch slot each).
  a.split_min_chunks = g_sched_split_us.load() == 0 ? 1 : 8;
  a.split_max = a.F.kind == VX_FILTER_ENTROPY && g_sched_split_us.load() != 0
                    ? 0
                    : grid / g_sched_split_div.load();
  if (ts) {
    const int p = ts->parity;
    // this frame records its costs in buf[p] and renders in the order the
    // side stream computed there from frame k - 2 (after its order is done).
    // A moving camera renders in the order of frame k - 1's costs instead
    // (buf[p ^ 1], computed on the side stream right behind that frame): the
    // heavy tiles move ~2 tiles per degree of orbit, and a 2-frame-old order
    // left them unsplit and late (profiles/r2/r2_ab_misc.txt).  The wait is
    // then on the previous frame's ordering kernel.
    const bool moving = VX_ORDER_FRESH && ts->have_prev &&
                        memcmp(&ts->prev_rs, rs, sizeof(vx_ray_setup)) != 0;
    ts->prev_rs = *rs;
    ts->have_prev = true;
    const int q = moving && ts->valid[p ^ 1] ? p ^ 1 : p;
    if (ts->valid[q]) VX_CUDA(cudaStreamWaitEvent(s, ts->order_done[q], 0));
    a.tile_cost = ts->buf[p] + grid + kSchedHdr;
    a.tile_order = ts->valid[q] ? ts->buf[q] : nullptr;
    if (ts->valid[q]) {
      const uint32_t* dm = ts->demand[q];
      const long long want = 7ll * dm[0] + 3ll * dm[1] + dm[2];
      const long long reserve = want + want / 4 + 32;
      if (reserve < a.split_max) a.split_max = (int)reserve;
    }
  }
  VX_TRACE("tile_sched", tt);
  if (checked)
    dispatch_raycast<true>(a, grid, s);
  else
    dispatch_raycast<false>(a, grid, s);
  VX_CHECK_LAUNCH();
  VX_TRACE("k4_launch", tt);
  OrderJob job;
  job.ts = ts;
  job.grid = grid;
  job.tiles_x = a.tiles_x;
  job.min_warps = raycast_min_warps(a.F.kind);
  if (ts && a.world == 1 && dilate_moving()) {
    // the order this frame's costs produce serves frame k + 2: expect the
    // camera to keep moving as it did from frame k - 2 (whose costs buf[p]
    // held) to this frame
    const int p = ts->parity;
    if (ts->have_rs[p]) camera_motion_tiles(&ts->last_rs[p], rs, vol, &job.rx, &job.ry);
    ts->last_rs[p] = *rs;
    ts->have_rs[p] = true;
  }
  if (defer) {
    *defer = job;
    return VX_OK;
  }
  return order_tiles(job, s);
}

// exact frame budget of render.py:469-473
static int frame_budget(vx_volume* vol, const vx_ray_setup* rs, double step, cudaStream_t s,
                        int* budget) {
  RayCamD C = make_cam(rs);
  Scratch sc(s);
  VX_CUDA(vx_malloc_async(reinterpret_cast<unsigned long long**>(&sc.p), 8, s));
  VX_CUDA(cudaMemsetAsync(sc.p, 0, 8, s));
  const int n = rs->width * rs->height;
  span_max_kernel<<<(n + 255) / 256, 256, 0, s>>>(C, vol->nx, vol->ny, vol->nz,
                                                   sc.get<unsigned long long>());
  VX_CHECK_LAUNCH();
  unsigned long long bits = 0;
  VX_CUDA(cudaMemcpyAsync(&bits, sc.p, 8, cudaMemcpyDeviceToHost, s));
  VX_CUDA(cudaStreamSynchronize(s));
  double longest;
  memcpy(&longest, &bits, 8);
  double q = ceil(longest / step);
  long long b = (long long)q + 1;
  if (b < 1) b = 1;
  if (b > INT_MAX) b = INT_MAX;
  *budget = (int)b;
  return VX_OK;
}

extern "C" int vx_render_device(vx_volume* vol, const vx_ray_setup* rs, const vx_render_params* rp,
                                const vx_filter_config* fc, const vx_partition* part,
                                vx_render_out* dev_out, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  return render_impl(vol, rs, rp, fc, part, dev_out, s, 0);
}

// K4 over a rank's tiles straight into another rank's frame (vx_group.cu)
int vx_render_tiles(vx_volume* vol, const vx_ray_setup* rs, const vx_render_params* rp,
                    const vx_filter_config* fc, const vx_partition* part, vx_render_out* dev_out,
                    cudaStream_t s, bool sys_atomics) {
  return render_impl(vol, rs, rp, fc, part, dev_out, s, 0, nullptr, sys_atomics);
}

// per-thread frame timing events (vx_last_render_ms)
static thread_local cudaEvent_t tl_ev[2] = {nullptr, nullptr};
static thread_local int tl_ev_device = -1;
static thread_local float tl_render_ms = -1.0f;
static thread_local bool tl_frame_timing = false;

extern "C" int vx_set_frame_timing(int on) {
  tl_frame_timing = on != 0;
  return VX_OK;
}

extern "C" int vx_last_render_ms(float* ms_out) {
  if (!ms_out) {
    vx_set_error("vx_last_render_ms: null argument");
    return VX_EINVAL;
  }
  *ms_out = tl_render_ms;
  return VX_OK;
}

static thread_local cudaEvent_t tl_copy_ev = nullptr;
static thread_local int tl_copy_dev = -1;

static cudaError_t copy_event(cudaEvent_t* ev) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (!tl_copy_ev || tl_copy_dev != dev) {
    e = cudaEventCreateWithFlags(&tl_copy_ev, cudaEventDisableTiming);
    if (e != cudaSuccess) return e;
    tl_copy_dev = dev;
  }
  *ev = tl_copy_ev;
  return cudaSuccess;
}

static int timing_events(cudaEvent_t** ev) {
  int dev = 0;
  VX_CUDA(cudaGetDevice(&dev));
  if (!tl_ev[0] || tl_ev_device != dev) {
    VX_CUDA(cudaEventCreate(&tl_ev[0]));
    VX_CUDA(cudaEventCreate(&tl_ev[1]));
    tl_ev_device = dev;
  }
  *ev = tl_ev;
  return VX_OK;
}

extern "C" int vx_render(vx_volume* vol, const vx_ray_setup* rs, const vx_render_params* rp,
                         const vx_filter_config* fc, const vx_partition* part, vx_render_out* out) {
  if (!vol || !rs || !rp || !fc || !out || !out->pixels) {
    vx_set_error("vx_render: null argument");
    return VX_EINVAL;
  }
  if (rs->width < 1 || rs->height < 1) {
    vx_set_error("image size must be >= 1x1, got %dx%d", rs->width, rs->height);
    return VX_EINVAL;
  }
  double tv = trace_on() ? trace_us() : 0.0;
  cudaStream_t s = vx_stream();
  const size_t npx = (size_t)rs->width * rs->height;
  // device staging: pixels | hit_voxel | hit_t | hit_value | intensity | hist | counters
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += (bytes + 255) & ~size_t(255);
    return o;
  };
  const size_t o_pix = take(npx);
  const size_t o_vox = out->hit_voxel ? take(npx * 12) : 0;
  const size_t o_t = out->hit_t ? take(npx * 4) : 0;
  const size_t o_val = out->hit_value ? take(npx * 8) : 0;
  const size_t o_int = out->intensity ? take(npx * 8) : 0;
  // the Python frame pool lays the counters out right behind the pixels (at
  // npx rounded to 64 B) in the same page-locked buffer: then one copy brings
  // pixels and counters back (saves a copy's fixed latency per frame)
  const size_t o_fused = (npx + 63) & ~size_t(63);
  const bool fused = !out->hit_voxel && !out->hit_t && !out->hit_value && !out->intensity &&
                     !out->diag && out->image_hist &&
                     reinterpret_cast<uint8_t*>(out->image_hist) == out->pixels + o_fused &&
                     out->hit_count == out->image_hist + 256 &&
                     out->samples == out->image_hist + 257;
  if (fused) off = o_fused;
  const size_t o_small = take(256 * 8 + 3 * 8 + 8 + 64);
  // per-thread staging, kept between frames (this call synchronises before
  // returning, so the next frame on this thread may reuse it)
  // (one per (thread, device): the stream is vx_stream()'s of that device)
  static thread_local struct Staging {
    uint8_t* p = nullptr;
    size_t cap = 0;
  } staging[64];
  {
    int dev = 0;
    VX_CUDA(cudaGetDevice(&dev));
    Staging& sg = staging[dev & 63];
    if (!sg.p || sg.cap < off) {
      if (sg.p) VX_CUDA(cudaFreeAsync(sg.p, s));
      sg.p = nullptr;
      VX_CUDA(vx_malloc_async(&sg.p, off, s));
      sg.cap = off;
    }
  }
  int cur_dev = 0;
  VX_CUDA(cudaGetDevice(&cur_dev));
  Staging& st = staging[cur_dev & 63];
  uint8_t* base = st.p;
  VX_CUDA(cudaMemsetAsync(base + o_small, 0, 256 * 8 + 3 * 8 + 8 + 64, s));
  if (part && part->world > 1) VX_CUDA(cudaMemsetAsync(base + o_pix, 0, npx, s));
  VX_TRACE("staging", tv);
  vx_render_out d;
  d.pixels = base + o_pix;
  d.hit_voxel = out->hit_voxel ? reinterpret_cast<int32_t*>(base + o_vox) : nullptr;
  d.hit_t = out->hit_t ? reinterpret_cast<float*>(base + o_t) : nullptr;
  d.hit_value = out->hit_value ? reinterpret_cast<double*>(base + o_val) : nullptr;
  d.intensity = out->intensity ? reinterpret_cast<double*>(base + o_int) : nullptr;
  uint64_t* small = reinterpret_cast<uint64_t*>(base + o_small);
  d.image_hist = small;
  d.hit_count = small + 256;
  d.samples = small + 257;
  d.trunc_flag = reinterpret_cast<int32_t*>(small + 258);
  d.diag = out->diag ? small + 259 : nullptr;
  const bool timed = tl_frame_timing;
  cudaEvent_t* ev = nullptr;
  int rc = VX_OK;
  if (timed) {
    rc = timing_events(&ev);
    if (rc) return rc;
    VX_CUDA(cudaEventRecord(ev[0], s));
  }
  OrderJob order;
  rc = render_impl(vol, rs, rp, fc, part, &d, s, 0, &order);
  if (rc) return rc;
  if (timed) VX_CUDA(cudaEventRecord(ev[1], s));
  float ms = 0.0f;
  // one synchronisation: counters and every requested output come back
  // together; the rare truncation re-render (below) copies again.  The copies
  // are queued right behind K4; the next frame's tile ordering goes behind
  // them and the host waits only for the copies (event), not for it.
  uint64_t small_h[267];
  cudaEvent_t copied = nullptr;
  VX_CUDA(copy_event(&copied));
  auto copy_back = [&]() -> int {
    if (fused) {  // pixels, padding, histogram, hit count, samples, flag
      VX_CUDA(cudaMemcpyAsync(out->pixels, d.pixels, o_fused + 259 * 8, cudaMemcpyDeviceToHost, s));
    } else {
      VX_CUDA(cudaMemcpyAsync(out->pixels, d.pixels, npx, cudaMemcpyDeviceToHost, s));
      VX_CUDA(cudaMemcpyAsync(small_h, small, sizeof(small_h), cudaMemcpyDeviceToHost, s));
    }
    if (out->hit_voxel)
      VX_CUDA(cudaMemcpyAsync(out->hit_voxel, d.hit_voxel, npx * 12, cudaMemcpyDeviceToHost, s));
    if (out->hit_t) VX_CUDA(cudaMemcpyAsync(out->hit_t, d.hit_t, npx * 4, cudaMemcpyDeviceToHost, s));
    if (out->hit_value)
      VX_CUDA(cudaMemcpyAsync(out->hit_value, d.hit_value, npx * 8, cudaMemcpyDeviceToHost, s));
    if (out->intensity)
      VX_CUDA(cudaMemcpyAsync(out->intensity, d.intensity, npx * 8, cudaMemcpyDeviceToHost, s));
    VX_CUDA(cudaEventRecord(copied, s));
    int r2 = order_tiles(order, s);
    order = OrderJob();
    if (r2) return r2;
    VX_CUDA(cudaEventSynchronize(copied));
    if (fused) memcpy(small_h, out->image_hist, 259 * 8);
    return VX_OK;
  };
  double tc = trace_on() ? trace_us() : 0.0;
  rc = copy_back();
  if (rc) return rc;
  VX_TRACE("copy_back+sync", tc);
  if (timed) VX_CUDA(cudaEventElapsedTime(&ms, ev[0], ev[1]));
  int32_t flag;
  memcpy(&flag, &small_h[258], 4);
  if (flag && rp->max_steps <= 0) {
    // a ray exhausted its own span budget: re-render with the exact frame budget
    int budget = 0;
    rc = frame_budget(vol, rs, rp->step_size, s, &budget);
    if (rc) return rc;
    VX_CUDA(cudaMemsetAsync(small, 0, 267 * 8, s));
    if (timed) VX_CUDA(cudaEventRecord(ev[0], s));
    rc = render_impl(vol, rs, rp, fc, part, &d, s, budget, &order);
    if (rc) return rc;
    if (timed) VX_CUDA(cudaEventRecord(ev[1], s));
    rc = copy_back();
    if (rc) return rc;
    float ms2 = 0.0f;
    if (timed) VX_CUDA(cudaEventElapsedTime(&ms2, ev[0], ev[1]));
    ms += ms2;
  }
  tl_render_ms = timed ? ms : -1.0f;
  if (!fused) {
    if (out->image_hist) memcpy(out->image_hist, small_h, 256 * 8);
    if (out->hit_count) out->hit_count[0] = small_h[256];
    if (out->samples) out->samples[0] = small_h[257];
  }
  if (out->diag) memcpy(out->diag, small_h + 259, 8 * 8);
  if (out->trunc_flag) out->trunc_flag[0] = 0;
  return VX_OK;
}

extern "C" int vx_march_rays(vx_volume* vol, const double* origins, const double* dirs,
                             const double* t_enter, const double* t_exit, const int32_t* max_steps,
                             int64_t n, const vx_render_params* rp, const vx_filter_config* fc,
                             uint8_t* hit_out, int32_t* voxel_out, float* t_out,
                             double* value_out) {
  if (!vol || !rp || !fc || n < 0) {
    vx_set_error("vx_march_rays: bad argument");
    return VX_EINVAL;
  }
  if (n == 0) return VX_OK;
  cudaStream_t s = vx_stream();
  MarchD M;
  FiltD F;
  int rc = make_march(vol, rp, fc, M);
  if (rc) return rc;
  rc = make_filter(fc, F);
  if (rc) return rc;
  const uint8_t* dist = nullptr;
  SlotPin pin(vol, s);
  if (M.skip) {
    rc = vx_get_dist_map(vol, M.thr, &dist, &pin.m, s);
    if (rc) return rc;
    if (!dist) M.skip = 0;
  }
  VolView V = vx_view(vol, dist);
  // one device block: in (o,d,te,tx,ms,lut) out (hit,vox,t,val)
  const size_t b_o = n * 24, b_te = n * 8, b_ms = n * 4, b_lut = 256 * 8;
  const size_t b_h = n, b_v = n * 12, b_t = n * 4, b_val = n * 8;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += (bytes + 255) & ~size_t(255);
    return o;
  };
  const size_t oo = take(b_o), od = take(b_o), ote = take(b_te), otx = take(b_te), oms = take(b_ms),
               olut = take(b_lut), oh = take(b_h), ov = take(b_v), ot = take(b_t), oval = take(b_val);
  Scratch sc(s);
  VX_CUDA(vx_malloc_async(reinterpret_cast<uint8_t**>(&sc.p), off, s));
  uint8_t* b = sc.get<uint8_t>();
  VX_CUDA(cudaMemcpyAsync(b + oo, origins, b_o, cudaMemcpyHostToDevice, s));
  VX_CUDA(cudaMemcpyAsync(b + od, dirs, b_o, cudaMemcpyHostToDevice, s));
  VX_CUDA(cudaMemcpyAsync(b + ote, t_enter, b_te, cudaMemcpyHostToDevice, s));
  VX_CUDA(cudaMemcpyAsync(b + otx, t_exit, b_te, cudaMemcpyHostToDevice, s));
  VX_CUDA(cudaMemcpyAsync(b + oms, max_steps, b_ms, cudaMemcpyHostToDevice, s));
  VX_CUDA(cudaMemcpyAsync(b + olut, fc->entropy_lut, b_lut, cudaMemcpyHostToDevice, s));
  const bool checked = filter_reach(F) > VX_PAD - 1;
  auto* pd = reinterpret_cast<const double*>(b + od);
  auto* po = reinterpret_cast<const double*>(b + oo);
  if (checked)
    dispatch_march<true>(V, M, F, reinterpret_cast<const double*>(b + olut), po, pd,
                         reinterpret_cast<const double*>(b + ote), reinterpret_cast<const double*>(b + otx),
                         reinterpret_cast<const int32_t*>(b + oms), n, b + oh,
                         reinterpret_cast<int32_t*>(b + ov), reinterpret_cast<float*>(b + ot),
                         reinterpret_cast<double*>(b + oval), s);
  else
    dispatch_march<false>(V, M, F, reinterpret_cast<const double*>(b + olut), po, pd,
                          reinterpret_cast<const double*>(b + ote), reinterpret_cast<const double*>(b + otx),
                          reinterpret_cast<const int32_t*>(b + oms), n, b + oh,
                          reinterpret_cast<int32_t*>(b + ov), reinterpret_cast<float*>(b + ot),
                          reinterpret_cast<double*>(b + oval), s);
  VX_CHECK_LAUNCH();
  VX_CUDA(cudaMemcpyAsync(hit_out, b + oh, b_h, cudaMemcpyDeviceToHost, s));
  VX_CUDA(cudaMemcpyAsync(voxel_out, b + ov, b_v, cudaMemcpyDeviceToHost, s));
  VX_CUDA(cudaMemcpyAsync(t_out, b + ot, b_t, cudaMemcpyDeviceToHost, s));
  VX_CUDA(cudaMemcpyAsync(value_out, b + oval, b_val, cudaMemcpyDeviceToHost, s));
  VX_CUDA(cudaStreamSynchronize(s));
  return VX_OK;
}

extern "C" int vx_ray_dirs(const vx_ray_setup* rs, double* dirs_out) {
  if (!rs || !dirs_out || rs->width < 1 || rs->height < 1) {
    vx_set_error("vx_ray_dirs: bad argument");
    return VX_EINVAL;
  }
  cudaStream_t s = vx_stream();
  const int64_t n = (int64_t)rs->width * rs->height;
  Scratch sc(s);
  VX_CUDA(vx_malloc_async(reinterpret_cast<double**>(&sc.p), n * 24, s));
  ray_dirs_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(make_cam(rs), sc.get<double>());
  VX_CHECK_LAUNCH();
  VX_CUDA(cudaMemcpyAsync(dirs_out, sc.p, n * 24, cudaMemcpyDeviceToHost, s));
  VX_CUDA(cudaStreamSynchronize(s));
  return VX_OK;
}

extern "C" int vx_ray_spans(const double origin[3], const double* dirs, int64_t n,
                            const int64_t dims[3], double* t_enter_out, double* t_exit_out) {
  if (!origin || !dirs || !dims || n < 0) {
    vx_set_error("vx_ray_spans: bad argument");
    return VX_EINVAL;
  }
  if (n == 0) return VX_OK;
  cudaStream_t s = vx_stream();
  Scratch sc(s);
  VX_CUDA(vx_malloc_async(reinterpret_cast<double**>(&sc.p), n * 40, s));
  double* dd = sc.get<double>();
  double* te = dd + 3 * n;
  double* tx = te + n;
  VX_CUDA(cudaMemcpyAsync(dd, dirs, n * 24, cudaMemcpyHostToDevice, s));
  ray_spans_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(
      origin[0], origin[1], origin[2], dd, n, (int)dims[0], (int)dims[1], (int)dims[2], te, tx);
  VX_CHECK_LAUNCH();
  VX_CUDA(cudaMemcpyAsync(t_enter_out, te, n * 8, cudaMemcpyDeviceToHost, s));
  VX_CUDA(cudaMemcpyAsync(t_exit_out, tx, n * 8, cudaMemcpyDeviceToHost, s));
  VX_CUDA(cudaStreamSynchronize(s));
  return VX_OK;
}

extern "C" int vx_filter_batch(vx_volume* vol, const int64_t* xs, const int64_t* ys,
                               const int64_t* zs, int64_t n, const vx_filter_config* fc,
                               double* out) {
  if (!vol || !fc || n < 0) {
    vx_set_error("vx_filter_batch: bad argument");
    return VX_EINVAL;
  }
  if (n == 0) return VX_OK;
  FiltD F;
  int rc = make_filter(fc, F, true);
  if (rc) return rc;
  cudaStream_t s = vx_stream();
  Scratch sc(s);
  const size_t bytes = n * 8 * 4 + 256 * 8;
  VX_CUDA(vx_malloc_async(reinterpret_cast<uint8_t**>(&sc.p), bytes, s));
  int64_t* dx = sc.get<int64_t>();
  int64_t* dy = dx + n;
  int64_t* dz = dy + n;
  double* dout = reinterpret_cast<double*>(dz + n);
  double* dlut = dout + n;
  VX_CUDA(cudaMemcpyAsync(dx, xs, n * 8, cudaMemcpyHostToDevice, s));
  VX_CUDA(cudaMemcpyAsync(dy, ys, n * 8, cudaMemcpyHostToDevice, s));
  VX_CUDA(cudaMemcpyAsync(dz, zs, n * 8, cudaMemcpyHostToDevice, s));
  VX_CUDA(cudaMemcpyAsync(dlut, fc->entropy_lut, 256 * 8, cudaMemcpyHostToDevice, s));
  VolView V = vx_view(vol, nullptr);
  const unsigned g = (unsigned)((n + 127) / 128);
#define VX_FB(K) filter_batch_kernel<K><<<g, 128, 0, s>>>(V, F, dlut, dx, dy, dz, n, dout)
  switch (F.kind) {
    case VX_FILTER_NONE: VX_FB(VX_FILTER_NONE); break;
    case VX_FILTER_MEAN: VX_FB(VX_FILTER_MEAN); break;
    case VX_FILTER_SIGMA: VX_FB(VX_FILTER_SIGMA); break;
    case VX_FILTER_OKADA: VX_FB(VX_FILTER_OKADA); break;
    case VX_FILTER_ENTROPY: VX_FB(VX_FILTER_ENTROPY); break;
    case kAxisCluster: VX_FB(kAxisCluster); break;
    default: VX_FB(VX_FILTER_LOCAL_CLUSTER); break;
  }
#undef VX_FB
  VX_CHECK_LAUNCH();
  VX_CUDA(cudaMemcpyAsync(out, dout, n * 8, cudaMemcpyDeviceToHost, s));
  VX_CUDA(cudaStreamSynchronize(s));
  return VX_OK;
}

extern "C" int vx_sobel_batch(vx_volume* vol, const int64_t* xs, const int64_t* ys,
                              const int64_t* zs, int64_t n, const double* fallback,
                              double* normals_out) {
  if (!vol || n < 0) {
    vx_set_error("vx_sobel_batch: bad argument");
    return VX_EINVAL;
  }
  if (n == 0) return VX_OK;
  cudaStream_t s = vx_stream();
  Scratch sc(s);
  VX_CUDA(vx_malloc_async(reinterpret_cast<uint8_t**>(&sc.p), n * 8 * 9, s));
  int64_t* dx = sc.get<int64_t>();
  int64_t* dy = dx + n;
  int64_t* dz = dy + n;
  double* dfb = reinterpret_cast<double*>(dz + n);
  double* dout = dfb + 3 * n;
  VX_CUDA(cudaMemcpyAsync(dx, xs, n * 8, cudaMemcpyHostToDevice, s));
  VX_CUDA(cudaMemcpyAsync(dy, ys, n * 8, cudaMemcpyHostToDevice, s));
  VX_CUDA(cudaMemcpyAsync(dz, zs, n * 8, cudaMemcpyHostToDevice, s));
  VX_CUDA(cudaMemcpyAsync(dfb, fallback, n * 24, cudaMemcpyHostToDevice, s));
  sobel_batch_kernel<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(vx_view(vol, nullptr), dx, dy,
                                                                  dz, n, dfb, dout);
  VX_CHECK_LAUNCH();
  VX_CUDA(cudaMemcpyAsync(normals_out, dout, n * 24, cudaMemcpyDeviceToHost, s));
  VX_CUDA(cudaStreamSynchronize(s));
  return VX_OK;
}

extern "C" int vx_phong_batch(const double* normals, const double* view_dirs, int64_t n,
                              const vx_render_params* rp, uint8_t* out) {
  if (!rp || n < 0) {
    vx_set_error("vx_phong_batch: bad argument");
    return VX_EINVAL;
  }
  if (n == 0) return VX_OK;
  cudaStream_t s = vx_stream();
  Scratch sc(s);
  VX_CUDA(vx_malloc_async(reinterpret_cast<uint8_t**>(&sc.p), n * 49, s));
  double* dn = sc.get<double>();
  double* dv = dn + 3 * n;
  uint8_t* dout = reinterpret_cast<uint8_t*>(dv + 3 * n);
  VX_CUDA(cudaMemcpyAsync(dn, normals, n * 24, cudaMemcpyHostToDevice, s));
  VX_CUDA(cudaMemcpyAsync(dv, view_dirs, n * 24, cudaMemcpyHostToDevice, s));
  phong_batch_kernel<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(dn, dv, n, make_shade(rp), dout);
  VX_CHECK_LAUNCH();
  VX_CUDA(cudaMemcpyAsync(out, dout, n, cudaMemcpyDeviceToHost, s));
  VX_CUDA(cudaStreamSynchronize(s));
  return VX_OK;
}

#ifdef VX_WARP_TIMING
extern "C" int vx_debug_warp_times(unsigned long long* t0, unsigned long long* t1, unsigned* sm,
                                   int n) {
  if (n > (1 << 20)) n = 1 << 20;
  VX_CUDA(cudaDeviceSynchronize());
  VX_CUDA(cudaMemcpyFromSymbol(t0, g_warp_t0, (size_t)n * 8));
  VX_CUDA(cudaMemcpyFromSymbol(t1, g_warp_t1, (size_t)n * 8));
  VX_CUDA(cudaMemcpyFromSymbol(sm, g_warp_sm, (size_t)n * 4));
  return VX_OK;
}
extern "C" int vx_debug_warp_diag(unsigned* out, int n) {
  if (n > (1 << 20)) n = 1 << 20;
  VX_CUDA(cudaDeviceSynchronize());
  VX_CUDA(cudaMemcpyFromSymbol(out, g_warp_diag, (size_t)n * 9 * 4));
  return VX_OK;
}
#endif
