// Internal declarations shared by the libvoxb200 translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>
#include <string>
#include <vector>

#include "../../include/voxb200.h"

// Voxel layout of the replica K4 reads (A/B): 0 = linear
// (x fastest, 16-voxel zero apron), 1 = 8^3 bricks of 512 B (linear inside:
// a 32 B sector is 8x4x1 voxels), 2 = 8^3 bricks, Morton order inside (a
// sector is 4x4x2 voxels).  Bricked builds keep the linear replica for the
// other kernels and add a bricked copy for K4.
#ifndef VX_BRICK_LAYOUT
#define VX_BRICK_LAYOUT 0
#endif

// Zero apron around the volume (voxels).  Covers the march's +/-1 voxel
// truncation slop, Sobel (reach 1) and every filter with reach <= VX_PAD-1;
// larger reach switches the filter to bounds-checked reads (same border
// policy as grid.py:34-44: reads outside the grid are 0).
#define VX_PAD 16
// Empty-space-skipping brick edge (voxels).
#define VX_BRICK 8
#define VX_BRICK_SHIFT 3
// Chebyshev brick-distance cap of the coarse exact-skip map (8^3 bricks).
#define VX_DIST_CAP 24
// Fine exact-skip map: 4^3 cells, Chebyshev cell distance capped at a
// per-volume cap (17 MB at 1024^3, L2-resident).  Long skips step over whole
// chunks by the exact base recurrence (one FP32 add per 16 samples), so the
// best cap grows with the volume: 32 cells up to 512^3, 64 at 1024^3, 128
// from 2048^3 (profiles/r2/r2_ab_skip_cap.txt); VX_FINE_CAP > 0 forces one.
#define VX_CELL 4
#define VX_CELL_SHIFT 2
#ifndef VX_FINE_CAP
#define VX_FINE_CAP 0
#endif
static inline int vx_fine_cap_for(int64_t nx, int64_t ny, int64_t nz) {
  if (VX_FINE_CAP > 0) return VX_FINE_CAP;
  int64_t m = nx > ny ? nx : ny;
  m = m > nz ? m : nz;
  const int64_t c = m / 16;
  return (int)(c < 32 ? 32 : (c > 128 ? 128 : c));
}
#define VX_DIST_CACHE 4

// offset of voxel (x, y, z) & 7 inside its 8^3 brick
__host__ __device__ __forceinline__ int vx_in_brick(int x, int y, int z) {
#if VX_BRICK_LAYOUT == 2
  auto spread = [](int v) { return (v & 1) | ((v & 2) << 2) | ((v & 4) << 4); };
  return spread(x) | (spread(y) << 1) | (spread(z) << 2);
#else
  return (z << 6) | (y << 3) | x;
#endif
}

// ---------------------------------------------------------------------------
// error plumbing
void vx_set_error(const char* fmt, ...);
int vx_cuda_fail(cudaError_t e, const char* what, const char* file, int line);
#define VX_CUDA(call)                                                     \
  do {                                                                    \
    cudaError_t _e = (call);                                              \
    if (_e != cudaSuccess) return vx_cuda_fail(_e, #call, __FILE__, __LINE__); \
  } while (0)
#define VX_CHECK_LAUNCH()                                                 \
  do {                                                                    \
    cudaError_t _e = cudaGetLastError();                                  \
    if (_e != cudaSuccess) return vx_cuda_fail(_e, "kernel launch", __FILE__, __LINE__); \
    vx_count_launch();                                                    \
  } while (0)

cudaStream_t vx_stream();          // per-thread stream
void vx_count_launch();
int vx_sm_count();

// ---------------------------------------------------------------------------
// device view of a volume replica
struct VolView {
  const uint8_t* origin;  // voxel (0,0,0) inside the padded allocation
  int64_t sy, sz;         // byte strides of rows / planes
  int nx, ny, nz;
  const uint8_t* dist;    // Chebyshev brick-distance map at brick (0,0,0)
  int64_t bsy, bsz;       // strides of the brick maps
  const uint8_t* dist2;   // Chebyshev cell-distance map at cell (0,0,0)
  int64_t csy, csz;       // strides of the cell maps
#if VX_BRICK_LAYOUT
  const uint8_t* bricks;  // bricked copy: brick (bx, by, bz) of the apron-padded grid
  int bbx, bby;           // bricks per row / per plane row (apron included)
#endif
  // orthant maps (nullable): map of orthant o at doct + o * oct_stride (cell
  // (0,0,0)); bit o of oct_mask set when that orthant's map is built
  const uint8_t* doct;
  int64_t oct_stride;
  int oct_mask;
#ifdef VX_DEBUG_CHECKS
  // bounds of the padded allocation and of the cell maps (checked build only)
  const uint8_t *lo, *hi, *d2lo, *d2hi, *dolo, *dohi;
#endif
};

// Checked build (-DVX_DEBUG_CHECKS, libvoxb200_checked.so): every voxel read
// must stay inside the zero apron (|overshoot| <= VX_PAD) and the allocation,
// every map read inside its map, every shared-scratch index inside its
// array; a violation prints the kernel's coordinates and traps (the stand-in
// for compute-sanitizer memcheck, which is closed on this pool).
#ifdef VX_DEBUG_CHECKS
#define VX_DCHECK(cond, fmt, ...)                                                      \
  do {                                                                                 \
    if (!(cond)) {                                                                     \
      printf("VX_DCHECK %s:%d block %d thread %d: " fmt "\n", __FILE__, __LINE__,       \
             (int)blockIdx.x, (int)(threadIdx.y * blockDim.x + threadIdx.x), __VA_ARGS__); \
      __trap();                                                                        \
    }                                                                                  \
  } while (0)
#else
#define VX_DCHECK(cond, fmt, ...) \
  do {                            \
  } while (0)
#endif

// Lifetime of a cached map slot (distance or accepted-cell map).  A render
// pins the slot from its lookup until its K4 is enqueued, then records the
// slot's per-stream use event behind that K4 and unpins it.  Eviction takes
// only unpinned slots and orders the rebuild (on the evicting thread's
// stream) after every recorded use; a freshly built map is published with a
// `ready` event that other streams wait on.  No host synchronisation happens
// under the volume mutex.
struct MapUse {
  cudaStream_t stream;
  cudaEvent_t ev;
};
struct MapSlot {
  uint8_t* map = nullptr;  // slot in vx_volume::bmax: brick map (map_bytes) then cell map (cmap_bytes)
  uint64_t stamp = 0;
  int pins = 0;
  cudaEvent_t ready = nullptr;
  std::vector<MapUse> uses;
  // Orthant maps: per ray-direction orthant, the distance to
  // the nearest occupied cell a ray of that orthant can still reach; built
  // on demand from the slot's occupancy (occ_src >= occ_thr) for the
  // orthants a frame's rays use.  oct: 8 * cmap_bytes, allocated on first use.
  const uint8_t* occ_src = nullptr;
  int occ_thr = 0;
  uint8_t* occ = nullptr;  // accepted-cell occupancy kept for orthant builds (cmap_bytes)
  uint8_t* oct = nullptr;
  unsigned oct_built = 0;
  cudaEvent_t oct_ready[8] = {};
};

struct DistEntry : MapSlot {
  int thr = -1;  // -1: empty
};

// Accepted-cell distance maps: the skip structure of one filter setting.
// Key = the filter parameters that decide `f >= T` at a voxel (opaque bytes,
// compared exactly).  valid && !built: the key was seen once (not built yet).
#define VX_ACC_CACHE 4
#define VX_ACC_KEY_BYTES 2096
struct AccEntry : MapSlot {
  bool valid = false;
  bool built = false;
  unsigned char key[VX_ACC_KEY_BYTES];
};

struct vx_volume {
  int nx, ny, nz;
  int device;
  uint8_t* alloc;   // padded allocation
  uint8_t* origin;  // voxel (0,0,0)
  int64_t px, py, pz;  // padded dims
  int64_t sy, sz;
  uint64_t alloc_bytes;
  // brick max map with a 1-brick apron: dims (nbx+2, nby+2, nbz+2); its
  // allocation also holds the cell max map and the slots of every cached
  // distance / accepted-cell map (one cudaMalloc at creation: a cudaMalloc
  // inside a frame measured 1-97 ms)
  uint8_t* bmax;
  int nbx, nby, nbz;
  int64_t bsy, bsz;
  uint64_t map_bytes;
  // cell (4^3) max map with a 1-cell apron: dims (ncx+2, ncy+2, ncz+2)
  uint8_t* cmax;
  int ncx, ncy, ncz;
  int fine_cap;  // distance cap of the cell maps (vx_fine_cap_for)
  int64_t csy, csz;
  uint64_t cmap_bytes;
  DistEntry dist[VX_DIST_CACHE];
  AccEntry acc[VX_ACC_CACHE];
  // two cell-map-sized scratch regions for the map builds (occupancy and the
  // distance passes' intermediate), claimed under `mu`; builds on different
  // streams are ordered through scratch_done
  uint8_t* scratch;
  cudaEvent_t scratch_done;
  uint8_t* bricks;  // VX_BRICK_LAYOUT: the bricked copy K4 reads
  int bbx, bby, bbz;
  uint64_t bricks_bytes;
  uint64_t stamp;
  uint64_t counts[256];
  std::mutex mu;
};

VolView vx_view(const vx_volume* v, const uint8_t* dist_map);
// The (cached) distance map of thr, built if needed (stream-ordered on s),
// pinned: pass *slot_out to vx_map_release once the work reading it is
// enqueued on s.  *map_out == nullptr (no skipping) when every slot is pinned.
int vx_get_dist_map(vx_volume* v, int thr, const uint8_t** map_out, MapSlot** slot_out,
                    cudaStream_t s);
// caller holds v->mu: the slot is being reused for a new map; order stream s
// after every recorded reader and after earlier builds' use of the scratch
int vx_map_claim(vx_volume* v, MapSlot* m, cudaStream_t s);
// caller holds v->mu: the slot's map (built on s) is complete on s
int vx_map_publish(vx_volume* v, MapSlot* m, cudaStream_t s);
// caller holds v->mu: stream s will read the slot's map (waits for its build)
int vx_map_pin(MapSlot* m, cudaStream_t s);
// unpin after the readers on s are enqueued (nullptr: no-op)
int vx_map_release(vx_volume* v, MapSlot* m, cudaStream_t s);
// caller holds v->mu and a pin of m: the orthant maps in `need` (bitmask) are
// built (stream-ordered on s) or awaited; returns the built mask
int vx_map_octants(vx_volume* v, MapSlot* m, unsigned need, unsigned* built_out, cudaStream_t s);
int vx_launch_dist_cells_oct(const vx_volume* v, const uint8_t* occ, uint8_t* out, int thr, int oct,
                             cudaStream_t s);

// launchers implemented across translation units
int vx_launch_hist(const uint8_t* dev, uint64_t n, uint64_t* dev_counts, cudaStream_t s);
int vx_launch_otsu(const uint64_t* dev_counts, int32_t* dev_T, cudaStream_t s);
// K1+K2 fused: dev_counts[256] overwritten, dev_T = Otsu T (-1: empty / >= 2^47)
int vx_launch_hist_otsu(const uint8_t* dev, uint64_t n, uint64_t* dev_counts, int32_t* dev_T,
                        cudaStream_t s);
int vx_launch_sub_bin0(uint64_t* dev_counts, uint64_t v, cudaStream_t s);
int vx_launch_entropy(const uint64_t* dev_counts, uint64_t n, double* dev_H, cudaStream_t s);
int vx_launch_brick_max(vx_volume* v, cudaStream_t s);
int vx_launch_dist_map(const vx_volume* v, int thr, uint8_t* map, cudaStream_t s);
// (callers hold v->mu: the builds use v->scratch)
int vx_launch_cell_max(vx_volume* v, cudaStream_t s);
// VX_BRICK_LAYOUT: the bricked copy of the (finished) linear replica
int vx_launch_brickify(vx_volume* v, cudaStream_t s);
// Chebyshev cell-distance map (cap VX_FINE_CAP) of the cells whose value in
// `occ` (cell-map layout, apron included) is >= thr
int vx_launch_dist_cells(const vx_volume* v, const uint8_t* occ, uint8_t* out, int thr,
                         cudaStream_t s);
int vx_launch_u16_to_u8(const uint16_t* src, uint8_t* dst, uint64_t n, cudaStream_t s);
int vx_launch_phantom(uint8_t* dst, int64_t row_pitch, int64_t plane_pitch, int64_t nx,
                      int64_t ny, int64_t nz, const double* shapes, int64_t n_shapes,
                      double noise_sigma, uint64_t noise_seed, const int64_t* spot_idx,
                      int64_t n_spots, int32_t spot_intensity, cudaStream_t s);
int vx_preload_render_kernels();
// K4 into device outputs that may live in another rank's memory (peer /
// IPC-mapped): sys_atomics selects system-scope counter atomics
int vx_render_tiles(vx_volume* vol, const vx_ray_setup* rs, const vx_render_params* rp,
                    const vx_filter_config* fc, const vx_partition* part, vx_render_out* dev_out,
                    cudaStream_t s, bool sys_atomics);
int vx_volume_alloc(int64_t nx, int64_t ny, int64_t nz, vx_volume** out);
int vx_volume_finish(vx_volume* v, const uint8_t* compact_dev, cudaStream_t s);

// RAII-free device scratch helpers (stream-ordered allocator)
template <typename T>
static inline cudaError_t vx_malloc_async(T** p, size_t bytes, cudaStream_t s) {
  return cudaMallocAsync(reinterpret_cast<void**>(p), bytes ? bytes : 16, s);
}
