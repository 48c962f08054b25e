// C-ABI plumbing: errors, per-thread streams, volume lifecycle, statistics
// entry points.  See include/voxb200.h for the contract of each function.

#include <algorithm>
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <new>

#include "vx_internal.cuh"

#define VX_VERSION 1

// ---------------------------------------------------------------------------
// errors / context

static thread_local char tl_error[512] = "";
// one stream per (thread, device), kept for the thread's life: switching
// devices and back keeps work on a device ordered on one stream
static thread_local cudaStream_t tl_stream[64] = {};
static thread_local uint64_t tl_launches = 0;

void vx_set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(tl_error, sizeof(tl_error), fmt, ap);
  va_end(ap);
}

int vx_cuda_fail(cudaError_t e, const char* what, const char* file, int line) {
  vx_set_error("CUDA error %s (%s) in %s at %s:%d", cudaGetErrorName(e), cudaGetErrorString(e),
               what, file, line);
  return e == cudaErrorMemoryAllocation ? VX_ENOMEM : VX_ECUDA;
}

void vx_count_launch() { ++tl_launches; }

cudaStream_t vx_stream() {
  int dev = 0;
  cudaGetDevice(&dev);
  cudaStream_t& st = tl_stream[dev & 63];
  if (!st) {
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    // keep freed stream-ordered scratch cached in the pool
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  }
  return st;
}

int vx_sm_count() {
  static std::atomic<int> cached[64];
  int dev = 0;
  cudaGetDevice(&dev);
  int v = cached[dev & 63].load();
  if (!v) {
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    if (v <= 0) v = 148;
    cached[dev & 63].store(v);
  }
  return v;
}

extern "C" const char* vx_last_error(void) { return tl_error; }
extern "C" int vx_version(void) { return VX_VERSION; }

extern "C" int vx_device_count(int* n_out) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) {
    cudaGetLastError();
    *n_out = 0;
    return vx_cuda_fail(e, "cudaGetDeviceCount", __FILE__, __LINE__);
  }
  *n_out = n;
  return VX_OK;
}

extern "C" int vx_set_device(int device) {
  VX_CUDA(cudaSetDevice(device));
  return VX_OK;
}

extern "C" int vx_synchronize(void) {
  VX_CUDA(cudaStreamSynchronize(vx_stream()));
  return VX_OK;
}

extern "C" int vx_host_alloc(uint64_t bytes, void** out) {
  if (!out) {
    vx_set_error("vx_host_alloc: null argument");
    return VX_EINVAL;
  }
  VX_CUDA(cudaHostAlloc(out, bytes ? bytes : 1, cudaHostAllocDefault));
  return VX_OK;
}

extern "C" int vx_host_free(void* p) {
  if (p) VX_CUDA(cudaFreeHost(p));
  return VX_OK;
}

extern "C" int vx_launch_counter(uint64_t* n_out, int reset) {
  if (n_out) *n_out = tl_launches;
  if (reset) tl_launches = 0;
  return VX_OK;
}

// ---------------------------------------------------------------------------
// volume lifecycle

VolView vx_view(const vx_volume* v, const uint8_t* dist_map) {
  VolView V;
  V.origin = v->origin;
  V.sy = v->sy;
  V.sz = v->sz;
  V.nx = v->nx;
  V.ny = v->ny;
  V.nz = v->nz;
  V.bsy = v->bsy;
  V.bsz = v->bsz;
  V.dist = dist_map ? dist_map + v->bsz + v->bsy + 1 : nullptr;
  V.csy = v->csy;
  V.csz = v->csz;
  V.dist2 = dist_map ? dist_map + v->map_bytes + v->csz + v->csy + 1 : nullptr;
#if VX_BRICK_LAYOUT
  V.bricks = v->bricks;
  V.bbx = v->bbx;
  V.bby = v->bby;
#endif
  V.doct = nullptr;
  V.oct_stride = 0;
  V.oct_mask = 0;
#ifdef VX_DEBUG_CHECKS
  V.dolo = V.dohi = nullptr;
  V.lo = v->alloc;
  V.hi = v->alloc + v->alloc_bytes;
  V.d2lo = dist_map ? dist_map + v->map_bytes : nullptr;
  V.d2hi = dist_map ? dist_map + v->map_bytes + v->cmap_bytes : nullptr;
#endif
  return V;
}

static bool dims_ok(int64_t nx, int64_t ny, int64_t nz) {
  return nx >= 1 && ny >= 1 && nz >= 1 && nx < (1 << 20) && ny < (1 << 20) && nz < (1 << 20);
}

int vx_volume_alloc(int64_t nx, int64_t ny, int64_t nz, vx_volume** out) {
  if (!dims_ok(nx, ny, nz)) {
    vx_set_error("dims must each be >= 1, got (%lld, %lld, %lld)", (long long)nx, (long long)ny,
                 (long long)nz);
    return VX_EINVAL;
  }
  vx_volume* v = new (std::nothrow) vx_volume();
  if (!v) {
    vx_set_error("host allocation failed");
    return VX_ENOMEM;
  }
  cudaGetDevice(&v->device);
  v->nx = (int)nx;
  v->ny = (int)ny;
  v->nz = (int)nz;
  v->px = ((nx + 2 * VX_PAD) + 15) & ~int64_t(15);
  v->py = ny + 2 * VX_PAD;
  v->pz = nz + 2 * VX_PAD;
  v->sy = v->px;
  v->sz = v->px * v->py;
  v->alloc_bytes = (uint64_t)(v->sz * v->pz);
  v->nbx = (int)((nx + 7) / 8);
  v->nby = (int)((ny + 7) / 8);
  v->nbz = (int)((nz + 7) / 8);
  v->bsy = v->nbx + 2;
  v->bsz = (int64_t)(v->nbx + 2) * (v->nby + 2);
  v->map_bytes = (uint64_t)v->bsz * (v->nbz + 2);
  v->ncx = (int)((nx + VX_CELL - 1) / VX_CELL);
  v->ncy = (int)((ny + VX_CELL - 1) / VX_CELL);
  v->ncz = (int)((nz + VX_CELL - 1) / VX_CELL);
  v->csy = v->ncx + 2;
  v->csz = (int64_t)(v->ncx + 2) * (v->ncy + 2);
  v->cmap_bytes = (uint64_t)v->csz * (v->ncz + 2);
  v->fine_cap = vx_fine_cap_for(nx, ny, nz);
  cudaError_t e = cudaEventCreateWithFlags(&v->scratch_done, cudaEventDisableTiming);
  if (e != cudaSuccess) {
    delete v;
    return vx_cuda_fail(e, "cudaEventCreate", __FILE__, __LINE__);
  }
  e = cudaMalloc(&v->alloc, v->alloc_bytes);
  if (e != cudaSuccess) {
    cudaEventDestroy(v->scratch_done);
    delete v;
    return vx_cuda_fail(e, "cudaMalloc(volume)", __FILE__, __LINE__);
  }
  const uint64_t slot = v->map_bytes + v->cmap_bytes;
  e = cudaMalloc(&v->bmax, slot * (1 + VX_DIST_CACHE + VX_ACC_CACHE) + 2 * v->cmap_bytes);
  if (e != cudaSuccess) {
    cudaFree(v->alloc);
    cudaEventDestroy(v->scratch_done);
    delete v;
    return vx_cuda_fail(e, "cudaMalloc(brick map)", __FILE__, __LINE__);
  }
  v->cmax = v->bmax + v->map_bytes;
  for (int i = 0; i < VX_DIST_CACHE; ++i) v->dist[i].map = v->bmax + slot * (1 + i);
  for (int i = 0; i < VX_ACC_CACHE; ++i) v->acc[i].map = v->bmax + slot * (1 + VX_DIST_CACHE + i);
  v->scratch = v->bmax + slot * (1 + VX_DIST_CACHE + VX_ACC_CACHE);
  v->origin = v->alloc + VX_PAD * v->sz + VX_PAD * v->sy + VX_PAD;
  *out = v;
  return VX_OK;
}

// compact device bytes -> padded layout + histogram + brick map
int vx_volume_finish(vx_volume* v, const uint8_t* compact_dev, cudaStream_t s) {
  uint64_t* dcounts = nullptr;
  VX_CUDA(vx_malloc_async(&dcounts, 257 * 8, s));
  const uint64_t n = (uint64_t)v->nx * v->ny * v->nz;
  // K1 (+ the fused K2 scan, whose T is recomputed by otsu() on demand)
  int rc = vx_launch_hist_otsu(compact_dev, n, dcounts, reinterpret_cast<int32_t*>(dcounts + 256), s);
  if (rc) return rc;
  VX_CUDA(cudaMemsetAsync(v->alloc, 0, v->alloc_bytes, s));
  cudaMemcpy3DParms p;
  memset(&p, 0, sizeof(p));
  p.srcPtr = make_cudaPitchedPtr(const_cast<uint8_t*>(compact_dev), v->nx, v->nx, v->ny);
  p.dstPtr = make_cudaPitchedPtr(v->alloc, v->px, v->px, v->py);
  p.dstPos = make_cudaPos(VX_PAD, VX_PAD, VX_PAD);
  p.extent = make_cudaExtent(v->nx, v->ny, v->nz);
  p.kind = cudaMemcpyDeviceToDevice;
  VX_CUDA(cudaMemcpy3DAsync(&p, s));
  VX_CUDA(cudaMemsetAsync(v->bmax, 0, v->map_bytes + v->cmap_bytes, s));
#if VX_BRICK_LAYOUT
  v->bbx = (int)((v->nx + 2 * VX_PAD + 7) / 8);
  v->bby = (int)((v->ny + 2 * VX_PAD + 7) / 8);
  v->bbz = (int)((v->nz + 2 * VX_PAD + 7) / 8);
  v->bricks_bytes = (uint64_t)v->bbx * v->bby * v->bbz * 512;
  if (!v->bricks) VX_CUDA(cudaMalloc(&v->bricks, v->bricks_bytes));
  rc = vx_launch_brickify(v, s);
  if (rc) return rc;
#endif
  rc = vx_launch_brick_max(v, s);
  if (rc) return rc;
  rc = vx_launch_cell_max(v, s);
  if (rc) return rc;
  uint64_t th[257];
  VX_CUDA(cudaMemcpyAsync(th, dcounts, 257 * 8, cudaMemcpyDeviceToHost, s));
  VX_CUDA(cudaFreeAsync(dcounts, s));
  VX_CUDA(cudaStreamSynchronize(s));
  memcpy(v->counts, th, 256 * 8);
  // Ready the first frame: the default filter setting thresholds at the
  // Otsu level, so its candidate distance map (thr = T) is built now, and
  // the frame kernels are loaded (~1 ms of GPU work and the lazy module
  // loads, out of the first frame; VOXB200_PREPARE=0 skips both).
  static const bool prepare = [] {
    const char* e = getenv("VOXB200_PREPARE");
    return !e || atoi(e) != 0;
  }();
  if (prepare) {
    int32_t T;
    memcpy(&T, &th[256], 4);
    const uint8_t* m = nullptr;
    MapSlot* slot = nullptr;
    if (T > 0 && T <= 255) {
      if ((rc = vx_get_dist_map(v, T, &m, &slot, s))) return rc;
      // and its eight orthant maps (~0.2 ms each at 1024^3): whatever the
      // first camera, its frame finds its orthants built
      unsigned built = 0;
      {
        std::lock_guard<std::mutex> lock(v->mu);
        rc = vx_map_octants(v, slot, 0xffu, &built, s);
      }
      if (rc) return rc;
      if ((rc = vx_map_release(v, slot, s))) return rc;
      // the first accepted-cell slot's occupancy and orthant blocks: a
      // cudaMalloc inside a frame measured 1-97 ms
      AccEntry& a0 = v->acc[0];
      if (!a0.occ) VX_CUDA(cudaMalloc(&a0.occ, v->cmap_bytes));
      if (!a0.oct) VX_CUDA(cudaMalloc(&a0.oct, 8 * v->cmap_bytes));
    }
    if ((rc = vx_preload_render_kernels())) return rc;
    // grow the stream-ordered pool once (it keeps freed memory: release
    // threshold above), so a first frame's staging comes from retained memory
    uint8_t* warm = nullptr;
    VX_CUDA(vx_malloc_async(&warm, 64ull << 20, s));
    VX_CUDA(cudaFreeAsync(warm, s));
  }
  return VX_OK;
}

static int create_from_device(const uint8_t* dev, int64_t nx, int64_t ny, int64_t nz,
                              vx_volume** out, cudaStream_t s) {
  vx_volume* v = nullptr;
  int rc = vx_volume_alloc(nx, ny, nz, &v);
  if (rc) return rc;
  rc = vx_volume_finish(v, dev, s);
  if (rc) {
    vx_volume_destroy(v);
    return rc;
  }
  *out = v;
  return VX_OK;
}

extern "C" int vx_volume_create_device_u8(const uint8_t* dev, int64_t nx, int64_t ny, int64_t nz,
                                          vx_volume** out) {
  if (!dev || !out) {
    vx_set_error("vx_volume_create_device_u8: null argument");
    return VX_EINVAL;
  }
  cudaStream_t s = vx_stream();
  VX_CUDA(cudaDeviceSynchronize());  // producer may be on another stream
  return create_from_device(dev, nx, ny, nz, out, s);
}

extern "C" int vx_volume_create_u8(const uint8_t* host, int64_t nx, int64_t ny, int64_t nz,
                                   vx_volume** out) {
  if (!host || !out) {
    vx_set_error("vx_volume_create_u8: null argument");
    return VX_EINVAL;
  }
  if (!dims_ok(nx, ny, nz)) {
    vx_set_error("dims must each be >= 1, got (%lld, %lld, %lld)", (long long)nx, (long long)ny,
                 (long long)nz);
    return VX_EINVAL;
  }
  cudaStream_t s = vx_stream();
  const uint64_t n = (uint64_t)nx * ny * nz;
  uint8_t* staging = nullptr;
  VX_CUDA(cudaMalloc(&staging, n));
  cudaError_t e = cudaMemcpyAsync(staging, host, n, cudaMemcpyHostToDevice, s);
  int rc = VX_OK;
  if (e != cudaSuccess)
    rc = vx_cuda_fail(e, "upload", __FILE__, __LINE__);
  else
    rc = create_from_device(staging, nx, ny, nz, out, s);
  cudaStreamSynchronize(s);
  cudaFree(staging);
  return rc;
}

extern "C" int vx_volume_create_u16(const uint16_t* host, int64_t nx, int64_t ny, int64_t nz,
                                    vx_volume** out) {
  if (!host || !out) {
    vx_set_error("vx_volume_create_u16: null argument");
    return VX_EINVAL;
  }
  if (!dims_ok(nx, ny, nz)) {
    vx_set_error("dims must each be >= 1, got (%lld, %lld, %lld)", (long long)nx, (long long)ny,
                 (long long)nz);
    return VX_EINVAL;
  }
  cudaStream_t s = vx_stream();
  const uint64_t n = (uint64_t)nx * ny * nz;
  uint8_t* staging = nullptr;
  VX_CUDA(cudaMalloc(&staging, n * 3));  // u16 words then u8 bytes
  uint16_t* wide = reinterpret_cast<uint16_t*>(staging);
  uint8_t* narrow = staging + 2 * n;
  int rc = VX_OK;
  cudaError_t e = cudaMemcpyAsync(wide, host, 2 * n, cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) rc = vx_cuda_fail(e, "upload", __FILE__, __LINE__);
  if (!rc) rc = vx_launch_u16_to_u8(wide, narrow, n, s);
  if (!rc) rc = create_from_device(narrow, nx, ny, nz, out, s);
  cudaStreamSynchronize(s);
  cudaFree(staging);
  return rc;
}

extern "C" int vx_volume_create_phantom(int64_t nx, int64_t ny, int64_t nz, const double* shapes,
                                        int64_t n_shapes, double noise_sigma, uint64_t noise_seed,
                                        const int64_t* spot_idx, int64_t n_spots,
                                        int32_t spot_intensity, vx_volume** out) {
  if (!out || (n_shapes && !shapes) || (n_spots && !spot_idx)) {
    vx_set_error("vx_volume_create_phantom: null argument");
    return VX_EINVAL;
  }
  if (!dims_ok(nx, ny, nz)) {
    vx_set_error("dims must each be >= 1, got (%lld, %lld, %lld)", (long long)nx, (long long)ny,
                 (long long)nz);
    return VX_EINVAL;
  }
  cudaStream_t s = vx_stream();
  const uint64_t n = (uint64_t)nx * ny * nz;
  uint8_t* staging = nullptr;
  VX_CUDA(cudaMalloc(&staging, n));
  int rc = VX_OK;
  cudaError_t e = cudaMemsetAsync(staging, 0, n, s);
  if (e != cudaSuccess) rc = vx_cuda_fail(e, "memset", __FILE__, __LINE__);
  if (!rc)
    rc = vx_launch_phantom(staging, nx, nx * ny, nx, ny, nz, shapes, n_shapes, noise_sigma,
                           noise_seed, spot_idx, n_spots, spot_intensity, s);
  if (!rc) rc = create_from_device(staging, nx, ny, nz, out, s);
  cudaStreamSynchronize(s);
  cudaFree(staging);
  return rc;
}

extern "C" int vx_phantom_device(uint8_t* dev_out, int64_t nx, int64_t ny, int64_t nz,
                                 const double* shapes, int64_t n_shapes, double noise_sigma,
                                 uint64_t noise_seed, const int64_t* spot_idx, int64_t n_spots,
                                 int32_t spot_intensity, void* stream) {
  if (!dev_out || !dims_ok(nx, ny, nz)) {
    vx_set_error("vx_phantom_device: bad argument");
    return VX_EINVAL;
  }
  cudaStream_t s = (cudaStream_t)stream;
  VX_CUDA(cudaMemsetAsync(dev_out, 0, (size_t)(nx * ny * nz), s));
  return vx_launch_phantom(dev_out, nx, nx * ny, nx, ny, nz, shapes, n_shapes, noise_sigma,
                           noise_seed, spot_idx, n_spots, spot_intensity, s);
}

extern "C" int vx_volume_destroy(vx_volume* v) {
  if (!v) return VX_OK;
  int cur = 0;
  cudaGetDevice(&cur);
  if (cur != v->device) cudaSetDevice(v->device);
  cudaDeviceSynchronize();
  auto drop = [](MapSlot& m) {
    if (m.ready) cudaEventDestroy(m.ready);
    for (auto& u : m.uses) cudaEventDestroy(u.ev);
    for (auto& e : m.oct_ready)
      if (e) cudaEventDestroy(e);
    if (m.oct) cudaFree(m.oct);
    if (m.occ) cudaFree(m.occ);
  };
  for (auto& d : v->dist) drop(d);
  for (auto& a : v->acc) drop(a);
  if (v->scratch_done) cudaEventDestroy(v->scratch_done);
  if (v->bmax) cudaFree(v->bmax);
  if (v->alloc) cudaFree(v->alloc);
  if (v->bricks) cudaFree(v->bricks);
  if (cur != v->device) cudaSetDevice(cur);
  delete v;
  return VX_OK;
}

extern "C" int vx_volume_skip_cap(const vx_volume* v, int32_t level, int32_t* cap_out) {
  if (!v || !cap_out) {
    vx_set_error("vx_volume_skip_cap: null argument");
    return VX_EINVAL;
  }
  *cap_out = level == 0 ? VX_DIST_CAP : v->fine_cap;
  return VX_OK;
}

extern "C" int vx_volume_dims(const vx_volume* v, int64_t dims_out[3]) {
  if (!v || !dims_out) {
    vx_set_error("vx_volume_dims: null argument");
    return VX_EINVAL;
  }
  dims_out[0] = v->nx;
  dims_out[1] = v->ny;
  dims_out[2] = v->nz;
  return VX_OK;
}

extern "C" int vx_volume_device_bytes(const vx_volume* v, uint64_t* bytes_out) {
  if (!v || !bytes_out) {
    vx_set_error("vx_volume_device_bytes: null argument");
    return VX_EINVAL;
  }
  *bytes_out = v->alloc_bytes + v->map_bytes + v->cmap_bytes;
  return VX_OK;
}

extern "C" int vx_volume_read(const vx_volume* v, uint8_t* host_out) {
  if (!v || !host_out) {
    vx_set_error("vx_volume_read: null argument");
    return VX_EINVAL;
  }
  cudaStream_t s = vx_stream();
  cudaMemcpy3DParms p;
  memset(&p, 0, sizeof(p));
  p.srcPtr = make_cudaPitchedPtr(v->alloc, v->px, v->px, v->py);
  p.srcPos = make_cudaPos(VX_PAD, VX_PAD, VX_PAD);
  p.dstPtr = make_cudaPitchedPtr(host_out, v->nx, v->nx, v->ny);
  p.extent = make_cudaExtent(v->nx, v->ny, v->nz);
  p.kind = cudaMemcpyDeviceToHost;
  VX_CUDA(cudaMemcpy3DAsync(&p, s));
  VX_CUDA(cudaStreamSynchronize(s));
  return VX_OK;
}

int vx_map_claim(vx_volume* v, MapSlot* m, cudaStream_t s) {
  for (auto& u : m->uses) VX_CUDA(cudaStreamWaitEvent(s, u.ev, 0));
  m->oct_built = 0;  // the orthant maps belong to the old map
  VX_CUDA(cudaStreamWaitEvent(s, v->scratch_done, 0));
  return VX_OK;
}

int vx_map_publish(vx_volume* v, MapSlot* m, cudaStream_t s) {
  if (!m->ready) VX_CUDA(cudaEventCreateWithFlags(&m->ready, cudaEventDisableTiming));
  VX_CUDA(cudaEventRecord(m->ready, s));
  VX_CUDA(cudaEventRecord(v->scratch_done, s));
  return VX_OK;
}

int vx_map_pin(MapSlot* m, cudaStream_t s) {
  if (m->ready) VX_CUDA(cudaStreamWaitEvent(s, m->ready, 0));
  ++m->pins;
  return VX_OK;
}

int vx_map_release(vx_volume* v, MapSlot* m, cudaStream_t s) {
  if (!m) return VX_OK;
  std::lock_guard<std::mutex> lock(v->mu);
  --m->pins;
  MapUse* use = nullptr;
  for (auto& u : m->uses)
    if (u.stream == s) use = &u;
  if (!use) {
    MapUse u;
    u.stream = s;
    VX_CUDA(cudaEventCreateWithFlags(&u.ev, cudaEventDisableTiming));
    m->uses.push_back(u);
    use = &m->uses.back();
  }
  VX_CUDA(cudaEventRecord(use->ev, s));
  return VX_OK;
}

int vx_map_octants(vx_volume* v, MapSlot* m, unsigned need, unsigned* built_out, cudaStream_t s) {
  need &= 0xffu;
  if (need && !m->oct) {
    // one block for all eight orthants, kept with the slot (reused by the
    // next setting that takes it)
    VX_CUDA(cudaMalloc(&m->oct, 8 * v->cmap_bytes));
  }
  for (int o = 0; o < 8; ++o) {
    if (!((need >> o) & 1u)) continue;
    if (!m->oct_ready[o]) VX_CUDA(cudaEventCreateWithFlags(&m->oct_ready[o], cudaEventDisableTiming));
    if ((m->oct_built >> o) & 1u) {  // built by some stream: wait for it
      VX_CUDA(cudaStreamWaitEvent(s, m->oct_ready[o], 0));
      continue;
    }
    VX_CUDA(cudaStreamWaitEvent(s, v->scratch_done, 0));
    int rc = vx_launch_dist_cells_oct(v, m->occ_src, m->oct + (uint64_t)o * v->cmap_bytes,
                                      m->occ_thr, o, s);
    if (rc) return rc;
    VX_CUDA(cudaEventRecord(m->oct_ready[o], s));
    VX_CUDA(cudaEventRecord(v->scratch_done, s));
    m->oct_built |= 1u << o;
  }
  *built_out = m->oct_built & need;
  return VX_OK;
}

int vx_get_dist_map(vx_volume* v, int thr, const uint8_t** map_out, MapSlot** slot_out,
                    cudaStream_t s) {
  *map_out = nullptr;
  *slot_out = nullptr;
  std::lock_guard<std::mutex> lock(v->mu);
  ++v->stamp;
  for (auto& d : v->dist) {
    if (d.thr >= 0 && d.thr == thr) {
      d.stamp = v->stamp;
      int rc = vx_map_pin(&d, s);
      if (rc) return rc;
      *map_out = d.map;
      *slot_out = &d;
      return VX_OK;
    }
  }
  DistEntry* victim = nullptr;
  for (auto& d : v->dist) {
    if (d.pins) continue;  // a render between lookup and launch still needs it
    if (d.thr < 0) {
      victim = &d;
      break;
    }
    if (!victim || d.stamp < victim->stamp) victim = &d;
  }
  if (!victim) return VX_OK;  // every slot in flight: this frame renders without skipping
  victim->thr = -1;
  int rc = vx_map_claim(v, victim, s);  // after every K4 that read the old map
  if (rc) return rc;
  rc = vx_launch_dist_map(v, thr, victim->map, s);
  if (rc) return rc;
  victim->occ_src = v->cmax;  // orthant maps threshold the cell max map
  victim->occ_thr = thr;
  if ((rc = vx_map_publish(v, victim, s))) return rc;
  if ((rc = vx_map_pin(victim, s))) return rc;
  victim->thr = thr;
  victim->stamp = v->stamp;
  *map_out = victim->map;
  *slot_out = victim;
  return VX_OK;
}

extern "C" int vx_volume_distance_map(vx_volume* v, int32_t thr, int32_t level,
                                      uint8_t* host_out, int64_t dims_out[3]) {
  const bool orthant = level >= 8 && level < 16;
  if (!v || (level != 0 && level != 1 && !orthant)) {
    vx_set_error("vx_volume_distance_map: bad argument");
    return VX_EINVAL;
  }
  const bool cells = level != 0;
  if (dims_out) {
    dims_out[0] = cells ? v->ncx + 2 : v->nbx + 2;
    dims_out[1] = cells ? v->ncy + 2 : v->nby + 2;
    dims_out[2] = cells ? v->ncz + 2 : v->nbz + 2;
  }
  if (!host_out) return VX_OK;
  cudaStream_t s = vx_stream();
  const uint8_t* map = nullptr;
  MapSlot* slot = nullptr;
  int rc = vx_get_dist_map(v, thr, &map, &slot, s);
  if (rc) return rc;
  if (!map) {
    vx_set_error("vx_volume_distance_map: every map slot is in use");
    return VX_EINVAL;
  }
  const uint8_t* src = level == 0 ? map : map + v->map_bytes;
  if (orthant) {
    unsigned built = 0;
    {
      std::lock_guard<std::mutex> lock(v->mu);
      rc = vx_map_octants(v, slot, 1u << (level - 8), &built, s);
    }
    if (rc) {
      vx_map_release(v, slot, s);
      return rc;
    }
    src = slot->oct + (uint64_t)(level - 8) * v->cmap_bytes;
  }
  cudaError_t e = cudaMemcpyAsync(host_out, src, cells ? v->cmap_bytes : v->map_bytes,
                                  cudaMemcpyDeviceToHost, s);
  rc = vx_map_release(v, slot, s);
  if (e != cudaSuccess) return vx_cuda_fail(e, "cudaMemcpyAsync(map)", __FILE__, __LINE__);
  if (rc) return rc;
  VX_CUDA(cudaStreamSynchronize(s));
  return VX_OK;
}

// ---------------------------------------------------------------------------
// statistics

extern "C" int vx_histogram(vx_volume* v, uint64_t counts_out[256]) {
  if (!v || !counts_out) {
    vx_set_error("vx_histogram: null argument");
    return VX_EINVAL;
  }
  memcpy(counts_out, v->counts, 256 * 8);
  return VX_OK;
}

extern "C" int vx_histogram_device(const uint8_t* dev, uint64_t n, uint64_t* dev_counts,
                                   void* stream) {
  if ((!dev && n) || !dev_counts) {
    vx_set_error("vx_histogram_device: null argument");
    return VX_EINVAL;
  }
  cudaStream_t s = (cudaStream_t)stream;
  return vx_launch_hist(dev, n, dev_counts, s);
}

extern "C" int vx_volume_histogram_slab(vx_volume* v, int64_t z0, int64_t z1, uint64_t* dev_counts,
                                        void* stream) {
  if (!v || !dev_counts || z0 < 0 || z1 > v->nz || z0 > z1) {
    vx_set_error("vx_volume_histogram_slab: bad argument (planes [%lld, %lld) of %d)",
                 (long long)z0, (long long)z1, v ? v->nz : 0);
    return VX_EINVAL;
  }
  if (z0 == z1) return VX_OK;
  cudaStream_t s = (cudaStream_t)stream;
  // whole padded planes are contiguous: count them, then take the apron's
  // zeros (every padded plane holds sz - nx*ny of them) out of bin 0
  const uint64_t planes = (uint64_t)(z1 - z0);
  int rc = vx_launch_hist(v->alloc + (uint64_t)(z0 + VX_PAD) * v->sz, planes * v->sz, dev_counts, s);
  if (rc) return rc;
  return vx_launch_sub_bin0(dev_counts, planes * ((uint64_t)v->sz - (uint64_t)v->nx * v->ny), s);
}

extern "C" int vx_histogram_host(const uint8_t* host, uint64_t n, uint64_t counts_out[256]) {
  if ((!host && n) || !counts_out) {
    vx_set_error("vx_histogram_host: null argument");
    return VX_EINVAL;
  }
  cudaStream_t s = vx_stream();
  uint8_t* buf = nullptr;
  VX_CUDA(vx_malloc_async(&buf, n + 256 * 8, s));
  uint64_t* dc = reinterpret_cast<uint64_t*>(buf);
  uint8_t* data = buf + 256 * 8;
  int rc = VX_OK;
  cudaError_t e = cudaMemsetAsync(dc, 0, 256 * 8, s);
  if (e == cudaSuccess && n) e = cudaMemcpyAsync(data, host, n, cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) rc = vx_cuda_fail(e, "upload", __FILE__, __LINE__);
  if (!rc) rc = vx_launch_hist(data, n, dc, s);
  if (!rc) {
    e = cudaMemcpyAsync(counts_out, dc, 256 * 8, cudaMemcpyDeviceToHost, s);
    if (e != cudaSuccess) rc = vx_cuda_fail(e, "download", __FILE__, __LINE__);
  }
  cudaFreeAsync(buf, s);
  e = cudaStreamSynchronize(s);
  if (!rc && e != cudaSuccess) rc = vx_cuda_fail(e, "sync", __FILE__, __LINE__);
  return rc;
}

extern "C" int vx_otsu_device(const uint64_t* dev_counts, int32_t* dev_T, void* stream) {
  if (!dev_counts || !dev_T) {
    vx_set_error("vx_otsu_device: null argument");
    return VX_EINVAL;
  }
  cudaStream_t s = (cudaStream_t)stream;
  return vx_launch_otsu(dev_counts, dev_T, s);
}

extern "C" int vx_histogram_otsu_device(const uint8_t* dev, uint64_t n, uint64_t* dev_counts,
                                        int32_t* dev_T, void* stream) {
  if ((!dev && n) || !dev_counts || !dev_T) {
    vx_set_error("vx_histogram_otsu_device: null argument");
    return VX_EINVAL;
  }
  return vx_launch_hist_otsu(dev, n, dev_counts, dev_T, (cudaStream_t)stream);
}

extern "C" int vx_otsu(const uint64_t counts[256], int32_t* T_out) {
  if (!counts || !T_out) {
    vx_set_error("vx_otsu: null argument");
    return VX_EINVAL;
  }
  unsigned __int128 total = 0;
  for (int i = 0; i < 256; ++i) total += counts[i];
  if (total == 0) {
    vx_set_error("histogram is empty (all bins zero)");
    return VX_EINVAL;
  }
  if (total >= ((unsigned __int128)1 << 47)) {
    vx_set_error("histogram total %.3e exceeds the exact 320-bit Otsu range (2^47)",
                 (double)total);
    return VX_ERANGE;
  }
  cudaStream_t s = vx_stream();
  uint8_t* buf = nullptr;
  VX_CUDA(vx_malloc_async(&buf, 256 * 8 + 16, s));
  uint64_t* dc = reinterpret_cast<uint64_t*>(buf);
  int32_t* dT = reinterpret_cast<int32_t*>(buf + 256 * 8);
  VX_CUDA(cudaMemcpyAsync(dc, counts, 256 * 8, cudaMemcpyHostToDevice, s));
  int rc = vx_launch_otsu(dc, dT, s);
  if (rc) return rc;
  VX_CUDA(cudaMemcpyAsync(T_out, dT, 4, cudaMemcpyDeviceToHost, s));
  VX_CUDA(cudaFreeAsync(buf, s));
  VX_CUDA(cudaStreamSynchronize(s));
  return VX_OK;
}

extern "C" int vx_entropy_from_counts_device(const uint64_t* dev_counts, uint64_t n,
                                             double* dev_H, void* stream) {
  if (!dev_counts || !dev_H) {
    vx_set_error("vx_entropy_from_counts_device: null argument");
    return VX_EINVAL;
  }
  cudaStream_t s = (cudaStream_t)stream;
  return vx_launch_entropy(dev_counts, n, dev_H, s);
}

extern "C" int vx_image_entropy(const uint8_t* host_pixels, int64_t n, double* H_out,
                                uint64_t counts_out[256]) {
  if (!host_pixels || n <= 0 || !H_out) {
    vx_set_error("empty image");
    return VX_EINVAL;
  }
  cudaStream_t s = vx_stream();
  uint8_t* buf = nullptr;
  VX_CUDA(vx_malloc_async(&buf, 256 * 8 + 16 + n, s));
  uint64_t* dc = reinterpret_cast<uint64_t*>(buf);
  double* dH = reinterpret_cast<double*>(buf + 256 * 8);
  uint8_t* data = buf + 256 * 8 + 16;
  VX_CUDA(cudaMemsetAsync(dc, 0, 256 * 8, s));
  VX_CUDA(cudaMemcpyAsync(data, host_pixels, n, cudaMemcpyHostToDevice, s));
  int rc = vx_launch_hist(data, (uint64_t)n, dc, s);
  if (!rc) rc = vx_launch_entropy(dc, (uint64_t)n, dH, s);
  if (rc) return rc;
  VX_CUDA(cudaMemcpyAsync(H_out, dH, 8, cudaMemcpyDeviceToHost, s));
  if (counts_out) VX_CUDA(cudaMemcpyAsync(counts_out, dc, 256 * 8, cudaMemcpyDeviceToHost, s));
  VX_CUDA(cudaFreeAsync(buf, s));
  VX_CUDA(cudaStreamSynchronize(s));
  return VX_OK;
}
