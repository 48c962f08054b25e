// Sort-first frame group: several GPUs (one process or thread each) render
// one frame together, every rank's K4 writing its tiles straight into rank
// 0's frame buffer over NVLink.
//
// Reference: render_frame splits a frame into row bands on a thread pool and
// is bit-identical for any worker count (render.py:514-541,
// test_render.py:242-251).  Here the unit is the 8x16 tile, dealt round-robin
// (tile t -> rank t % world) so early-terminating hit rays and long miss
// rays balance; pixels are per-ray pure functions, so the frame is identical
// for any world size.
//
// Per frame there is no collective.  Rank 0 owns two frame slots (pixels +
// the 259 fused counters: image histogram, hit count, samples, truncation
// flag).  Every rank's K4 stores its pixels into slot f & 1 of rank 0 (peer
// or IPC-mapped pointer) and adds its counters with system-scope atomics.
// Completion and buffer reuse are two monotonic 32-bit flags written with
// stream memory operations (no kernel, no SM spins):
//   rank r > 0:  wait  consumed_r >= f - 2      (its local flag; rank 0 has
//                                                released slot f & 1)
//                K4 -> slot f & 1 of rank 0
//                write done_r[rank 0] = f       (fenced: K4's stores first)
//   rank 0:      K4 -> slot f & 1
//                wait  done_r >= f  for every r (its local flags)
//                ... the caller consumes the frame (D2H copy, display) ...
//   release:     zero slot f & 1's counters, write consumed_r[r] = f
// The waits are cyclic 32-bit compares (CU_STREAM_WAIT_VALUE_GEQ), so the
// counters may wrap.  Only the stream front end blocks; nothing spins.
//
// Ranks that share one GPU (a functional test on a one-GPU box) must not
// wait on each other on the device (a context blocked on another context of
// the same GPU can time out, B200_PROFILING.md): VX_GROUP_SYNC_HOST leaves
// the ordering to the caller (stream sync + a host barrier per frame); the
// data path -- peer stores and system-scope atomics into rank 0's slot -- is
// the same.

#include <cuda.h>  // driver types of the stream memory operations (entry points fetched at run time)
#include <unistd.h>

#include <cstring>
#include <mutex>
#include <new>

#include "vx_internal.cuh"

namespace {

constexpr uint32_t kBlobMagic = 0x56584742u;  // "VXGB"
constexpr int kMaxWorld = 64;
constexpr uint64_t kFlagBytes = 4096;  // done[64] at 0, consumed at 512
constexpr uint64_t kConsumedOff = 512;
constexpr int kCounters = 260;         // 256 bins, hits, samples, trunc flag, pad

struct GroupBlob {
  uint32_t magic;
  int32_t rank, world, device;
  int32_t pid, pad;
  uint64_t host_hash;
  uint64_t dev_ptr;
  uint64_t bytes;
  int64_t max_pixels;
  uint8_t uuid[16];
  cudaIpcMemHandle_t ipc;
};
static_assert(sizeof(GroupBlob) <= VX_GROUP_BLOB_BYTES, "group blob size");

typedef CUresult (*PfnValue32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
PfnValue32 g_wait32 = nullptr, g_write32 = nullptr;
std::once_flag g_memops_once;
int g_memops_rc = VX_OK;

int load_memops() {
  std::call_once(g_memops_once, [] {
    cudaDriverEntryPointQueryResult q1, q2;
    void* w = nullptr;
    void* x = nullptr;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &w, cudaEnableDefault, &q1) != cudaSuccess ||
        cudaGetDriverEntryPoint("cuStreamWriteValue32", &x, cudaEnableDefault, &q2) != cudaSuccess ||
        q1 != cudaDriverEntryPointSuccess || q2 != cudaDriverEntryPointSuccess || !w || !x) {
      cudaGetLastError();
      g_memops_rc = VX_ECUDA;
      return;
    }
    g_wait32 = reinterpret_cast<PfnValue32>(w);
    g_write32 = reinterpret_cast<PfnValue32>(x);
  });
  if (g_memops_rc) vx_set_error("stream memory operations (cuStreamWaitValue32) unavailable");
  return g_memops_rc;
}

int cu_check(CUresult r, const char* what) {
  if (r == CUDA_SUCCESS) return VX_OK;
  vx_set_error("%s failed (CUresult %d)", what, (int)r);
  return VX_ECUDA;
}

// a fenced stream write and a satisfied wait on `flag` (device memory)
int memop_probe(uint8_t* flag) {
  cudaStream_t ps;
  VX_CUDA(cudaStreamCreateWithFlags(&ps, cudaStreamNonBlocking));
  int rc = cu_check(g_write32((CUstream)ps, (CUdeviceptr)flag, 1u, 0), "cuStreamWriteValue32(probe)");
  if (!rc)
    rc = cu_check(g_wait32((CUstream)ps, (CUdeviceptr)flag, 1u, CU_STREAM_WAIT_VALUE_GEQ),
                  "cuStreamWaitValue32(probe)");
  cudaError_t e = cudaStreamSynchronize(ps);
  cudaStreamDestroy(ps);
  if (rc) return rc;
  if (e != cudaSuccess) return vx_cuda_fail(e, "stream memop probe", __FILE__, __LINE__);
  return VX_OK;
}

uint64_t host_hash() {
  char name[256] = {0};
  gethostname(name, sizeof(name) - 1);
  uint64_t h = 1469598103934665603ull;  // FNV-1a
  for (const char* c = name; *c; ++c) h = (h ^ (uint8_t)*c) * 1099511628211ull;
  return h;
}

uint64_t slot_pixels(int64_t max_pixels) { return ((uint64_t)max_pixels + 255) & ~uint64_t(255); }

}  // namespace

struct vx_group {
  int rank = 0, world = 1, device = 0, sync = VX_GROUP_SYNC_HOST;
  int64_t max_pixels = 0;
  uint64_t slot_bytes = 0;
  uint8_t* local = nullptr;  // this rank's block: flags (+ the two frame slots on rank 0)
  uint64_t local_bytes = 0;
  uint8_t* peer[kMaxWorld] = {};   // blocks this rank writes into (self = local)
  bool ipc_open[kMaxWorld] = {};
  bool connected = false;
  uint32_t frame = 0;     // frames this rank has rendered
  uint32_t released = 0;  // rank 0: frames released back to the peers
  GroupBlob blob;
};

static uint8_t* slot_of(const vx_group* g, uint32_t f) {
  return g->peer[0] + kFlagBytes + (uint64_t)(f & 1u) * g->slot_bytes;
}

extern "C" int vx_group_create(int32_t rank, int32_t world, int64_t max_pixels, vx_group** out,
                               uint8_t* blob_out) {
  if (!out || !blob_out || world < 1 || world > kMaxWorld || rank < 0 || rank >= world ||
      max_pixels < 1) {
    vx_set_error("vx_group_create: bad argument (rank %d, world %d, max_pixels %lld; world <= %d)",
                 rank, world, (long long)max_pixels, kMaxWorld);
    return VX_EINVAL;
  }
  vx_group* g = new (std::nothrow) vx_group();
  if (!g) {
    vx_set_error("host allocation failed");
    return VX_ENOMEM;
  }
  g->rank = rank;
  g->world = world;
  g->max_pixels = max_pixels;
  g->slot_bytes = (slot_pixels(max_pixels) + kCounters * 8 + 255) & ~uint64_t(255);
  cudaError_t e0 = cudaGetDevice(&g->device);
  if (e0 != cudaSuccess) {
    delete g;
    return vx_cuda_fail(e0, "cudaGetDevice", __FILE__, __LINE__);
  }
  g->local_bytes = kFlagBytes + (rank == 0 ? 2 * g->slot_bytes : 0);
  cudaError_t e = cudaMalloc(&g->local, g->local_bytes);
  if (e != cudaSuccess) {
    delete g;
    return vx_cuda_fail(e, "cudaMalloc(group block)", __FILE__, __LINE__);
  }
  e = cudaMemset(g->local, 0, g->local_bytes);
  if (e != cudaSuccess) {
    cudaFree(g->local);
    delete g;
    return vx_cuda_fail(e, "cudaMemset(group block)", __FILE__, __LINE__);
  }
  GroupBlob& b = g->blob;
  memset(&b, 0, sizeof(b));
  b.magic = kBlobMagic;
  b.rank = rank;
  b.world = world;
  b.device = g->device;
  b.pid = (int32_t)getpid();
  b.host_hash = host_hash();
  b.dev_ptr = (uint64_t)(uintptr_t)g->local;
  b.bytes = g->local_bytes;
  b.max_pixels = max_pixels;
  cudaDeviceProp prop;
  e = cudaGetDeviceProperties(&prop, g->device);
  if (e == cudaSuccess) memcpy(b.uuid, &prop.uuid, 16);
  e = cudaIpcGetMemHandle(&b.ipc, g->local);
  if (e != cudaSuccess) {
    cudaFree(g->local);
    delete g;
    return vx_cuda_fail(e, "cudaIpcGetMemHandle", __FILE__, __LINE__);
  }
  memset(blob_out, 0, VX_GROUP_BLOB_BYTES);
  memcpy(blob_out, &b, sizeof(b));
  *out = g;
  return VX_OK;
}

extern "C" int vx_group_connect(vx_group* g, const uint8_t* blobs, int32_t sync) {
  if (!g || !blobs || g->connected) {
    vx_set_error("vx_group_connect: bad argument or already connected");
    return VX_EINVAL;
  }
  bool shared_gpu = false, one_process = true;
  GroupBlob bs[kMaxWorld];
  for (int r = 0; r < g->world; ++r) {
    memcpy(&bs[r], blobs + (size_t)r * VX_GROUP_BLOB_BYTES, sizeof(GroupBlob));
    const GroupBlob& b = bs[r];
    if (b.magic != kBlobMagic || b.rank != r || b.world != g->world ||
        b.max_pixels != g->max_pixels) {
      vx_set_error("vx_group_connect: blob %d does not belong to this group (rank %d, world %d, "
                   "max_pixels %lld)", r, b.rank, b.world, (long long)b.max_pixels);
      return VX_EINVAL;
    }
    if (b.host_hash != g->blob.host_hash) {
      vx_set_error("vx_group_connect: rank %d runs on another host (peer memory is node-local)", r);
      return VX_EINVAL;
    }
    for (int q = 0; q < r; ++q)
      if (!memcmp(bs[q].uuid, b.uuid, 16)) shared_gpu = true;
    if (b.pid != g->blob.pid) one_process = false;
  }
  if (sync == VX_GROUP_SYNC_AUTO) sync = shared_gpu ? VX_GROUP_SYNC_HOST : VX_GROUP_SYNC_DEVICE;
  // Ranks of one process sharing a GPU are streams of one context: their
  // flag waits are ordinary cross-stream waits (like cudaStreamWaitEvent).
  // Across processes on one GPU a blocked context can time out: refused.
  if (sync == VX_GROUP_SYNC_DEVICE && shared_gpu && !one_process) {
    vx_set_error("vx_group_connect: device-side frame flags need one GPU per rank (ranks share a "
                 "GPU: use VX_GROUP_SYNC_HOST)");
    return VX_EINVAL;
  }
  if (sync != VX_GROUP_SYNC_DEVICE && sync != VX_GROUP_SYNC_HOST) {
    vx_set_error("vx_group_connect: bad sync mode %d", sync);
    return VX_EINVAL;
  }
  if (sync == VX_GROUP_SYNC_DEVICE) {
    int rc = load_memops();
    if (rc) return rc;
    // probe on this rank's own flag block: an unsupported driver fails here
    // (the caller can fall back to VX_GROUP_SYNC_HOST), not inside a frame
    rc = memop_probe(g->local + kConsumedOff + 64);
    if (rc) return rc;
  }
  for (int r = 0; r < g->world; ++r) {
    // rank 0 writes every peer's consumed flag; peers write into rank 0
    if (r == g->rank) {
      g->peer[r] = g->local;
      continue;
    }
    if (g->rank != 0 && r != 0) continue;
    const GroupBlob& b = bs[r];
    if (b.pid == g->blob.pid) {  // same process (one thread per GPU): plain peer pointer
      if (b.device != g->device) {
        int ok = 0;
        VX_CUDA(cudaDeviceCanAccessPeer(&ok, g->device, b.device));
        if (!ok) {
          vx_set_error("vx_group_connect: device %d cannot access device %d", g->device, b.device);
          return VX_EINVAL;
        }
        cudaError_t e = cudaDeviceEnablePeerAccess(b.device, 0);
        if (e == cudaErrorPeerAccessAlreadyEnabled)
          cudaGetLastError();
        else if (e != cudaSuccess)
          return vx_cuda_fail(e, "cudaDeviceEnablePeerAccess", __FILE__, __LINE__);
      }
      g->peer[r] = reinterpret_cast<uint8_t*>((uintptr_t)b.dev_ptr);
    } else {
      void* p = nullptr;
      VX_CUDA(cudaIpcOpenMemHandle(&p, b.ipc, cudaIpcMemLazyEnablePeerAccess));
      g->peer[r] = static_cast<uint8_t*>(p);
      g->ipc_open[r] = true;
    }
  }
  if (sync == VX_GROUP_SYNC_DEVICE && g->world > 1) {
    // probe the flag writes across the mapping (rank r > 0: its done slot in
    // rank 0's block; rank 0: every peer's consumed flag) with the value the
    // flags already hold (0), so a driver or topology that cannot do them
    // fails here and the caller can fall back to VX_GROUP_SYNC_HOST
    cudaStream_t ps;
    VX_CUDA(cudaStreamCreateWithFlags(&ps, cudaStreamNonBlocking));
    int rc = VX_OK;
    for (int r = 0; r < g->world && !rc; ++r) {
      uint8_t* flag = nullptr;
      if (g->rank > 0 && r == 0) flag = g->peer[0] + 4 * g->rank;
      if (g->rank == 0 && r > 0) flag = g->peer[r] + kConsumedOff;
      if (flag) rc = cu_check(g_write32((CUstream)ps, (CUdeviceptr)flag, 0u, 0), "peer flag probe");
    }
    cudaError_t e = cudaStreamSynchronize(ps);
    cudaStreamDestroy(ps);
    if (!rc && e != cudaSuccess) rc = vx_cuda_fail(e, "peer flag probe", __FILE__, __LINE__);
    if (rc) {
      for (int r = 0; r < g->world; ++r)
        if (g->ipc_open[r]) {
          cudaIpcCloseMemHandle(g->peer[r]);
          g->ipc_open[r] = false;
        }
      for (int r = 0; r < g->world; ++r)
        if (r != g->rank) g->peer[r] = nullptr;
      return rc;
    }
  }
  g->sync = sync;
  g->connected = true;
  return VX_OK;
}

extern "C" int vx_group_probe_device_sync(void) {
  int rc = load_memops();
  if (rc) return rc;
  uint8_t* flag = nullptr;
  VX_CUDA(cudaMalloc(&flag, 64));
  VX_CUDA(cudaMemset(flag, 0, 64));
  rc = memop_probe(flag);
  cudaFree(flag);
  return rc;
}

extern "C" int vx_group_info(const vx_group* g, int32_t* sync_out, uint32_t* frame_out) {
  if (!g) {
    vx_set_error("vx_group_info: null group");
    return VX_EINVAL;
  }
  if (sync_out) *sync_out = g->sync;
  if (frame_out) *frame_out = g->frame;
  return VX_OK;
}

extern "C" int vx_group_render(vx_group* g, vx_volume* vol, const vx_ray_setup* rs,
                               const vx_render_params* rp, const vx_filter_config* fc,
                               void* stream, vx_group_frame* out) {
  if (!g || !g->connected || !vol || !rs || !rp || !fc) {
    vx_set_error("vx_group_render: null argument or group not connected");
    return VX_EINVAL;
  }
  if ((int64_t)rs->width * rs->height > g->max_pixels) {
    vx_set_error("vx_group_render: %dx%d frame exceeds the group's %lld pixels", rs->width,
                 rs->height, (long long)g->max_pixels);
    return VX_EINVAL;
  }
  const uint32_t f = g->frame + 1;
  if (g->rank == 0 && f - g->released > 2u) {
    vx_set_error("vx_group_render: frame %u's slot is still held (release frame %u first)", f,
                 f - 2);
    return VX_EINVAL;
  }
  cudaStream_t s = (cudaStream_t)stream;
  const bool dev_sync = g->sync == VX_GROUP_SYNC_DEVICE && g->world > 1;
  if (dev_sync && g->rank > 0) {  // rank 0 has released slot f & 1 (frame f - 2)
    int rc = cu_check(g_wait32((CUstream)s, (CUdeviceptr)(g->local + kConsumedOff), f - 2u,
                               CU_STREAM_WAIT_VALUE_GEQ),
                      "cuStreamWaitValue32(consumed)");
    if (rc) return rc;
  }
  uint8_t* slot = slot_of(g, f);
  uint64_t* counters = reinterpret_cast<uint64_t*>(slot + slot_pixels(g->max_pixels));
  vx_render_out d;
  memset(&d, 0, sizeof(d));
  d.pixels = slot;
  d.image_hist = counters;
  d.hit_count = counters + 256;
  d.samples = counters + 257;
  d.trunc_flag = reinterpret_cast<int32_t*>(counters + 258);
  vx_partition part;
  part.rank = g->rank;
  part.world = g->world;
  int rc = vx_render_tiles(vol, rs, rp, fc, &part, &d, s, g->world > 1);
  if (rc) return rc;
  if (dev_sync && g->rank > 0) {  // fenced: this stream's K4 stores land first
    rc = cu_check(g_write32((CUstream)s, (CUdeviceptr)(g->peer[0] + 4 * g->rank), f, 0),
                  "cuStreamWriteValue32(done)");
    if (rc) return rc;
  }
  if (dev_sync && g->rank == 0) {
    for (int r = 1; r < g->world; ++r) {
      rc = cu_check(g_wait32((CUstream)s, (CUdeviceptr)(g->local + 4 * r), f,
                             CU_STREAM_WAIT_VALUE_GEQ),
                    "cuStreamWaitValue32(done)");
      if (rc) return rc;
    }
  }
  g->frame = f;
  if (out) {
    out->pixels = slot;
    out->counters = counters;
    out->frame = f;
  }
  return VX_OK;
}

extern "C" int vx_group_release(vx_group* g, void* stream) {
  if (!g || !g->connected) {
    vx_set_error("vx_group_release: group not connected");
    return VX_EINVAL;
  }
  if (g->rank != 0) return VX_OK;
  if (g->released == g->frame) {
    vx_set_error("vx_group_release: no rendered frame to release");
    return VX_EINVAL;
  }
  cudaStream_t s = (cudaStream_t)stream;
  const uint32_t f = g->released + 1;
  uint8_t* slot = slot_of(g, f);
  VX_CUDA(cudaMemsetAsync(slot + slot_pixels(g->max_pixels), 0, kCounters * 8, s));
  if (g->sync == VX_GROUP_SYNC_DEVICE) {
    for (int r = 1; r < g->world; ++r) {
      int rc = cu_check(g_write32((CUstream)s, (CUdeviceptr)(g->peer[r] + kConsumedOff), f, 0),
                        "cuStreamWriteValue32(consumed)");
      if (rc) return rc;
    }
  }
  g->released = f;
  return VX_OK;
}

extern "C" int vx_group_download(vx_group* g, uint8_t* host_pixels, uint64_t* host_counters,
                                 int64_t n_pixels, void* stream) {
  if (!g || !g->connected || g->rank != 0 || g->frame == g->released || n_pixels < 0 ||
      n_pixels > g->max_pixels) {
    vx_set_error("vx_group_download: rank 0 of a connected group with an unreleased frame only");
    return VX_EINVAL;
  }
  cudaStream_t s = (cudaStream_t)stream;
  const uint8_t* slot = slot_of(g, g->released + 1);
  if (host_pixels && n_pixels)
    VX_CUDA(cudaMemcpyAsync(host_pixels, slot, (size_t)n_pixels, cudaMemcpyDeviceToHost, s));
  if (host_counters)
    VX_CUDA(cudaMemcpyAsync(host_counters, slot + slot_pixels(g->max_pixels), 259 * 8,
                            cudaMemcpyDeviceToHost, s));
  VX_CUDA(cudaStreamSynchronize(s));
  return VX_OK;
}

extern "C" int vx_group_destroy(vx_group* g) {
  if (!g) return VX_OK;
  int cur = 0;
  cudaGetDevice(&cur);
  if (cur != g->device) cudaSetDevice(g->device);
  cudaDeviceSynchronize();
  for (int r = 0; r < g->world; ++r)
    if (g->ipc_open[r]) cudaIpcCloseMemHandle(g->peer[r]);
  if (g->local) cudaFree(g->local);
  if (cur != g->device) cudaSetDevice(cur);
  delete g;
  return VX_OK;
}
