// One process driving several GPUs: SURVEY.md §8b's `vx_init(n_devices,
// device_ids)` and the multi-device volume / frame built on it.
//
// The frame split is the same sort-first tile deal as the multi-process
// group (vx_group.cu): the ranks are the listed devices, every device holds a
// full replica, K4 on device r renders tiles t with t % n == r straight into
// device 0's frame slot over NVLink (peer pointers; peer access enabled by
// vx_group_connect), and the frame is complete on device 0's stream once
// every rank's done flag is in (VX_GROUP_SYNC_DEVICE).  With several ranks
// on one GPU (a one-GPU box) the same calls run host-ordered.  One host
// thread enqueues every rank's work (all calls are asynchronous); the
// reference's equivalent is the row-band thread pool of render_frame
// (render.py:514-541), bit-identical for any worker count like this split.

#include <cstring>
#include <mutex>
#include <new>
#include <vector>

#include "vx_internal.cuh"

namespace {

std::mutex g_init_mu;
std::vector<int> g_devices;  // vx_init's list (empty: the current device)

struct DeviceGuard {  // restores the calling thread's device
  int prev = 0;
  DeviceGuard() { cudaGetDevice(&prev); }
  ~DeviceGuard() { cudaSetDevice(prev); }
};

}  // namespace

struct vx_multi {
  std::vector<int> dev;
  std::vector<vx_volume*> vol;
  std::vector<vx_group*> grp;
  int64_t max_pixels = 0;
  int sync = VX_GROUP_SYNC_HOST;
  int64_t nx = 0, ny = 0, nz = 0;
};

extern "C" int vx_init(int n_devices, const int* device_ids) {
  if (n_devices < 1 || n_devices > 64 || !device_ids) {
    vx_set_error("vx_init: need 1..64 device ids");
    return VX_EINVAL;
  }
  int count = 0;
  VX_CUDA(cudaGetDeviceCount(&count));
  for (int i = 0; i < n_devices; ++i)
    if (device_ids[i] < 0 || device_ids[i] >= count) {
      vx_set_error("vx_init: device %d out of range (%d visible)", device_ids[i], count);
      return VX_EINVAL;
    }
  std::lock_guard<std::mutex> lk(g_init_mu);
  g_devices.assign(device_ids, device_ids + n_devices);
  return VX_OK;
}

static void multi_free(vx_multi* m) {
  DeviceGuard g;
  for (size_t r = 0; r < m->grp.size(); ++r)
    if (m->grp[r]) {
      cudaSetDevice(m->dev[r]);
      vx_group_destroy(m->grp[r]);
    }
  for (size_t r = 0; r < m->vol.size(); ++r)
    if (m->vol[r]) {
      cudaSetDevice(m->dev[r]);
      vx_volume_destroy(m->vol[r]);
    }
  delete m;
}

extern "C" int vx_multi_volume_create_u8(const uint8_t* host, int64_t nx, int64_t ny, int64_t nz,
                                         vx_multi** out) {
  if (!host || !out) {
    vx_set_error("vx_multi_volume_create_u8: null argument");
    return VX_EINVAL;
  }
  vx_multi* m = new (std::nothrow) vx_multi();
  if (!m) {
    vx_set_error("host allocation failed");
    return VX_ENOMEM;
  }
  {
    std::lock_guard<std::mutex> lk(g_init_mu);
    m->dev = g_devices;
  }
  DeviceGuard guard;
  if (m->dev.empty()) m->dev.push_back(guard.prev);
  m->nx = nx;
  m->ny = ny;
  m->nz = nz;
  m->vol.assign(m->dev.size(), nullptr);
  m->grp.assign(m->dev.size(), nullptr);
  // the replica of the first device from the host bytes; the others copied
  // from it device to device (over NVLink between GPUs) and built there
  int rc = VX_OK;
  uint8_t* compact0 = nullptr;
  cudaSetDevice(m->dev[0]);
  rc = vx_volume_create_u8(host, nx, ny, nz, &m->vol[0]);
  if (!rc && m->dev.size() > 1) {
    const uint64_t n = (uint64_t)nx * ny * nz;
    cudaError_t e = cudaMalloc(&compact0, n);
    if (e == cudaSuccess) e = cudaMemcpy(compact0, host, n, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) rc = vx_cuda_fail(e, "compact replica source", __FILE__, __LINE__);
    for (size_t r = 1; r < m->dev.size() && !rc; ++r) {
      cudaSetDevice(m->dev[r]);
      uint8_t* c = nullptr;
      e = cudaMalloc(&c, n);
      if (e == cudaSuccess) e = cudaMemcpyPeer(c, m->dev[r], compact0, m->dev[0], n);
      if (e != cudaSuccess) {
        rc = vx_cuda_fail(e, "cudaMemcpyPeer(replica)", __FILE__, __LINE__);
      } else {
        rc = vx_volume_create_device_u8(c, nx, ny, nz, &m->vol[r]);
      }
      if (c) cudaFree(c);
    }
  }
  if (compact0) {
    cudaSetDevice(m->dev[0]);
    cudaFree(compact0);
  }
  if (rc) {
    multi_free(m);
    return rc;
  }
  *out = m;
  return VX_OK;
}

// the frame groups of the devices for frames up to max_pixels (in memory:
// the ranks are this process's)
static int multi_groups(vx_multi* m, int64_t npx) {
  if (m->grp[0] && m->max_pixels >= npx) return VX_OK;
  DeviceGuard guard;
  for (size_t r = 0; r < m->grp.size(); ++r)
    if (m->grp[r]) {
      cudaSetDevice(m->dev[r]);
      vx_group_destroy(m->grp[r]);
      m->grp[r] = nullptr;
    }
  const int n = (int)m->dev.size();
  std::vector<uint8_t> blobs((size_t)n * VX_GROUP_BLOB_BYTES);
  for (int r = 0; r < n; ++r) {
    cudaSetDevice(m->dev[r]);
    int rc = vx_group_create(r, n, npx, &m->grp[r], blobs.data() + (size_t)r * VX_GROUP_BLOB_BYTES);
    if (rc) return rc;
  }
  for (int r = 0; r < n; ++r) {
    cudaSetDevice(m->dev[r]);
    int rc = vx_group_connect(m->grp[r], blobs.data(), VX_GROUP_SYNC_AUTO);
    if (rc) return rc;
  }
  int32_t sync = 0;
  vx_group_info(m->grp[0], &sync, nullptr);
  m->sync = sync;
  m->max_pixels = npx;
  return VX_OK;
}

extern "C" int vx_multi_render(vx_multi* m, const vx_ray_setup* rs, const vx_render_params* rp,
                               const vx_filter_config* fc, vx_render_out* out) {
  if (!m || !rs || !rp || !fc || !out || !out->pixels) {
    vx_set_error("vx_multi_render: null argument");
    return VX_EINVAL;
  }
  const int64_t npx = (int64_t)rs->width * rs->height;
  if (rs->width < 1 || rs->height < 1) {
    vx_set_error("image size must be >= 1x1, got %dx%d", rs->width, rs->height);
    return VX_EINVAL;
  }
  if (m->dev.size() == 1) {  // one device: the plain frame
    DeviceGuard guard;
    cudaSetDevice(m->dev[0]);
    return vx_render(m->vol[0], rs, rp, fc, nullptr, out);
  }
  int rc = multi_groups(m, npx);
  if (rc) return rc;
  DeviceGuard guard;
  const int n = (int)m->dev.size();
  // every rank's tiles, enqueued from this thread on each device's stream;
  // rank 0 last, so its stream's flag waits come after the peers' work
  for (int r = n - 1; r >= 0; --r) {
    cudaSetDevice(m->dev[r]);
    if ((rc = vx_group_render(m->grp[r], m->vol[r], rs, rp, fc, vx_stream(), nullptr))) return rc;
  }
  if (m->sync == VX_GROUP_SYNC_HOST)  // ranks share a GPU: order on the host
    for (int r = 1; r < n; ++r) {
      cudaSetDevice(m->dev[r]);
      VX_CUDA(cudaStreamSynchronize(vx_stream()));
    }
  cudaSetDevice(m->dev[0]);
  uint64_t counters[259];
  rc = vx_group_download(m->grp[0], out->pixels, counters, npx, vx_stream());
  if (rc) return rc;
  if ((rc = vx_group_release(m->grp[0], vx_stream()))) return rc;
  int32_t flag;
  memcpy(&flag, &counters[258], 4);
  if (flag && rp->max_steps <= 0) {
    // a ray exhausted its own step budget: the exact frame budget, on device 0
    return vx_render(m->vol[0], rs, rp, fc, nullptr, out);
  }
  if (out->image_hist) memcpy(out->image_hist, counters, 256 * 8);
  if (out->hit_count) out->hit_count[0] = counters[256];
  if (out->samples) out->samples[0] = counters[257];
  if (out->trunc_flag) out->trunc_flag[0] = 0;
  return VX_OK;
}

extern "C" int vx_multi_histogram(vx_multi* m, uint64_t counts_out[256]) {
  if (!m || !counts_out) {
    vx_set_error("vx_multi_histogram: null argument");
    return VX_EINVAL;
  }
  // z-slab shards of the replicas, one per device, summed
  DeviceGuard guard;
  const int n = (int)m->dev.size();
  const int64_t per = (m->nz + n - 1) / n;
  std::vector<uint64_t*> dc(n, nullptr);
  int rc = VX_OK;
  for (int r = 0; r < n && !rc; ++r) {
    cudaSetDevice(m->dev[r]);
    cudaError_t e = cudaMalloc(&dc[r], 256 * 8);
    if (e == cudaSuccess) e = cudaMemsetAsync(dc[r], 0, 256 * 8, vx_stream());
    if (e != cudaSuccess) {
      rc = vx_cuda_fail(e, "slab histogram buffer", __FILE__, __LINE__);
      break;
    }
    const int64_t z0 = r * per < m->nz ? r * per : m->nz;
    const int64_t z1 = z0 + per < m->nz ? z0 + per : m->nz;
    rc = vx_volume_histogram_slab(m->vol[r], z0, z1, dc[r], vx_stream());
  }
  memset(counts_out, 0, 256 * 8);
  for (int r = 0; r < n; ++r) {
    if (!dc[r]) continue;
    cudaSetDevice(m->dev[r]);
    uint64_t h[256];
    if (!rc) {
      cudaError_t e = cudaMemcpyAsync(h, dc[r], 256 * 8, cudaMemcpyDeviceToHost, vx_stream());
      if (e == cudaSuccess) e = cudaStreamSynchronize(vx_stream());
      if (e != cudaSuccess) rc = vx_cuda_fail(e, "slab histogram download", __FILE__, __LINE__);
      else
        for (int b = 0; b < 256; ++b) counts_out[b] += h[b];
    }
    cudaFree(dc[r]);
  }
  return rc;
}

extern "C" int vx_multi_info(const vx_multi* m, int32_t* n_devices_out, int32_t* sync_out) {
  if (!m) {
    vx_set_error("vx_multi_info: null argument");
    return VX_EINVAL;
  }
  if (n_devices_out) *n_devices_out = (int32_t)m->dev.size();
  if (sync_out) *sync_out = m->sync;
  return VX_OK;
}

extern "C" int vx_multi_destroy(vx_multi* m) {
  if (m) multi_free(m);
  return VX_OK;
}
