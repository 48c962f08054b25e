// Direct-to-device volume ingestion: load_raw
// (volume.py:122-151) and load_slice_stack (volume.py:163-188) stream the
// file payload through page-locked staging slots straight into the device
// replica, instead of building the whole volume in host memory first and
// uploading it afterwards.
//
// Pipeline (three slots):
//   reader thread : pread() the next chunk of payload bytes into a free slot
//   this thread   : H2D copy of the slot -> [u16: (v+128)/257 on device]
//                   -> D2H of the 8-bit chunk / host memcpy into the
//                   caller's Volume bytes, then release the slot
// so the file read of chunk i+1 overlaps the DMA and host copy of chunk i.
// The 8-bit chunks land in a compact device buffer; vx_volume_finish then
// builds the padded replica, K1 histogram and max maps exactly as for an
// in-memory upload (same bytes, same results).

#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <condition_variable>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "vx_internal.cuh"

namespace {

struct Segment {
  int fd;
  int64_t offset;  // payload start in the file
  int64_t bytes;   // payload bytes
};

constexpr int kSlots = 3;

struct Slot {
  uint8_t* pin_in = nullptr;   // chunk of file bytes
  uint8_t* pin_u8 = nullptr;   // 8-bit chunk back from the device (u16 + host copy)
  int64_t dst = 0;             // destination offset in 8-bit elements
  int64_t bytes = 0;           // file bytes in pin_in
  bool full = false;
  bool last = false;
};

struct Pipe {
  std::mutex mu;
  std::condition_variable cv;
  Slot slot[kSlots];
  std::string error;
};

bool read_full(int fd, uint8_t* dst, int64_t off, int64_t n, std::string& err) {
  while (n > 0) {
    const ssize_t r = pread(fd, dst, (size_t)n, (off_t)off);
    if (r < 0) {
      err = std::string("read failed: ") + strerror(errno);
      return false;
    }
    if (r == 0) {
      err = "unexpected end of file";
      return false;
    }
    dst += r;
    off += r;
    n -= r;
  }
  return true;
}

// page-locked staging kept across loads (pinning 300 MB costs ~0.3 s):
// one cached block per size, handed out exclusively
std::mutex g_pin_mu;
std::vector<std::pair<size_t, uint8_t*>> g_pin_cache;

uint8_t* pin_get(size_t bytes) {
  {
    std::lock_guard<std::mutex> lk(g_pin_mu);
    for (auto it = g_pin_cache.begin(); it != g_pin_cache.end(); ++it) {
      if (it->first == bytes) {
        uint8_t* p = it->second;
        g_pin_cache.erase(it);
        return p;
      }
    }
  }
  void* p = nullptr;
  return cudaHostAlloc(&p, bytes, cudaHostAllocDefault) == cudaSuccess
             ? static_cast<uint8_t*>(p)
             : nullptr;
}

void pin_put(size_t bytes, uint8_t* p) {
  if (!p) return;
  std::lock_guard<std::mutex> lk(g_pin_mu);
  if (g_pin_cache.size() < 2 * kSlots) {
    g_pin_cache.emplace_back(bytes, p);
    return;
  }
  cudaFreeHost(p);
}

int64_t chunk_bytes(int bpp) {
  int64_t mb = 64;
  if (const char* e = getenv("VOXB200_IO_CHUNK_MB")) mb = atoll(e) > 0 ? atoll(e) : 64;
  int64_t c = mb << 20;
  return c - c % (2 * bpp);
}

// stream the segments' payload (bpp bytes per voxel, little endian) into a
// new volume; host_u8 (nullable) receives the 8-bit voxels as well
int ingest(const std::vector<Segment>& segs, int bpp, int64_t nx, int64_t ny, int64_t nz,
           uint8_t* host_u8, vx_volume** out) {
  const int64_t n = nx * ny * nz;
  int64_t total = 0;
  for (const auto& s : segs) total += s.bytes;
  if (total != n * bpp) {
    vx_set_error("payload holds %lld bytes, dims need %lld", (long long)total,
                 (long long)(n * bpp));
    return VX_EINVAL;
  }
  cudaStream_t s = vx_stream();
  const int64_t chunk = std::min<int64_t>(chunk_bytes(bpp), total);
  Pipe P;
  uint8_t* compact = nullptr;
  uint8_t* dev_in = nullptr;  // u16 device staging, one chunk per slot
  int rc = VX_OK;
  auto fail = [&](cudaError_t e, const char* what) {
    if (!rc) rc = vx_cuda_fail(e, what, __FILE__, __LINE__);
  };
  cudaError_t e = cudaMalloc(&compact, (size_t)n);
  if (e != cudaSuccess) fail(e, "cudaMalloc(compact volume)");
  if (!rc && bpp == 2) {
    e = cudaMalloc(&dev_in, (size_t)chunk * kSlots);
    if (e != cudaSuccess) fail(e, "cudaMalloc(u16 staging)");
  }
  cudaEvent_t ev[kSlots] = {};
  for (int i = 0; i < kSlots && !rc; ++i) {
    Slot& sl = P.slot[i];
    sl.pin_in = pin_get((size_t)chunk);
    if (bpp == 2 && host_u8) sl.pin_u8 = pin_get((size_t)chunk / 2);
    if (!sl.pin_in || (bpp == 2 && host_u8 && !sl.pin_u8)) {
      vx_set_error("cudaHostAlloc of the ingestion staging failed");
      rc = VX_ENOMEM;
      break;
    }
    e = cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming);
    if (e != cudaSuccess) fail(e, "staging events");
  }

  bool abort_read = false;
  std::thread reader;
  if (!rc) {
    reader = std::thread([&]() {
      size_t seg = 0;
      int64_t seg_off = 0, dst = 0;
      for (int k = 0; dst < n; k = (k + 1) % kSlots) {
        Slot& sl = P.slot[k];
        {
          std::unique_lock<std::mutex> lk(P.mu);
          P.cv.wait(lk, [&] { return !sl.full || abort_read; });
          if (abort_read) return;
        }
        // gather up to `chunk` bytes across segment boundaries
        int64_t got = 0;
        std::string err;
        while (got < chunk && seg < segs.size()) {
          const int64_t take = std::min(chunk - got, segs[seg].bytes - seg_off);
          if (!read_full(segs[seg].fd, sl.pin_in + got, segs[seg].offset + seg_off, take, err))
            break;
          got += take;
          seg_off += take;
          if (seg_off == segs[seg].bytes) {
            ++seg;
            seg_off = 0;
          }
        }
        std::lock_guard<std::mutex> lk(P.mu);
        if (!err.empty()) {
          P.error = err;
          sl.full = true;
          sl.last = true;
          P.cv.notify_all();
          return;
        }
        sl.dst = dst;
        sl.bytes = got;
        dst += got / bpp;
        sl.last = dst >= n;
        sl.full = true;
        P.cv.notify_all();
      }
    });
  }

  for (int k = 0; !rc; k = (k + 1) % kSlots) {
    Slot& sl = P.slot[k];
    {
      std::unique_lock<std::mutex> lk(P.mu);
      P.cv.wait(lk, [&] { return sl.full; });
      if (!P.error.empty()) {
        vx_set_error("%s", P.error.c_str());
        rc = VX_EINVAL;
        break;
      }
    }
    const int64_t m = sl.bytes / bpp;  // 8-bit voxels in this chunk
    if (bpp == 1) {
      e = cudaMemcpyAsync(compact + sl.dst, sl.pin_in, (size_t)m, cudaMemcpyHostToDevice, s);
      if (e != cudaSuccess) fail(e, "chunk upload");
      if (host_u8) memcpy(host_u8 + sl.dst, sl.pin_in, (size_t)m);  // overlaps the DMA
    } else {
      uint8_t* din = dev_in + (int64_t)k * chunk;
      e = cudaMemcpyAsync(din, sl.pin_in, (size_t)sl.bytes, cudaMemcpyHostToDevice, s);
      if (e != cudaSuccess) fail(e, "chunk upload");
      if (!rc) rc = vx_launch_u16_to_u8(reinterpret_cast<const uint16_t*>(din), compact + sl.dst,
                                        (uint64_t)m, s);
      if (!rc && host_u8) {
        e = cudaMemcpyAsync(sl.pin_u8, compact + sl.dst, (size_t)m, cudaMemcpyDeviceToHost, s);
        if (e != cudaSuccess) fail(e, "chunk readback");
      }
    }
    if (!rc) {
      e = cudaEventRecord(ev[k], s);
      if (e == cudaSuccess) e = cudaEventSynchronize(ev[k]);
      if (e != cudaSuccess) fail(e, "chunk pipeline");
    }
    if (!rc && bpp == 2 && host_u8) memcpy(host_u8 + sl.dst, sl.pin_u8, (size_t)m);
    const bool last = sl.last;
    {
      std::lock_guard<std::mutex> lk(P.mu);
      sl.full = false;
      P.cv.notify_all();
    }
    if (last) break;
  }
  if (reader.joinable()) {
    {
      std::lock_guard<std::mutex> lk(P.mu);
      abort_read = true;
      P.cv.notify_all();
    }
    reader.join();
  }
  if (!rc) {
    vx_volume* v = nullptr;
    rc = vx_volume_alloc(nx, ny, nz, &v);
    if (!rc) {
      rc = vx_volume_finish(v, compact, s);
      if (rc)
        vx_volume_destroy(v);
      else
        *out = v;
    }
  }
  cudaStreamSynchronize(s);
  for (int i = 0; i < kSlots; ++i) {
    pin_put((size_t)chunk, P.slot[i].pin_in);
    pin_put((size_t)chunk / 2, P.slot[i].pin_u8);
    if (ev[i]) cudaEventDestroy(ev[i]);
  }
  if (dev_in) cudaFree(dev_in);
  if (compact) cudaFree(compact);
  return rc;
}

struct Fds {
  std::vector<int> fds;
  ~Fds() {
    for (int fd : fds)
      if (fd >= 0) close(fd);
  }
};

int open_file(const char* path, Fds& F, int64_t* size) {
  const int fd = open(path, O_RDONLY | O_CLOEXEC);
  if (fd < 0) {
    vx_set_error("%s: %s", path, strerror(errno));
    return VX_EINVAL;
  }
  F.fds.push_back(fd);
  struct stat st;
  if (fstat(fd, &st) != 0) {
    vx_set_error("%s: %s", path, strerror(errno));
    return VX_EINVAL;
  }
  *size = (int64_t)st.st_size;
  posix_fadvise(fd, 0, 0, POSIX_FADV_SEQUENTIAL);
  return VX_OK;
}

}  // namespace

extern "C" int vx_volume_load_raw(const char* path, int64_t nx, int64_t ny, int64_t nz,
                                  int32_t bit_depth, uint8_t* host_u8_out, vx_volume** out) {
  if (!path || !out) {
    vx_set_error("vx_volume_load_raw: null argument");
    return VX_EINVAL;
  }
  if (bit_depth != 8 && bit_depth != 16) {
    vx_set_error("bit_depth must be 8 or 16, got %d", bit_depth);
    return VX_EINVAL;
  }
  if (nx < 1 || ny < 1 || nz < 1) {
    vx_set_error("dims must each be >= 1, got (%lld, %lld, %lld)", (long long)nx, (long long)ny,
                 (long long)nz);
    return VX_EINVAL;
  }
  Fds F;
  int64_t size = 0;
  int rc = open_file(path, F, &size);
  if (rc) return rc;
  const int bpp = bit_depth / 8;
  const int64_t expected = nx * ny * nz * bpp;
  if (size != expected) {  // volume.py:137-142
    vx_set_error("%s: expected %lld bytes for dims (%lld, %lld, %lld) at %d-bit, file has %lld",
                 path, (long long)expected, (long long)nx, (long long)ny, (long long)nz, bit_depth,
                 (long long)size);
    return VX_EINVAL;
  }
  std::vector<Segment> segs{{F.fds[0], 0, size}};
  return ingest(segs, bpp, nx, ny, nz, host_u8_out, out);
}

extern "C" int vx_volume_load_slices(const char* const* paths, const int64_t* payload_offsets,
                                     int64_t n_slices, int64_t width, int64_t height,
                                     uint8_t* host_u8_out, vx_volume** out) {
  if (!paths || !payload_offsets || !out || n_slices < 1 || width < 1 || height < 1) {
    vx_set_error("vx_volume_load_slices: bad argument");
    return VX_EINVAL;
  }
  Fds F;
  std::vector<Segment> segs;
  const int64_t plane = width * height;
  for (int64_t i = 0; i < n_slices; ++i) {
    int64_t size = 0;
    int rc = open_file(paths[i], F, &size);
    if (rc) return rc;
    if (size - payload_offsets[i] < plane) {  // images.py:47-48
      vx_set_error("%s: PGM payload shorter than %lldx%lld", paths[i], (long long)width,
                   (long long)height);
      return VX_EINVAL;
    }
    segs.push_back({F.fds.back(), payload_offsets[i], plane});
  }
  return ingest(segs, 1, width, height, n_slices, host_u8_out, out);
}
