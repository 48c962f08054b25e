/*
 * voxb200.h — C-ABI of libvoxb200.so, the B200 (sm_100a) implementation of
 * the arXiv 1807.03119 hot path: volume load -> Otsu histogram/threshold ->
 * first-hit ray cast with the per-hit local noise filter (and the four
 * comparison filters), Sobel normal, Phong shading -> image entropy.
 *
 * The reference (`voxray`, /root/reference/pkg/src/voxray) is pure Python;
 * it has no FFI.  Its operator API is the Python module surface
 * (pkg/src/voxray/__init__.py:3-43).  Each entry point below names the
 * reference function it replaces; the Python mirror in
 * paper_1807_03119_b200/ binds them with ctypes.
 *
 * Conventions
 *  - every function returns an int status (VX_OK = 0); on failure
 *    vx_last_error() returns a thread-local message.
 *  - plain pointers and sizes only; "host" pointers are CPU memory, "dev"
 *    pointers are CUDA device memory of the current device.
 *  - the library is re-entrant: each calling thread gets its own CUDA stream
 *    for the host-buffer entry points; the *_device entry points run on the
 *    cudaStream_t the caller passes (0 = legacy default stream).  The only
 *    shared mutable state is per-volume caches (mutex protected).
 *  - volume layout: voxel (x, y, z) of an (nx, ny, nz) volume, x fastest,
 *    exactly the reference's `Volume.data[z, y, x]` (volume.py:3-5).
 */
#ifndef VOXB200_H
#define VOXB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum vx_status {
  VX_OK = 0,
  VX_EINVAL = 1, /* bad argument (maps to the reference's *Error classes) */
  VX_ENOMEM = 2, /* device allocation failed                              */
  VX_ECUDA = 3,  /* CUDA runtime error                                    */
  VX_ERANGE = 5  /* value outside the exact-arithmetic range              */
};

/* FilterKind (filters.py:43-57), same order as the reference enum */
enum vx_filter_kind {
  VX_FILTER_NONE = 0,
  VX_FILTER_MEAN = 1,
  VX_FILTER_SIGMA = 2,
  VX_FILTER_OKADA = 3,
  VX_FILTER_ENTROPY = 4,
  VX_FILTER_LOCAL_CLUSTER = 5,
  /* vx_filter_batch only: axis_cluster_average_batch (filters.py:177-178) */
  VX_FILTER_AXIS_CLUSTER = 6
};

typedef struct vx_volume vx_volume; /* opaque device replica of a Volume */

/* Host-computed camera constants (render.py:188-201): the shim passes the
 * exact FP64 values numpy computes in Camera.basis() (render.py:49-62). */
typedef struct {
  double right[3], up[3], fwd[3];
  double origin[3]; /* Camera.position */
  double tan_f;     /* math.tan(math.radians(fov_y_deg) / 2.0)  render.py:191 */
  double aspect;    /* width / height                           render.py:192 */
  int32_t width, height;
} vx_ray_setup;

/* March + shading constants (render.py:108-150, 258-290, 385-403). */
typedef struct {
  double step_size; /* RenderParams.step_size                              */
  int32_t max_steps; /* > 0: explicit cap (RenderParams.max_steps); <= 0: derive
                        from the longest span exactly as render.py:469-473  */
  int32_t chunk;     /* max(1, min(16, int(15/step))) if step < 15 else 1    */
  int32_t need_clip; /* chunk * step > 15  (render.py:286-287)               */
  int32_t skip;      /* 1: exact empty-space skipping (default), 0: off      */
  double ambient, diffuse, specular, shininess;
  double light[3];   /* normalised light direction (render.py:512-513)      */
  int32_t background;
  int32_t _pad;
} vx_render_params;

/* Resolved FilterConfig (filters.py:60-126) plus the host statistics the
 * filters need (histogram.py:109-116, filters.py:212-218). */
typedef struct {
  int32_t kind;           /* vx_filter_kind                                  */
  int32_t kernel_size;    /* M, odd >= 3                                     */
  int32_t cluster_offset; /* d >= 1                                          */
  int32_t entropy_pairwise; /* vx_filter_batch only: 1 = numpy's 8-way pairwise
                               order (the reference's single-coordinate batch) */
  double threshold;       /* resolved T (float)                              */
  double sigma_band;      /* sigma_mult * global_sigma (FP64, host)          */
  double okada_threshold; /* T_d                                             */
  double entropy_threshold; /* T_e                                           */
  double entropy_lut[256];  /* entropy_terms(probabilities)                  */
} vx_filter_config;

/* Sort-first image partition for multi-GPU (tiles of 8x16 pixels dealt
 * round-robin: tile t belongs to rank t % world). world = 1: whole frame. */
typedef struct {
  int32_t rank, world;
} vx_partition;

/* Render outputs.  Host variants: host pointers; *_device variants: device
 * pointers.  Every pointer except pixels is nullable. */
typedef struct {
  uint8_t* pixels;       /* height*width, row-major from the top-left      */
  int32_t* hit_voxel;    /* height*width*3 (x,y,z), -1 on miss              */
  float* hit_t;          /* height*width, sample t of the accepted hit      */
  double* hit_value;     /* height*width, filter value at the hit          */
  double* intensity;     /* height*width, pre-quantisation Phong I          */
  uint64_t* image_hist;  /* [256] grey-level histogram of pixels (fused K6) */
  uint64_t* hit_count;   /* [1]                                             */
  uint64_t* samples;     /* [1] march samples taken (diagnostic)            */
  uint64_t* diag;        /* [8] march statistics (diagnostic, nullable):
                            distance lookups, skips, chunks skipped, (unused),
                            sample groups, filter evaluations, hits, ray
                            iterations                                        */
  int32_t* trunc_flag;   /* [1] set to 1 when a ray exhausted its own
                            span-derived step budget max(1, ceil(span/step)+1)
                            without ending; only then can the frame-wide
                            max_steps of render.py:469-473 differ from it.
                            The host variant re-renders with the exact frame
                            budget in that case; device callers must check.   */
} vx_render_out;

/* ---- device / errors ---------------------------------------------------- */
const char* vx_last_error(void);
int vx_version(void);
int vx_device_count(int* n_out);
int vx_set_device(int device);
int vx_synchronize(void);

/* ---- volume (volume.py:34-82, 122-151; grid.py:22-31) -------------------- */
/* K3: upload (nz,ny,nx) x-fastest uint8, build the zero-padded device layout,
 * the 8^3 brick-max map, and the 256-bin histogram (K1). */
int vx_volume_create_u8(const uint8_t* host, int64_t nx, int64_t ny, int64_t nz,
                        vx_volume** out);
/* K3 with the 16-bit rescale of load_raw (volume.py:148-150):
 * floor(v*255/65535 + 0.5) == (v + 128) / 257 for every v. */
int vx_volume_create_u16(const uint16_t* host, int64_t nx, int64_t ny, int64_t nz,
                         vx_volume** out);
/* same from a device buffer (e.g. a torch tensor) */
int vx_volume_create_device_u8(const uint8_t* dev, int64_t nx, int64_t ny, int64_t nz,
                               vx_volume** out);
/* load_raw (volume.py:122-151) straight to the device: the headerless
 * little-endian file is streamed through page-locked slots (file reads
 * overlapped with the uploads), 16-bit data rescaled on the device.
 * host_u8_out (nullable, nx*ny*nz bytes) also receives the 8-bit voxels
 * (the reference Volume's host bytes).  Size mismatch -> VX_EINVAL with the
 * reference's "expected N bytes ... file has M" message. */
int vx_volume_load_raw(const char* path, int64_t nx, int64_t ny, int64_t nz, int32_t bit_depth,
                       uint8_t* host_u8_out, vx_volume** out);
/* load_slice_stack (volume.py:163-188) straight to the device: n_slices 8-bit
 * PGM payloads (width*height bytes at payload_offsets[i] of paths[i], headers
 * parsed by the caller) stacked along z. */
int vx_volume_load_slices(const char* const* paths, const int64_t* payload_offsets,
                          int64_t n_slices, int64_t width, int64_t height, uint8_t* host_u8_out,
                          vx_volume** out);
int vx_volume_destroy(vx_volume* vol);
int vx_volume_dims(const vx_volume* vol, int64_t dims_out[3]);
int vx_volume_read(const vx_volume* vol, uint8_t* host_out); /* compact copy back */
int vx_volume_device_bytes(const vx_volume* vol, uint64_t* bytes_out);
/* distance cap of the volume's skip maps: level 0 = 8^3 bricks, else the 4^3
 * cell maps (grows with the volume: 32 cells up to 512^3 ... 128 at 2048^3) */
int vx_volume_skip_cap(const vx_volume* vol, int32_t level, int32_t* cap_out);

/* ---- statistics (histogram.py:59-133, metrics.py:26-33) ------------------ */
/* K1: counts of the volume's voxels (cached at creation). */
int vx_histogram(vx_volume* vol, uint64_t counts_out[256]);
/* K1 over n host bytes (uploaded) */
int vx_histogram_host(const uint8_t* host, uint64_t n, uint64_t counts_out[256]);
/* K1 over n device bytes, accumulating into dev_counts[256] (not zeroed),
 * asynchronously on `stream` (a cudaStream_t used as given: 0 is the legacy default
 * stream, so work queued by torch on its default stream is ordered before it). */
int vx_histogram_device(const uint8_t* dev, uint64_t n, uint64_t* dev_counts, void* stream);
/* K1 over the z-planes [z0, z1) of a replica, accumulated into dev_counts[256]
 * asynchronously on `stream`: the z-slab shard of the multi-GPU histogram
 * (SURVEY.md §8e); every rank counts its slab of the replica it holds. */
int vx_volume_histogram_slab(vx_volume* vol, int64_t z0, int64_t z1, uint64_t* dev_counts,
                             void* stream);
/* K2: exact Otsu threshold (320-bit cross-multiplied argmin, ties -> smallest
 * T) of histogram.py:59-101; total must be < 2^47. */
int vx_otsu(const uint64_t counts[256], int32_t* T_out);
/* K2 on device counts; writes the threshold to dev_T (int32) */
int vx_otsu_device(const uint64_t* dev_counts, int32_t* dev_T, void* stream);
/* K1+K2 in ONE launch over n device bytes: dev_counts[256] is overwritten with
 * the counts (np.bincount, histogram.py:120) and dev_T receives the exact Otsu
 * threshold (histogram.py:59-101), or -1 when n == 0 or n >= 2^47.  The last
 * block to finish runs the Otsu scan.  Asynchronous on `stream`. */
int vx_histogram_otsu_device(const uint8_t* dev, uint64_t n, uint64_t* dev_counts,
                             int32_t* dev_T, void* stream);
/* K6: image entropy of n grey pixels (metrics.py:26-33); also returns counts */
int vx_image_entropy(const uint8_t* host_pixels, int64_t n, double* H_out,
                     uint64_t counts_out[256]);
/* K6 finalisation from a device histogram (numpy pairwise summation order) */
int vx_entropy_from_counts_device(const uint64_t* dev_counts, uint64_t n, double* dev_H,
                                  void* stream);

/* ---- render (render.py:188-560) ------------------------------------------ */
/* K4: one frame; fused K6 image histogram; host outputs. */
int vx_render(vx_volume* vol, const vx_ray_setup* rs, const vx_render_params* rp,
              const vx_filter_config* fc, const vx_partition* part, vx_render_out* out);
/* K4 into device outputs, asynchronous on `stream`.  Outputs are written, not
 * accumulated, except image_hist / hit_count / samples which are atomically
 * accumulated (zero them first). */
int vx_render_device(vx_volume* vol, const vx_ray_setup* rs, const vx_render_params* rp,
                     const vx_filter_config* fc, const vx_partition* part,
                     vx_render_out* dev_out, void* stream);
/* march_ray (render.py:426-464) for n arbitrary rays: origins/dirs FP64 (n,3),
 * dirs already normalised, per-ray t spans from vx_ray_spans, max_steps per
 * ray.  Outputs hit (u8), voxel (i32 x3), t (f32), value (f64). */
int vx_march_rays(vx_volume* vol, const double* origins, const double* dirs,
                  const double* t_enter, const double* t_exit, const int32_t* max_steps,
                  int64_t n, const vx_render_params* rp, const vx_filter_config* fc,
                  uint8_t* hit_out, int32_t* voxel_out, float* t_out, double* value_out);
/* primary_ray_dirs (render.py:188-201): (H*W,3) FP64 */
int vx_ray_dirs(const vx_ray_setup* rs, double* dirs_out);
/* ray_box_spans (render.py:204-230) for n rays from one origin */
int vx_ray_spans(const double origin[3], const double* dirs, int64_t n, const int64_t dims[3],
                 double* t_enter_out, double* t_exit_out);
/* apply_filter_batch (filters.py:230-266): K5, any integer coords */
int vx_filter_batch(vx_volume* vol, const int64_t* xs, const int64_t* ys, const int64_t* zs,
                    int64_t n, const vx_filter_config* fc, double* out);
/* sobel_normal_batch (render.py:360-377): fallback (n,3) used when |g|<1e-12 */
int vx_sobel_batch(vx_volume* vol, const int64_t* xs, const int64_t* ys, const int64_t* zs,
                   int64_t n, const double* fallback, double* normals_out);
/* shade_phong_batch (render.py:385-403) */
int vx_phong_batch(const double* normals, const double* view_dirs, int64_t n,
                   const vx_render_params* rp, uint8_t* out);

/* ---- multi-GPU frame group -------------------------------
 * The multi-GPU comm init of SURVEY.md §8b's `vx_init`: sort-first rendering
 * over `world` ranks (one process or one thread per GPU, same node), the
 * reference's worker-band split (render.py:514-541, bit-identical for any
 * worker count, test_render.py:242-251) at GPU granularity.  Every rank holds
 * a full replica (vx_volume_*), renders the 8x16 tiles t with t % world ==
 * rank, and its K4 stores them straight into rank 0's frame slot over
 * NVLink (peer / CUDA-IPC pointers); the image histogram, hit count and
 * samples are added there with system-scope atomics.  No collective per
 * frame: completion and slot reuse are monotonic flags written and awaited
 * with stream memory operations (VX_GROUP_SYNC_DEVICE), or ordered by the
 * caller's host barrier (VX_GROUP_SYNC_HOST: ranks sharing one GPU).
 *
 *   vx_group_create    -> this rank's blob (VX_GROUP_BLOB_BYTES)
 *   (caller all-gathers the blobs in rank order: MPI, torch.distributed, ...)
 *   vx_group_connect   opens the peers' blocks (IPC, or peer access in-process)
 *   per frame, every rank: vx_group_render; rank 0 then consumes the frame
 *   (vx_group_download or its device pointers) and calls vx_group_release.
 */
#define VX_GROUP_BLOB_BYTES 256
enum vx_group_sync {
  VX_GROUP_SYNC_AUTO = -1,  /* device flags when every rank has its own GPU   */
  VX_GROUP_SYNC_DEVICE = 0, /* stream-memop flags, no host round trip         */
  VX_GROUP_SYNC_HOST = 1    /* caller orders frames (stream sync + barrier)   */
};
typedef struct vx_group vx_group;
typedef struct {
  uint8_t* pixels;    /* device pointer (rank 0's slot), height*width       */
  uint64_t* counters; /* device: [256] image histogram, [256] hits,
                         [257] samples, [258] truncation flag (int32)        */
  uint32_t frame;     /* 1-based frame number of this rank                   */
  uint32_t _pad;
} vx_group_frame;
int vx_group_create(int32_t rank, int32_t world, int64_t max_pixels, vx_group** out,
                    uint8_t* blob_out);
int vx_group_connect(vx_group* g, const uint8_t* blobs, int32_t sync);
int vx_group_info(const vx_group* g, int32_t* sync_out, uint32_t* frame_out);
/* VX_OK when this device supports the stream memory operations of
 * VX_GROUP_SYNC_DEVICE (all ranks should agree before connecting). */
int vx_group_probe_device_sync(void);
/* This rank's tiles of the next frame, asynchronously on `stream`.  On rank 0
 * (device sync) the stream then waits for every rank's tiles: work queued
 * behind this call sees the whole frame.  Rank 0 may hold at most two
 * unreleased frames. */
int vx_group_render(vx_group* g, vx_volume* vol, const vx_ray_setup* rs,
                    const vx_render_params* rp, const vx_filter_config* fc, void* stream,
                    vx_group_frame* out);
/* rank 0: the oldest unreleased frame is consumed: zero its counters and
 * hand its slot back to the peers (stream-ordered).  No-op on other ranks. */
int vx_group_release(vx_group* g, void* stream);
/* rank 0: copy the oldest unreleased frame to host memory and synchronise */
int vx_group_download(vx_group* g, uint8_t* host_pixels, uint64_t* host_counters,
                      int64_t n_pixels, void* stream);
int vx_group_destroy(vx_group* g);

/* ---- one process, several GPUs (SURVEY.md §8b vx_init) -------------------
 * vx_init selects the devices (device_ids[0] renders the frame's owner
 * slot).  vx_multi_volume_create_u8 builds a replica on every listed device
 * (host upload to the first, device-to-device copies to the others);
 * vx_multi_render renders one frame split over them (the frame group of
 * vx_group_*, ranks = the listed devices, peer stores into the first
 * device's frame, device flags when the devices are distinct) and returns the
 * host frame like vx_render; vx_multi_histogram sums z-slab histograms of the
 * replicas.  The same device may be listed twice (functional tests on one
 * GPU: the frames are then ordered on the host). */
typedef struct vx_multi vx_multi;
int vx_init(int n_devices, const int* device_ids);
int vx_multi_volume_create_u8(const uint8_t* host, int64_t nx, int64_t ny, int64_t nz,
                              vx_multi** out);
int vx_multi_render(vx_multi* m, const vx_ray_setup* rs, const vx_render_params* rp,
                    const vx_filter_config* fc, vx_render_out* host_out);
int vx_multi_histogram(vx_multi* m, uint64_t counts_out[256]);
int vx_multi_info(const vx_multi* m, int32_t* n_devices_out, int32_t* sync_out);
int vx_multi_destroy(vx_multi* m);

/* ---- phantom input generator (volume.py:317-368; inputs only) ------------ */
/* shape kinds: 0 sphere, 1 shell, 2 box; params per shape:
 * [kind, cx, cy, cz, intensity, radius, thickness, ex, ey, ez] as doubles.
 * spot_idx: host array of flat indices (rng.uniform_indices) */
int vx_volume_create_phantom(int64_t nx, int64_t ny, int64_t nz, const double* shapes,
                             int64_t n_shapes, double noise_sigma, uint64_t noise_seed,
                             const int64_t* spot_idx, int64_t n_spots, int32_t spot_intensity,
                             vx_volume** out);
/* same, into a compact device buffer of nx*ny*nz bytes (histogram sweeps) */
int vx_phantom_device(uint8_t* dev_out, int64_t nx, int64_t ny, int64_t nz,
                      const double* shapes, int64_t n_shapes, double noise_sigma,
                      uint64_t noise_seed, const int64_t* spot_idx, int64_t n_spots,
                      int32_t spot_intensity, void* stream);

/* C4 input generator: u16[i] = clamp(257*v8[i] + e_i, 0, 65535),
 * e_i = (splitmix64 stream(seed) draw i0+i mod 257) - 128, so load_raw's
 * 16-bit rescale (volume.py:148-150) returns v8 exactly.  Device buffers. */
int vx_u16_dither_device(const uint8_t* dev_v8, uint64_t n, uint64_t i0, uint64_t seed,
                         uint16_t* dev_out, void* stream);

/* ---- pinned host memory (frame outputs DMA'd without staging) ------------ */
int vx_host_alloc(uint64_t bytes, void** out);
int vx_host_free(void* ptr);

/* ---- diagnostics ---------------------------------------------------------- */
/* number of kernels this thread launched since the last reset */
int vx_launch_counter(uint64_t* n_out, int reset);
/* Frame timing of this thread's vx_render calls (Frame.timing,
 * render.py:550-554): when on (default off: two events cost ~10 us of
 * latency per frame), vx_last_render_ms returns the CUDA-event device time
 * of the last frame's K4 launch(es), copy-back excluded; -1 when off. */
int vx_set_frame_timing(int on);
/* K4 scheduling (process-wide; results never depend on it): tile_order 1/0
 * (-1: env VOXB200_TILE_ORDER, default on) reorders a frame's 8x16 tiles by
 * the previous frame's per-tile cost, heaviest first, for frames of at least
 * min_grid_tiles tiles (-1: 4 per SM).  Tiles that would outlast the frame's
 * ideal length (total cost / concurrent tile slots) are rendered with every
 * ray split into 2 segments on 2 lanes, twice that length into 4, when the
 * heaviest took >= split_min_us; at most grid / split_max_div extra blocks
 * (split_min_us 0: a quarter of the tiles split in 4 and a quarter in 2,
 * for tests; the entropy filter is not split by default). */
int vx_set_schedule(int32_t tile_order, int32_t min_grid_tiles, int32_t split_min_us,
                    int32_t split_max_div);
int vx_last_render_ms(float* ms_out);
/* exact-skip structures for threshold thr, copied to host (tests):
 * level 0 = Chebyshev distance in 8^3 bricks to the nearest brick whose max
 * reaches thr (dims ceil(n/8)+2 per axis, 1-brick apron, capped at 24);
 * level 1 = the same over 4^3 cells (dims ceil(n/4)+2, capped at 32);
 * level 8 + o = the orthant-o cell map: distance to the nearest cell >= thr
 * among the cells a ray moving toward -axis a for every bit a of o (else
 * +axis a) can still reach (the skip map of such rays). */
int vx_volume_distance_map(vx_volume* vol, int32_t thr, int32_t level, uint8_t* host_out,
                           int64_t dims_out[3]);

#ifdef __cplusplus
}
#endif
#endif /* VOXB200_H */
