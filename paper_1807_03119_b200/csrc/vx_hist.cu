// K1 (256-bin voxel histogram), K2 (exact Otsu scan), K6 (image entropy).
//
// Reference: histogram.py:119-133 (np.bincount), histogram.py:59-101 (otsu),
// metrics.py:26-33 (image_entropy).

#include "vx_internal.cuh"

namespace {

constexpr int kHistThreads = 512;
constexpr int kHistBlocksPerSM = 4;

__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// Per-block sub-histogram laid out [bin][lane] (32 KiB): lane l always hits
// bank l, so a warp's 32 shared atomics are conflict-free whatever the data
// (CT volumes are dominated by a background spike; a per-warp [bin] table
// would serialise on it).
__device__ __forceinline__ void count_word(uint32_t* lane_base, uint32_t w) {
  atomicAdd(lane_base + ((w & 0xffu) << 5), 1u);
  atomicAdd(lane_base + (((w >> 8) & 0xffu) << 5), 1u);
  atomicAdd(lane_base + (((w >> 16) & 0xffu) << 5), 1u);
  atomicAdd(lane_base + ((w >> 24) << 5), 1u);
}

__global__ void __launch_bounds__(kHistThreads)
hist256_kernel(const uint8_t* __restrict__ data, uint64_t n, unsigned long long* __restrict__ out) {
  __shared__ uint32_t sh[256 * 32];
  for (int i = threadIdx.x; i < 256 * 32; i += blockDim.x) sh[i] = 0u;
  __syncthreads();

  const uint32_t lane = threadIdx.x & 31u;
  uint32_t* lane_base = sh + lane;

  const uintptr_t addr = reinterpret_cast<uintptr_t>(data);
  uint64_t head = (16u - (addr & 15u)) & 15u;
  if (head > n) head = n;
  const uint64_t nvec = (n - head) >> 4;
  const uint64_t tail_start = head + (nvec << 4);
  const uint4* vec = reinterpret_cast<const uint4*>(data + head);

  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t nthreads = (uint64_t)gridDim.x * blockDim.x;

  // head / tail bytes
  if (tid < head) atomicAdd(lane_base + ((uint32_t)data[tid] << 5), 1u);
  if (tid < n - tail_start) atomicAdd(lane_base + ((uint32_t)data[tail_start + tid] << 5), 1u);

  // body: 4 x 16 B in flight per thread
  uint64_t i = tid;
  for (; i + 3 * nthreads < nvec; i += 4 * nthreads) {
    uint4 a = ld_stream(vec + i);
    uint4 b = ld_stream(vec + i + nthreads);
    uint4 c = ld_stream(vec + i + 2 * nthreads);
    uint4 d = ld_stream(vec + i + 3 * nthreads);
    count_word(lane_base, a.x); count_word(lane_base, a.y);
    count_word(lane_base, a.z); count_word(lane_base, a.w);
    count_word(lane_base, b.x); count_word(lane_base, b.y);
    count_word(lane_base, b.z); count_word(lane_base, b.w);
    count_word(lane_base, c.x); count_word(lane_base, c.y);
    count_word(lane_base, c.z); count_word(lane_base, c.w);
    count_word(lane_base, d.x); count_word(lane_base, d.y);
    count_word(lane_base, d.z); count_word(lane_base, d.w);
  }
  for (; i < nvec; i += nthreads) {
    uint4 a = ld_stream(vec + i);
    count_word(lane_base, a.x); count_word(lane_base, a.y);
    count_word(lane_base, a.z); count_word(lane_base, a.w);
  }
  __syncthreads();

  // merge the 32 lane columns of each bin (rotated to stay conflict-free)
  for (int b = threadIdx.x; b < 256; b += blockDim.x) {
    uint32_t s = 0;
#pragma unroll 8
    for (int j = 0; j < 32; ++j) s += sh[b * 32 + ((j + b) & 31)];
    if (s) atomicAdd(out + b, (unsigned long long)s);
  }
}

// ---------------------------------------------------------------------------
// K2: exact Otsu.  For each T the objective N*sigma_w^2(T) is kept as the
// exact fraction num/den of histogram.py:92-97 and candidates are compared by
// cross-multiplication (histogram.py:98); ties resolve to the smallest T.
// With N < 2^47 voxels: a <= 65025*N < 2^63, num < 2^158 (3 limbs),
// den < 2^94 (2 limbs), products < 2^252.

struct U192 { unsigned long long w[3]; };
struct U128 { unsigned long long w[2]; };

__device__ __forceinline__ void mul64(unsigned long long a, unsigned long long b,
                                      unsigned long long& lo, unsigned long long& hi) {
  lo = a * b;
  hi = __umul64hi(a, b);
}

__device__ U128 mul_64_64(unsigned long long a, unsigned long long b) {
  U128 r;
  mul64(a, b, r.w[0], r.w[1]);
  return r;
}

__device__ U128 sub_128(U128 a, U128 b) {  // a >= b
  U128 r;
  r.w[0] = a.w[0] - b.w[0];
  unsigned long long borrow = a.w[0] < b.w[0] ? 1ull : 0ull;
  r.w[1] = a.w[1] - b.w[1] - borrow;
  return r;
}

__device__ U192 mul_128_64(U128 a, unsigned long long b) {
  U192 r;
  unsigned long long lo0, hi0, lo1, hi1;
  mul64(a.w[0], b, lo0, hi0);
  mul64(a.w[1], b, lo1, hi1);
  r.w[0] = lo0;
  r.w[1] = lo1 + hi0;
  unsigned long long c = r.w[1] < lo1 ? 1ull : 0ull;
  r.w[2] = hi1 + c;
  return r;
}

__device__ U192 add_192(U192 a, U192 b) {
  U192 r;
  unsigned long long c = 0;
  for (int i = 0; i < 3; ++i) {
    unsigned long long s = a.w[i] + b.w[i];
    unsigned long long c1 = s < a.w[i] ? 1ull : 0ull;
    unsigned long long s2 = s + c;
    unsigned long long c2 = s2 < s ? 1ull : 0ull;
    r.w[i] = s2;
    c = c1 | c2;
  }
  return r;
}

// 192 x 128 -> 320-bit product (5 limbs), schoolbook
__device__ void mul_192_128(const U192& a, const U128& b, unsigned long long r[5]) {
  for (int i = 0; i < 5; ++i) r[i] = 0;
  for (int i = 0; i < 3; ++i) {
    unsigned long long carry = 0;
    for (int j = 0; j < 2; ++j) {
      unsigned long long lo, hi;
      mul64(a.w[i], b.w[j], lo, hi);
      unsigned long long s = r[i + j] + lo;
      unsigned long long c1 = s < lo ? 1ull : 0ull;
      unsigned long long s2 = s + carry;
      unsigned long long c2 = s2 < s ? 1ull : 0ull;
      r[i + j] = s2;
      carry = hi + c1 + c2;
    }
    int k = i + 2;
    while (carry && k < 5) {
      unsigned long long s = r[k] + carry;
      carry = s < carry ? 1ull : 0ull;
      r[k] = s;
      ++k;
    }
  }
}

// true iff numA/denA < numB/denB  (numA*denB < numB*denA)
__device__ bool frac_less(const U192& numA, const U128& denA, const U192& numB, const U128& denB) {
  unsigned long long l[5], r[5];
  mul_192_128(numA, denB, l);
  mul_192_128(numB, denA, r);
  for (int i = 4; i >= 0; --i) {
    if (l[i] != r[i]) return l[i] < r[i];
  }
  return false;
}

__global__ void __launch_bounds__(256) otsu_kernel(const unsigned long long* __restrict__ counts,
                                                   int32_t* __restrict__ T_out) {
  __shared__ unsigned long long sn[256], sb[256], sa[256];
  __shared__ U192 snum[256];
  __shared__ U128 sden[256];
  __shared__ int st[256];
  const int t = threadIdx.x;
  const unsigned long long c = counts[t];
  sn[t] = c;
  sb[t] = c * (unsigned long long)t;
  sa[t] = c * (unsigned long long)(t * t);
  __syncthreads();
  // inclusive Hillis-Steele scans (u64 is exact: N < 2^47)
  for (int off = 1; off < 256; off <<= 1) {
    unsigned long long vn = 0, vb = 0, va = 0;
    if (t >= off) { vn = sn[t - off]; vb = sb[t - off]; va = sa[t - off]; }
    __syncthreads();
    sn[t] += vn; sb[t] += vb; sa[t] += va;
    __syncthreads();
  }
  const unsigned long long N = sn[255], B = sb[255], A = sa[255];
  const unsigned long long n0 = sn[t], b0 = sb[t], a0 = sa[t];
  const unsigned long long n1 = N - n0, b1 = B - b0, a1 = A - a0;
  U192 num;
  U128 den;
  if (n0 && n1) {
    U128 x0 = sub_128(mul_64_64(a0, n0), mul_64_64(b0, b0));
    U128 x1 = sub_128(mul_64_64(a1, n1), mul_64_64(b1, b1));
    num = add_192(mul_128_64(x0, n1), mul_128_64(x1, n0));
    den = mul_64_64(n0, n1);
  } else if (n0) {
    U128 x0 = sub_128(mul_64_64(a0, n0), mul_64_64(b0, b0));
    num.w[0] = x0.w[0]; num.w[1] = x0.w[1]; num.w[2] = 0;
    den.w[0] = n0; den.w[1] = 0;
  } else {
    U128 x1 = sub_128(mul_64_64(a1, n1), mul_64_64(b1, b1));
    num.w[0] = x1.w[0]; num.w[1] = x1.w[1]; num.w[2] = 0;
    den.w[0] = n1; den.w[1] = 0;
  }
  snum[t] = num;
  sden[t] = den;
  st[t] = t;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (t < s) {
      const int o = t + s;
      bool take = frac_less(snum[o], sden[o], snum[t], sden[t]);
      if (!take && !frac_less(snum[t], sden[t], snum[o], sden[o]) && st[o] < st[t]) take = true;
      if (take) { snum[t] = snum[o]; sden[t] = sden[o]; st[t] = st[o]; }
    }
    __syncthreads();
  }
  if (t == 0) *T_out = (N == 0 || N >= (1ull << 47)) ? -1 : st[0];
}

// ---------------------------------------------------------------------------
// K6 finalisation: H = -sum(p * log2 p) over non-empty bins, p = c / n, in
// numpy's pairwise summation order (numpy/_core/src/umath/loops_utils.h
// pairwise_sum: <8 sequential from 0, <=128 eight accumulators, else split).
__device__ double pw_block(const double* a, int n) {
  if (n < 8) {
    double r = 0.0;
    for (int i = 0; i < n; ++i) r = __dadd_rn(r, a[i]);
    return r;
  }
  double r[8];
  for (int j = 0; j < 8; ++j) r[j] = a[j];
  int i = 8;
  for (; i < n - (n % 8); i += 8)
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], a[i + j]);
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < n; ++i) res = __dadd_rn(res, a[i]);
  return res;
}

__device__ double pw_level(const double* a, int n) {  // n <= 256
  if (n <= 128) return pw_block(a, n);
  int n2 = n / 2;
  n2 -= n2 % 8;
  return __dadd_rn(pw_block(a, n2), pw_block(a + n2, n - n2));
}

// n <= 256 (non-empty bins): at most two split levels
__device__ double pairwise(const double* a, int n) {
  if (n <= 128) return pw_block(a, n);
  int n2 = n / 2;
  n2 -= n2 % 8;
  return __dadd_rn(pw_level(a, n2), pw_level(a + n2, n - n2));
}

__global__ void entropy_kernel(const unsigned long long* __restrict__ counts, uint64_t n,
                               double* __restrict__ H_out) {
  __shared__ double terms[256];
  if (threadIdx.x != 0) return;
  int k = 0;
  const double dn = (double)n;
  for (int b = 0; b < 256; ++b) {
    unsigned long long c = counts[b];
    if (c) {
      double p = __ddiv_rn((double)c, dn);
      terms[k++] = __dmul_rn(p, log2(p));
    }
  }
  double s = pairwise(terms, k);
  *H_out = -s;
}

}  // namespace

int vx_launch_hist(const uint8_t* dev, uint64_t n, uint64_t* dev_counts, cudaStream_t s) {
  if (n == 0) return VX_OK;
  int sms = vx_sm_count();
  uint64_t want = (n / 16 + kHistThreads - 1) / kHistThreads;
  uint64_t grid = (uint64_t)sms * kHistBlocksPerSM;
  if (want < grid) grid = want ? want : 1;
  hist256_kernel<<<(unsigned)grid, kHistThreads, 0, s>>>(dev, n,
                                                        reinterpret_cast<unsigned long long*>(dev_counts));
  VX_CHECK_LAUNCH();
  return VX_OK;
}

int vx_launch_otsu(const uint64_t* dev_counts, int32_t* dev_T, cudaStream_t s) {
  otsu_kernel<<<1, 256, 0, s>>>(reinterpret_cast<const unsigned long long*>(dev_counts), dev_T);
  VX_CHECK_LAUNCH();
  return VX_OK;
}

int vx_launch_entropy(const uint64_t* dev_counts, uint64_t n, double* dev_H, cudaStream_t s) {
  entropy_kernel<<<1, 32, 0, s>>>(reinterpret_cast<const unsigned long long*>(dev_counts), n, dev_H);
  VX_CHECK_LAUNCH();
  return VX_OK;
}
