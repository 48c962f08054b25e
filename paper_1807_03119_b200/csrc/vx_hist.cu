// K1 (256-bin voxel histogram), K2 (exact Otsu scan), K6 (image entropy).
//
// Reference: histogram.py:119-133 (np.bincount), histogram.py:59-101 (otsu),
// metrics.py:26-33 (image_entropy).

#include "vx_internal.cuh"

namespace {

#ifdef VX_HIST_TIMING
__device__ unsigned long long g_ht[16];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define VX_HT(k) do { if (threadIdx.x == 0 && gridDim.x > 1) { asm volatile("" ::: "memory"); g_ht[k] = gtimer(); } } while (0)
#else
#define VX_HT(k) do {} while (0)
#endif
#ifdef VX_HIST_TIMING
// block-level marks: [8] first block start (min), [9] last counting done
// (max), [10] last merge + global atomics done (max), [11] first block end
#define VX_HTMIN(k) do { if (threadIdx.x == 0) atomicMin(&g_ht[k], gtimer()); } while (0)
#define VX_HTMAX(k) do { if (threadIdx.x == 0) atomicMax(&g_ht[k], gtimer()); } while (0)
#else
#define VX_HTMIN(k) do {} while (0)
#define VX_HTMAX(k) do {} while (0)
#endif

#ifndef VX_HIST_THREADS
#define VX_HIST_THREADS 512
#endif
#ifndef VX_HIST_BLOCKS_PER_SM
#define VX_HIST_BLOCKS_PER_SM 4
#endif
constexpr int kHistThreads = VX_HIST_THREADS;
constexpr int kHistBlocksPerSM = VX_HIST_BLOCKS_PER_SM;
#ifndef VX_HIST_STATIC_SMALL
#define VX_HIST_STATIC_SMALL 6
#endif
#ifndef VX_HIST_STATIC_LARGE
#define VX_HIST_STATIC_LARGE 0
#endif
// the Otsu tail in a dedicated, pre-warmed extra block (hist_otsu_kernel)
#ifndef VX_HIST_WAITER
#define VX_HIST_WAITER 1
#endif

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
  // byte k isolated by one PRMT, then address = lane_base + 32*byte (one
  // IMAD): 3 instructions per byte with the atomic, where shift + mask + add
  // took 4 -- the count loop is issue-bound below ~1 GB (ncu at 512^3:
  // issue active 71 %, "not selected" the top stall)
  atomicAdd(lane_base + (__byte_perm(w, 0u, 0x4440u) << 5), 1u);
  atomicAdd(lane_base + (__byte_perm(w, 0u, 0x4441u) << 5), 1u);
  atomicAdd(lane_base + (__byte_perm(w, 0u, 0x4442u) << 5), 1u);
  atomicAdd(lane_base + (__byte_perm(w, 0u, 0x4443u) << 5), 1u);
}

// Counts this block's share of data[0, n) into the [bin][lane] shared table
// `sh` (zeroed here) and reduces it to per-bin block totals tot[256].
__device__ __forceinline__ void count_vec4(uint32_t* lane_base, const uint4& a, const uint4& b,
                                           const uint4& c, const uint4& d) {
  count_word(lane_base, a.x); count_word(lane_base, a.y);
  count_word(lane_base, a.z); count_word(lane_base, a.w);
  count_word(lane_base, b.x); count_word(lane_base, b.y);
  count_word(lane_base, b.z); count_word(lane_base, b.w);
  count_word(lane_base, c.x); count_word(lane_base, c.y);
  count_word(lane_base, c.z); count_word(lane_base, c.w);
  count_word(lane_base, d.x); count_word(lane_base, d.y);
  count_word(lane_base, d.z); count_word(lane_base, d.w);
}

// next != nullptr: after a fixed grid-stride share of static_eighths/8 of
// the data, blocks take 4*blockDim.x-vector chunks (32 KB) of the rest from
// the counter *next (zeroed before the launch).  Measured with %globaltimer
// marks: with fixed shares only, the first block finished counting at
// 18.5 us and the last at 27.1 us (512^3; 136 vs 187 us at 1024^3) -- SMs
// see unequal bandwidth -- so the kernel ended with the slowest SM's share.
// The next chunk's index is fetched while the current chunk's loads are in
// flight.  nblk: the number of counting blocks (the grid may hold one more).
__device__ __forceinline__ void hist_block_local(const uint8_t* __restrict__ data, uint64_t n,
                                                 uint32_t* sh, uint32_t* tot,
                                                 unsigned int* next, unsigned nblk,
                                                 int static_eighths) {
  __shared__ unsigned int chunk_idx[2];
  for (int i = threadIdx.x; i < 256 * 32; i += blockDim.x) sh[i] = 0u;
  if (next && threadIdx.x == 0) chunk_idx[0] = atomicAdd(next, 1u);
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
  const uint64_t nthreads = (uint64_t)nblk * blockDim.x;  // the counting blocks' threads

  // head / tail bytes
  if (tid < head) atomicAdd(lane_base + ((uint32_t)data[tid] << 5), 1u);
  if (tid < n - tail_start) atomicAdd(lane_base + ((uint32_t)data[tail_start + tid] << 5), 1u);

  // grid-stride shares over [0, nstat) -- no per-chunk barrier -- then, with
  // a chunk counter, 32 KB chunks of [nstat, nvec) to whichever block is free
  const uint64_t bd = blockDim.x, ch = 4 * bd;
  const uint64_t round = 4 * nthreads;  // whole rounds: every thread's 4 vectors in range
  const uint64_t nstat = (next ? nvec * (uint64_t)static_eighths / 8 : nvec) / round * round;
  for (uint64_t i = tid; i < nstat; i += round) {
    const uint4 a = ld_stream(vec + i), b = ld_stream(vec + i + nthreads),
                c = ld_stream(vec + i + 2 * nthreads), d = ld_stream(vec + i + 3 * nthreads);
    count_vec4(lane_base, a, b, c, d);
  }
  if (next) {
    int p = 0;
    for (;;) {
      const uint64_t c0 = nstat + (uint64_t)chunk_idx[p] * ch;
      if (c0 >= nvec) break;
      if (threadIdx.x == 0) chunk_idx[p ^ 1] = atomicAdd(next, 1u);
      const uint64_t j = c0 + threadIdx.x;
      if (c0 + ch <= nvec) {
        const uint4 a = ld_stream(vec + j), b = ld_stream(vec + j + bd),
                    c = ld_stream(vec + j + 2 * bd), d = ld_stream(vec + j + 3 * bd);
        count_vec4(lane_base, a, b, c, d);
      } else {  // the last, partial chunk
        const uint4 z = make_uint4(0u, 0u, 0u, 0u);
        uint4 v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) v[k] = j + k * bd < nvec ? ld_stream(vec + j + k * bd) : z;
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (j + k * bd < nvec) {
            count_word(lane_base, v[k].x); count_word(lane_base, v[k].y);
            count_word(lane_base, v[k].z); count_word(lane_base, v[k].w);
          }
      }
      __syncthreads();  // chunk_idx[p ^ 1] published; chunk_idx[p] free again
      p ^= 1;
    }
  } else {
  // remainder (< 4 vectors per thread): loads issued together, so a thread
  // waits on one memory round trip instead of up to four in a row
  const uint64_t i = nstat + tid;
  if (i < nvec) {
    uint4 v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint64_t j = i + k * nthreads;
      v[k] = j < nvec ? ld_stream(vec + j) : make_uint4(0u, 0u, 0u, 0u);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (i + k * nthreads < nvec) {
        count_word(lane_base, v[k].x); count_word(lane_base, v[k].y);
        count_word(lane_base, v[k].z); count_word(lane_base, v[k].w);
      }
    }
  }
  }  // static shares
  __syncthreads();
  VX_HTMAX(9);
  VX_HTMIN(11);

  // merge the 32 lane columns of each bin (rotated to stay conflict-free)
  for (int b = threadIdx.x; b < 256; b += blockDim.x) {
    uint32_t s = 0;
#pragma unroll 8
    for (int j = 0; j < 32; ++j) s += sh[b * 32 + ((j + b) & 31)];
    tot[b] = s;
  }
}

// Block-local histogram, then the block's 256 totals into out[256] (u64
// atomics; a DSMEM pre-merge across 2/4/8-block clusters measured no faster).
__device__ __forceinline__ void hist_block(const uint8_t* __restrict__ data, uint64_t n,
                                           uint32_t* sh, uint32_t* tot, unsigned long long* out,
                                           unsigned int* next = nullptr, unsigned nblk = 0,
                                           int static_eighths = 0) {
  VX_HTMIN(8);
  hist_block_local(data, n, sh, tot, next, nblk ? nblk : gridDim.x, static_eighths);
  __syncthreads();
  for (int b = threadIdx.x; b < 256; b += blockDim.x)
    if (tot[b]) atomicAdd(out + b, (unsigned long long)tot[b]);
}

__global__ void __launch_bounds__(kHistThreads)
hist256_kernel(const uint8_t* __restrict__ data, uint64_t n, unsigned long long* __restrict__ out) {
  __shared__ __align__(16) uint32_t sh[256 * 32];
  __shared__ uint32_t tot[256];
  hist_block(data, n, sh, tot, out);
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

struct OtsuSmem {
  unsigned long long sn[256], sb[256], sa[256];  // inclusive prefix sums
  unsigned long long wt[8][3];                    // warp totals
  double wmin[8];
  unsigned wmask[8];
};

__device__ __forceinline__ unsigned long long shfl_up_u64(unsigned long long v, int d) {
  return __shfl_up_sync(0xffffffffu, v, d);
}

__device__ __forceinline__ double u128_to_double(U128 x) {
  return __dadd_rn(__dmul_rn(__ull2double_rn(x.w[1]), 18446744073709551616.0),
                   __ull2double_rn(x.w[0]));
}

// Exact objective N*sigma_w^2(T) = num/den of histogram.py:92-97 from the
// prefix sums (n0, b0, a0) and the totals; an empty class contributes 0.
__device__ void otsu_exact(unsigned long long n0, unsigned long long b0, unsigned long long a0,
                           unsigned long long N, unsigned long long B, unsigned long long A,
                           U192& num, U128& den) {
  const unsigned long long n1 = N - n0, b1 = B - b0, a1 = A - a0;
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
}

// Exact Otsu of the 256 counts held by threads 0..255 (thread t holds bin t;
// `c` is ignored for t >= 256).  Every thread of the block must call it.
//
// Screen, then decide exactly.  Each T gets an FP64 estimate f_d of its exact
// objective f = num/den: x0 = a0*n0 - b0^2 and x1 are formed EXACTLY in
// 128-bit integers (no cancellation in floating point), then
// f_d = (n1*x0 + n0*x1) / (n0*n1) over positive terms only, so
// |f_d - f| <= 8 * 2^-53 * f, and f_d = 0 exactly when f = 0.  Hence the exact
// argmin T* satisfies f_d(T*) <= min_T f_d * (1 + 2^-30), and only T passing
// that screen are compared exactly (320-bit cross products, histogram.py:98),
// in increasing T with a strict compare (ties -> smallest T).  T with c[T] = 0
// (T > 0) repeat the partition of T - 1, so they can never be the smallest
// minimiser and are screened out; this keeps exact-tie plateaus of sparse
// histograms to one candidate each.  Typically one candidate survives; the
// former all-exact argmin tree took ~9 us of a single block.
// one out-of-line copy: the waiter block's warm-up pass then warms the very
// instructions its real pass executes (an inlined second copy stays cold)
#ifndef VX_OTSU_NOINLINE
#define VX_OTSU_NOINLINE 1
#endif
#if VX_OTSU_NOINLINE
__device__ __noinline__
#else
__device__
#endif
void otsu_block(unsigned long long c, OtsuSmem& S, int32_t* __restrict__ T_out) {
  const int t = threadIdx.x;
  const int lane = t & 31, w = t >> 5;
  const bool on = t < 256;
  unsigned long long n = 0, b = 0, a = 0;
  if (on) {
    // warp-inclusive scans of n, sum i*c, sum i^2*c (u64 is exact: N < 2^47)
    n = c;
    b = c * (unsigned long long)t;
    a = c * (unsigned long long)(t * t);
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const unsigned long long vn = shfl_up_u64(n, d), vb = shfl_up_u64(b, d),
                               va = shfl_up_u64(a, d);
      if (lane >= d) { n += vn; b += vb; a += va; }
    }
    if (lane == 31) { S.wt[w][0] = n; S.wt[w][1] = b; S.wt[w][2] = a; }
  }
  VX_HT(6);
  __syncthreads();
  VX_HT(0);
  unsigned long long N = 0, B = 0, A = 0;
  for (int k = 0; k < 8; ++k) {
    if (k < w) { n += S.wt[k][0]; b += S.wt[k][1]; a += S.wt[k][2]; }
    N += S.wt[k][0]; B += S.wt[k][1]; A += S.wt[k][2];
  }
  const bool valid = N != 0 && N < (1ull << 47);
  double f = __longlong_as_double(0x7ff0000000000000ll);  // +inf: not a candidate
  if (on) {
    S.sn[t] = n; S.sb[t] = b; S.sa[t] = a;
    if (valid && (t == 0 || c != 0)) {
      const unsigned long long n1 = N - n, b1 = B - b, a1 = A - a;
      if (n && n1) {
        const double x0 = u128_to_double(sub_128(mul_64_64(a, n), mul_64_64(b, b)));
        const double x1 = u128_to_double(sub_128(mul_64_64(a1, n1), mul_64_64(b1, b1)));
        const double dn0 = (double)n, dn1 = (double)n1;
        f = __ddiv_rn(__dadd_rn(__dmul_rn(dn1, x0), __dmul_rn(dn0, x1)), __dmul_rn(dn0, dn1));
      } else if (n) {
        f = __ddiv_rn(u128_to_double(sub_128(mul_64_64(a, n), mul_64_64(b, b))), (double)n);
      } else {
        f = __ddiv_rn(u128_to_double(sub_128(mul_64_64(a1, n1), mul_64_64(b1, b1))), (double)n1);
      }
    }
    double m = f;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) m = fmin(m, __shfl_xor_sync(0xffffffffu, m, d));
    if (lane == 0) S.wmin[w] = m;
  }
  __syncthreads();
  VX_HT(1);
  if (on) {
    double m = S.wmin[0];
    for (int k = 1; k < 8; ++k) m = fmin(m, S.wmin[k]);
    const double cut = __dmul_ru(m, 1.0 + 0x1p-30);
    const unsigned mask = __ballot_sync(0xffffffffu, f <= cut);
    if (lane == 0) S.wmask[w] = mask;
  }
  __syncthreads();
  VX_HT(2);
  if (t != 0) return;
  if (!valid) {
    *T_out = -1;
    return;
  }
  // a single survivor is the argmin: the exact objective is formed only
  // when a second candidate has to be compared with the best so far
  int best = -1;
  bool have = false;  // bnum / bden hold best's exact objective
  U192 bnum;
  U128 bden;
  for (int k = 0; k < 8; ++k) {
    unsigned mk = S.wmask[k];
    while (mk) {
      const int T = k * 32 + __ffs(mk) - 1;
      mk &= mk - 1;
      if (best < 0) {
        best = T;
        continue;
      }
      if (!have) {
        otsu_exact(S.sn[best], S.sb[best], S.sa[best], N, B, A, bnum, bden);
        have = true;
      }
      U192 num;
      U128 den;
      otsu_exact(S.sn[T], S.sb[T], S.sa[T], N, B, A, num, den);
      if (frac_less(num, den, bnum, bden)) {
        best = T;
        bnum = num;
        bden = den;
      }
    }
  }
  *T_out = best;
  VX_HT(3);
}

__global__ void __launch_bounds__(256) otsu_kernel(const unsigned long long* __restrict__ counts,
                                                   int32_t* __restrict__ T_out) {
  __shared__ OtsuSmem S;
  otsu_block(counts[threadIdx.x], S, T_out);
}

// K1+K2 in one launch (histogram.py:119-133 then :59-101).  Counting blocks
// add their bins into the workspace and take a ticket; one extra block runs
// the exact Otsu scan once every ticket is in (VX_HIST_WAITER, below; or,
// without it, the last block to take a ticket), copies the bins to
// counts_out and re-zeroes the workspace for the next call on this stream.
// One launch, no memset: the stand-alone K1 + K2 pair costs two launch gaps
// and a fill kernel, which is 10-20 us at 256^3-512^3.
// The blocks' bin totals land in kHistRepl copies of the 256 bins (block b
// adds into copy b % kHistRepl) to spread ~600 blocks x 256 u64 atomics over
// more L2 lines (measured: 256^3 ~1 us faster than one copy, larger sizes
// unchanged; profiles/r2/r2_ab_hist.txt).
#ifndef VX_HIST_REPL
#define VX_HIST_REPL 8
#endif
constexpr int kHistRepl = VX_HIST_REPL;
struct HistWs {
  unsigned long long bins[kHistRepl][256];
  unsigned int ticket;
  unsigned int next;  // chunk counter of the dynamic shares
};

// bin b summed over the copies (L2: written by other SMs' atomics)
__device__ __forceinline__ unsigned long long hist_ws_bin(const HistWs* ws, int b) {
  unsigned long long c = 0;
#pragma unroll
  for (int r = 0; r < kHistRepl; ++r) c += __ldcg(&ws->bins[r][b]);
  return c;
}

// zero every copy for the next launch on this stream (after the bins were read)
__device__ __forceinline__ void hist_ws_clear(HistWs* ws) {
  for (int i = threadIdx.x; i < kHistRepl * 256; i += blockDim.x) (&ws->bins[0][0])[i] = 0ull;
}

__global__ void __launch_bounds__(kHistThreads, kHistBlocksPerSM)
hist_otsu_kernel(const uint8_t* __restrict__ data, uint64_t n, HistWs* __restrict__ ws,
                 unsigned long long* __restrict__ counts_out, int32_t* __restrict__ T_out,
                 int static_eighths) {
  static_assert(sizeof(OtsuSmem) <= 256 * 32 * 4, "Otsu scratch must fit the histogram table");
  __shared__ __align__(16) uint32_t sh[256 * 32];
  __shared__ uint32_t tot[256];
  OtsuSmem& S = *reinterpret_cast<OtsuSmem*>(sh);
#if VX_HIST_WAITER
  // The Otsu tail runs in one extra block (the last index, so it takes the
  // first slot a counting block frees): it executes the whole Otsu code once
  // on a synthetic histogram -- its SM's instruction caches warm while the
  // counting finishes; executed cold by the last counting block, the scan
  // phase alone took ~3.5 us (0.26 us warm; %globaltimer marks, profiles/r2/
  // r2_ab_hist.txt) -- then waits for every counting block's ticket.  No
  // counting block waits on it, so the wait cannot deadlock.
  const unsigned nblk = gridDim.x - 1;
  if (blockIdx.x == nblk) {
    __shared__ int32_t warm_T;
    otsu_block(1ull + (threadIdx.x % 7u), S, &warm_T);
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned v;
      for (;;) {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(&ws->ticket) : "memory");
        if (v >= nblk) break;
        __nanosleep(64);
      }
    }
    __syncthreads();
#ifdef VX_HIST_PROBE  // with -DVX_HIST_TIMING (profiles/r2/r2_ab_hist.txt)
    if (VX_HIST_PROBE > 0) {  // timing probe: let in-flight bin atomics drain first
      const unsigned long long t0 = gtimer();
      while (gtimer() - t0 < (unsigned long long)VX_HIST_PROBE) {}
      __syncthreads();
    }
#endif
    VX_HT(7);
    unsigned long long c = 0;
    if (threadIdx.x < 256) c = hist_ws_bin(ws, threadIdx.x);
#ifdef VX_HIST_PROBE
    // timing probe: the mark waits for the loads
    if (c == 0x7fffffffffffffffull) asm volatile("trap;");
    __syncthreads();
#endif
    VX_HT(4);
    otsu_block(c, S, T_out);
    VX_HT(5);
    if (threadIdx.x < 256) counts_out[threadIdx.x] = c;
    hist_ws_clear(ws);
    if (threadIdx.x == 0) {
      ws->ticket = 0u;
      ws->next = 0u;
    }
    return;
  }
  hist_block(data, n, sh, tot, ws->bins[blockIdx.x % kHistRepl], &ws->next, nblk, static_eighths);
  VX_HTMAX(10);
  // the block's bin atomics precede thread 0's fence (barrier), which
  // precedes its ticket
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(&ws->ticket, 1u);
  }
#else
  __shared__ bool last;
  hist_block(data, n, sh, tot, ws->bins[blockIdx.x % kHistRepl], &ws->next, 0, static_eighths);
  VX_HTMAX(10);
  // the block's bin atomics precede thread 0's fence (barrier), which
  // precedes its ticket; one fencing thread per block, as in the CUDA
  // guide's last-block reduction.  The last block's tail (bins, scan,
  // screen, exact compare) runs cold: ~7 us (%globaltimer marks,
  // -DVX_HIST_TIMING, scripts/hist_tail_times.py).
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(&ws->ticket, 1u) == gridDim.x - 1;
    if (last) __threadfence();
  }
  __syncthreads();
  if (!last) return;
  VX_HT(7);
  unsigned long long c = 0;
  if (threadIdx.x < 256) c = hist_ws_bin(ws, threadIdx.x);
  VX_HT(4);
  otsu_block(c, S, T_out);
  VX_HT(5);
  // outputs and the workspace reset leave after the scan (off its path)
  if (threadIdx.x < 256) counts_out[threadIdx.x] = c;
  hist_ws_clear(ws);
  if (threadIdx.x == 0) {
    ws->ticket = 0u;
    ws->next = 0u;
  }
#endif
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

// 256 threads: bin b's term p*log2(p) on thread b (the FP64 log2 is the
// cost: one thread doing all 256 took ~60 us), compacted in bin order over
// the non-empty bins, then thread 0 adds them in numpy's pairwise order
// (~256 dependent FP64 adds).
__global__ void __launch_bounds__(256) entropy_kernel(const unsigned long long* __restrict__ counts,
                                                      uint64_t n, double* __restrict__ H_out) {
  __shared__ double terms[256];
  __shared__ int warp_base[9];
  const int b = threadIdx.x;
  const unsigned long long c = counts[b];
  double t = 0.0;
  if (c) {
    const double p = __ddiv_rn((double)c, (double)n);
    t = __dmul_rn(p, log2(p));
  }
  const unsigned m = __ballot_sync(0xffffffffu, c != 0);
  const int w = b >> 5, lane = b & 31;
  if (lane == 0) warp_base[w + 1] = __popc(m);
  __syncthreads();
  if (b == 0) {
    warp_base[0] = 0;
    for (int i = 1; i <= 8; ++i) warp_base[i] += warp_base[i - 1];
  }
  __syncthreads();
  if (c) terms[warp_base[w] + __popc(m & ((1u << lane) - 1u))] = t;
  __syncthreads();
  if (b == 0) *H_out = -pairwise(terms, warp_base[8]);
}

// bin 0 of a slab histogram counted over whole padded planes: minus the
// apron's zeros (vx_volume_histogram_slab)
__global__ void sub_bin0_kernel(unsigned long long* counts, unsigned long long v) {
  counts[0] -= v;
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

// one zeroed workspace per (device, stream): the kernel's Otsu block leaves
// it zeroed, and launches on one stream are ordered
static std::mutex g_ws_mu;
static struct WsSlot { int dev; cudaStream_t s; HistWs* p; } g_ws[64];
static int g_ws_n = 0;

static int hist_ws(cudaStream_t s, HistWs** out) {
  int dev = 0;
  VX_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_ws_mu);
  for (int i = 0; i < g_ws_n; ++i)
    if (g_ws[i].dev == dev && g_ws[i].s == s) {
      *out = g_ws[i].p;
      return VX_OK;
    }
  HistWs* p = nullptr;
  VX_CUDA(cudaMalloc(&p, sizeof(HistWs)));
  VX_CUDA(cudaMemset(p, 0, sizeof(HistWs)));
  const int slot = g_ws_n < 64 ? g_ws_n++ : (int)(((uintptr_t)s >> 4) % 64);
  // a recycled slot's old workspace stays allocated: a launch may still use it
  g_ws[slot] = {dev, s, p};
  *out = p;
  return VX_OK;
}

int vx_launch_hist_otsu(const uint8_t* dev, uint64_t n, uint64_t* dev_counts, int32_t* dev_T,
                        cudaStream_t s) {
  HistWs* ws = nullptr;
  int rc = hist_ws(s, &ws);
  if (rc) return rc;
  const int sms = vx_sm_count();
  uint64_t want = (n / 16 + kHistThreads - 1) / kHistThreads;
  uint64_t grid = (uint64_t)sms * kHistBlocksPerSM;
  if (want < grid) grid = want ? want : 1;
  // eighths of the data dealt as fixed grid-stride shares, the rest as 32 KB
  // chunks to whichever block is free.  All chunks from 512 MiB up (1024^3
  // 190 -> 184 us, 2048^3 1.44 -> 1.36 ms); below, a chunked tail only
  // (the per-chunk barriers cost more than the imbalance over all of it:
  // 512^3 35.3 -> 36.9 us)
  const int static_eighths = n >= (1ull << 29) ? VX_HIST_STATIC_LARGE : VX_HIST_STATIC_SMALL;
  hist_otsu_kernel<<<(unsigned)grid + VX_HIST_WAITER, kHistThreads, 0, s>>>(
      dev, n, ws, reinterpret_cast<unsigned long long*>(dev_counts), dev_T, static_eighths);
  VX_CHECK_LAUNCH();
  return VX_OK;
}

#ifdef VX_HIST_TIMING
extern "C" int vx_debug_hist_times(unsigned long long* out) {
  VX_CUDA(cudaMemcpyFromSymbol(out, g_ht, 16 * 8));
  unsigned long long init[16];
  for (int i = 0; i < 16; ++i) init[i] = (i == 8 || i == 11) ? ~0ull : 0ull;
  VX_CUDA(cudaMemcpyToSymbol(g_ht, init, 16 * 8));
  return VX_OK;
}
#endif

int vx_launch_otsu(const uint64_t* dev_counts, int32_t* dev_T, cudaStream_t s) {
  otsu_kernel<<<1, 256, 0, s>>>(reinterpret_cast<const unsigned long long*>(dev_counts), dev_T);
  VX_CHECK_LAUNCH();
  return VX_OK;
}

int vx_launch_entropy(const uint64_t* dev_counts, uint64_t n, double* dev_H, cudaStream_t s) {
  entropy_kernel<<<1, 256, 0, s>>>(reinterpret_cast<const unsigned long long*>(dev_counts), n, dev_H);
  VX_CHECK_LAUNCH();
  return VX_OK;
}

int vx_launch_sub_bin0(uint64_t* dev_counts, uint64_t v, cudaStream_t s) {
  if (!v) return VX_OK;
  sub_bin0_kernel<<<1, 1, 0, s>>>(reinterpret_cast<unsigned long long*>(dev_counts), v);
  VX_CHECK_LAUNCH();
  return VX_OK;
}
