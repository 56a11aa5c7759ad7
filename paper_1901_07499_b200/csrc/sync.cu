// PN packet detection on the device: normalised sliding correlation of every
// antenna stream against the bipolar PN preamble + per-row argmax.
//
// Restates sync.detect_packet (sync.py:26-44) over kernels.corr_metrics
// (kernels/numba_backend.py:55-87, numpy_backend.py:48-70):
//   metric[w] = |sum_i c[i] * conj(s[w+i])| / (|c| * sqrt(sum_i |s[w+i]|^2)),
//   0 where the denominator is <= 1e-30; peak = first argmax per antenna.
//
// Two kernels:
//  * corr_kernel — fp32 metric for every window.  A CTA stages one tile of the
//    stream (TW + P - 1 samples) and the chips (as (c, c) pairs, the packed
//    broadcast operand of FFMA2) in shared memory; each thread owns K
//    consecutive windows and slides a K-register sample window along the
//    chips, so one LDS.64 feeds K packed complex MACs (K odd: the stride-K
//    LDS.64 of a warp is bank-conflict free).  Window energy is summed
//    directly for the thread's first window and slid K-1 times.  Per-row
//    (metric, first index) maximum by 64-bit atomicMax on an ordered key.
//  * refine_kernel — recomputes in fp64, from the samples, every window whose
//    fp32 metric lies within the fp32 error bound (2 * 3 P 2^-24) of the row's
//    fp32 maximum and takes the fp64 argmax with first-index tie break, so the
//    peak index / metric are the reference's up to cf32 input quantisation.
#include <cstdint>

#include "ofdmrx_fft.cuh"
#include "ofdmrx_internal.h"

namespace ofdmrx {

namespace {

constexpr int SYNC_THREADS = 128;
constexpr int SYNC_K = 15;  // windows per thread (odd)
constexpr int SYNC_TW = SYNC_THREADS * SYNC_K;
constexpr int REFINE_THREADS = 256;

__device__ __forceinline__ unsigned long long peak_key(float m, long long w) {
  return ((unsigned long long)__float_as_uint(m) << 32) | (unsigned long long)(0xffffffffu - (uint32_t)w);
}

__device__ __forceinline__ const float2* row_ptr(const SyncParams& p, long long row) {
  const long long f = row / p.n_ant, n = row - f * p.n_ant;
  return p.rx + f * p.frame_stride + n * p.row_stride;
}

__global__ void __launch_bounds__(SYNC_THREADS) corr_kernel(const SyncParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int K = SYNC_K;
  const int P = p.n_chips;
  float2* cs = reinterpret_cast<float2*>(smem_raw);  // [P] (c, c)
  float2* xs = cs + P;                               // [TW + P - 1 + K] samples of this tile
  __shared__ double cn_part[SYNC_THREADS / 32];
  const long long row = blockIdx.x;
  const long long w0 = (long long)blockIdx.y * SYNC_TW;
  const float2* src = row_ptr(p, row);
  const int t = threadIdx.x;

  double c2 = 0.0;
  for (int i = t; i < P; i += SYNC_THREADS) {
    const float c = p.chips[i];
    cs[i] = make_float2(c, c);
    c2 += (double)c * (double)c;
  }
  const int nx = SYNC_TW + P - 1 + K;
  for (int i = t; i < nx; i += SYNC_THREADS) {
    const long long g = w0 + i;
    xs[i] = g < p.n_samples ? __ldg(src + g) : make_float2(0.0f, 0.0f);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c2 += __shfl_xor_sync(0xffffffffu, c2, o);
  if ((t & 31) == 0) cn_part[t >> 5] = c2;
  __syncthreads();
  double cn2 = 0.0;
#pragma unroll
  for (int i = 0; i < SYNC_THREADS / 32; ++i) cn2 += cn_part[i];
  const float cn = (float)sqrt(cn2);

  const int base = t * K;
  c2_t acc[K], x[K];
#pragma unroll
  for (int k = 0; k < K; ++k) acc[k] = 0ull;
#pragma unroll
  for (int k = 0; k < K - 1; ++k) x[k] = pk(xs[base + k]);
  c2_t e2 = 0ull;  // (sum re^2, sum im^2) of window 0
  int i = 0;
  for (; i + K <= P; i += K) {
#pragma unroll
    for (int j = 0; j < K; ++j) {
      // register slot of sample base + m is m % K (i is a multiple of K)
      x[(j + K - 1) % K] = pk(xs[base + i + j + K - 1]);
      const c2_t c = pk(cs[i + j]);
      e2 = fma2(x[j], x[j], e2);
#pragma unroll
      for (int k = 0; k < K; ++k) acc[k] = fma2(c, x[(j + k) % K], acc[k]);
    }
  }
  for (; i < P; ++i) {  // P % K tail straight from shared memory
    const c2_t c = pk(cs[i]);
    const c2_t s0 = pk(xs[base + i]);
    e2 = fma2(s0, s0, e2);
#pragma unroll
    for (int k = 0; k < K; ++k) acc[k] = fma2(c, pk(xs[base + i + k]), acc[k]);
  }

  // sum c * s == sum c * conj(s) up to the sign of the imaginary part: |.| is the same
  float best = -1.0f;
  long long best_w = 0;
  float m[K];
  {
    const float2 ev = upk(e2);
    float e = ev.x + ev.y;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      if (k > 0) {  // slide the energy window by one sample
        const float2 h = xs[base + k - 1], tl = xs[base + k - 1 + P];
        e = fmaxf(e + (tl.x * tl.x + tl.y * tl.y) - (h.x * h.x + h.y * h.y), 0.0f);
      }
      const float2 a = upk(acc[k]);
      const float den = cn * sqrtf(e);
      m[k] = den > 1e-30f ? sqrtf(a.x * a.x + a.y * a.y) / den : 0.0f;
      const long long w = w0 + base + k;
      if (w < p.wins && m[k] > best) {  // NaN never wins
        best = m[k];
        best_w = w;
      }
    }
  }
  __syncthreads();  // xs free: stage the metrics for a coalesced store
  float* ms = reinterpret_cast<float*>(xs);
#pragma unroll
  for (int k = 0; k < K; ++k) ms[base + k] = m[k];
  if (p.keys != nullptr) {
    unsigned long long key = best >= 0.0f ? peak_key(best, best_w) : 0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long ok = __shfl_xor_sync(0xffffffffu, key, o);
      key = ok > key ? ok : key;
    }
    if ((t & 31) == 0 && key != 0ull) atomicMax(p.keys + row, key);
  }
  __syncthreads();
  float* dst = p.metrics + row * p.wins + w0;
  const long long nw = p.wins - w0 < SYNC_TW ? p.wins - w0 : SYNC_TW;
  for (int w = t; w < nw; w += SYNC_THREADS) dst[w] = ms[w];
}

__global__ void __launch_bounds__(REFINE_THREADS) refine_kernel(const SyncParams p, int32_t* peak_idx,
                                                                 double* peak_metric) {
  const long long row = blockIdx.x;
  const int t = threadIdx.x;
  const unsigned long long key = p.keys[row];
  __shared__ double sb[REFINE_THREADS / 32];
  __shared__ long long sw[REFINE_THREADS / 32];
  double best = -1.0;
  long long best_w = 0;
  if (key != 0ull) {
    const float m32 = __uint_as_float((uint32_t)(key >> 32));
    const float delta = 3.0f * (float)p.n_chips * 5.9604645e-8f + 1e-6f;  // fp32 metric error bound
    const float thr = m32 - 2.0f * delta;
    const float2* src = row_ptr(p, row);
    const float* mrow = p.metrics + row * p.wins;
    double cn2 = 0.0;
    for (int i = 0; i < p.n_chips; ++i) cn2 += (double)p.chips[i] * (double)p.chips[i];
    const double cn = sqrt(cn2);
    for (long long w = t; w < p.wins; w += REFINE_THREADS) {
      if (!(mrow[w] >= thr)) continue;
      double cr = 0.0, ci = 0.0, e = 0.0;
      for (int i = 0; i < p.n_chips; ++i) {
        const float2 s = __ldg(src + w + i);
        const double c = p.chips[i];
        cr = fma(c, (double)s.x, cr);
        ci = fma(-c, (double)s.y, ci);
        e = fma((double)s.x, (double)s.x, fma((double)s.y, (double)s.y, e));
      }
      const double den = cn * sqrt(e);
      const double mv = den > 1e-30 ? sqrt(cr * cr + ci * ci) / den : 0.0;
      if (mv > best || (mv == best && w < best_w)) {
        best = mv;
        best_w = w;
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, o);
    const long long ow = __shfl_xor_sync(0xffffffffu, best_w, o);
    if (ob > best || (ob == best && ow < best_w)) {
      best = ob;
      best_w = ow;
    }
  }
  if ((t & 31) == 0) {
    sb[t >> 5] = best;
    sw[t >> 5] = best_w;
  }
  __syncthreads();
  if (t == 0) {
    for (int i = 1; i < REFINE_THREADS / 32; ++i)
      if (sb[i] > best || (sb[i] == best && sw[i] < best_w)) {
        best = sb[i];
        best_w = sw[i];
      }
    // no finite metric at all (all windows NaN): report window 0, metric 0
    peak_idx[row] = best >= 0.0 ? (int32_t)best_w : 0;
    peak_metric[row] = best >= 0.0 ? best : 0.0;
  }
}

}  // namespace

size_t sync_smem_bytes(int n_chips) { return (size_t)(2 * n_chips - 1 + SYNC_TW + SYNC_K) * sizeof(float2); }

cudaError_t launch_corr(const SyncParams& p, cudaStream_t s) {
  if ((long long)p.n_frames * p.n_ant == 0 || p.wins <= 0) return cudaSuccess;
  const size_t smem = sync_smem_bytes(p.n_chips);
  static bool attr_set = false;
  if (!attr_set) {
    // enough for the largest PN the ABI accepts (8192 chips)
    cudaError_t e = cudaFuncSetAttribute(corr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)sync_smem_bytes(8192));
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  if (p.keys != nullptr) {
    cudaError_t e = cudaMemsetAsync(p.keys, 0, (size_t)p.n_frames * p.n_ant * sizeof(unsigned long long), s);
    if (e != cudaSuccess) return e;
  }
  const dim3 grid((unsigned)((long long)p.n_frames * p.n_ant), (unsigned)((p.wins + SYNC_TW - 1) / SYNC_TW));
  corr_kernel<<<grid, SYNC_THREADS, smem, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_refine(const SyncParams& p, int32_t* peak_idx, double* peak_metric, cudaStream_t s) {
  const long long rows = (long long)p.n_frames * p.n_ant;
  if (rows == 0) return cudaSuccess;
  refine_kernel<<<(unsigned)rows, REFINE_THREADS, 0, s>>>(p, peak_idx, peak_metric);
  return cudaGetLastError();
}

}  // namespace ofdmrx
