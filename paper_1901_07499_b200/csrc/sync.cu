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
  extern __shared__ __align__(128) unsigned char smem_raw[];
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
                                                                 double* peak_metric, int bound_mode) {
  const long long row = blockIdx.x;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const unsigned long long key = p.keys[row];
  __shared__ double sb[REFINE_THREADS / 32];
  __shared__ long long sw[REFINE_THREADS / 32];
  double best = -1.0;
  long long best_w = 0;
  if (key != 0ull) {
    const float m32 = __uint_as_float((uint32_t)(key >> 32));
    const float delta = 3.0f * (float)p.n_chips * 5.9604645e-8f + 1e-6f;  // fp32 metric error bound
    // bound_mode: metrics hold upper bounds and the key the max lower bound
    const float thr = bound_mode ? m32 : m32 - 2.0f * delta;
    const float2* src = row_ptr(p, row);
    const float* mrow = p.metrics + row * p.wins;
    double cn2 = 0.0;
    for (int i = lane; i < p.n_chips; i += 32) cn2 += (double)p.chips[i] * (double)p.chips[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cn2 += __shfl_xor_sync(0xffffffffu, cn2, o);
    const double cn = sqrt(cn2);
    // each warp screens 32 windows per step; candidates are re-scored by the
    // whole warp (chips split over lanes, shuffle-reduced)
    // screen 4 steps (1024 windows per CTA) per iteration: independent loads in flight
    for (long long w00 = (long long)warp * 32; w00 < p.wins; w00 += 4LL * REFINE_THREADS) {
      float mv4[4];
#pragma unroll
      for (int u4 = 0; u4 < 4; ++u4) {
        const long long wl = w00 + (long long)u4 * REFINE_THREADS + lane;
        mv4[u4] = wl < p.wins ? mrow[wl] : -1.0f;
      }
#pragma unroll 1
      for (int u4 = 0; u4 < 4; ++u4) {
      const long long w0 = w00 + (long long)u4 * REFINE_THREADS;
      const bool cand = mv4[u4] >= thr;
      unsigned mask = __ballot_sync(0xffffffffu, cand);
      while (mask) {
        const int j = __ffs(mask) - 1;
        mask &= mask - 1;
        const long long w = w0 + j;
        double cr = 0.0, ci = 0.0, e = 0.0;
        for (int i = lane; i < p.n_chips; i += 32) {
          const float2 sv = __ldg(src + w + i);
          const double c = p.chips[i];
          cr = fma(c, (double)sv.x, cr);
          ci = fma(-c, (double)sv.y, ci);
          e = fma((double)sv.x, (double)sv.x, fma((double)sv.y, (double)sv.y, e));
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          cr += __shfl_xor_sync(0xffffffffu, cr, o);
          ci += __shfl_xor_sync(0xffffffffu, ci, o);
          e += __shfl_xor_sync(0xffffffffu, e, o);
        }
        const double den = cn * sqrt(e);
        const double mv = den > 1e-30 ? sqrt(cr * cr + ci * ci) / den : 0.0;
        if (mv > best || (mv == best && w < best_w)) {  // warp-uniform
          best = mv;
          best_w = w;
        }
      }
      }
    }
  }
  if (lane == 0) {
    sb[warp] = best;
    sw[warp] = best_w;
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

// ---------------------------------------------------------------------------
// Overlap-save FFT correlation (64 <= P <= 960): block b of a row covers
// samples [b*L, b*L + 1024), L = 1024 - P + 1 windows.  R = IFFT(FFT(s) .
// conj(FFT(c))) gives corr[n] for n < L without wrap-around; the receive
// path's 1024-point FFT does both transforms (IFFT = conj(FFT(conj(.)))).
// ~96 FP32 lane-ops per window instead of 2P = 510 for the direct form.
// Window energies come from an fp32 prefix sum over the block.  Each window
// carries an error bound delta_w (FFT error ~ u log2(N) |s_block| |c|, prefix
// cancellation ~ u E_block): detect writes m + delta_w to the scratch metrics
// and keys the row on max(m - delta_w), so refine_kernel re-scores exactly
// the windows that can still be the maximum.
// ---------------------------------------------------------------------------
constexpr int CF_N = 1024;
constexpr int CF_LANES = 8;  // 32-thread FFT lanes per CTA

__device__ __forceinline__ float cf_delta(float eblock, float e) {
  if (eblock <= 0.0f) return 0.0f;  // all-zero block: exact zeros
  const float ratio = eblock / fmaxf(e, 1e-30f * eblock + 1e-37f);
  // measured normwise error of the two fp32 1024-point FFTs ~2e-5 (x5 margin)
  return 1e-4f * sqrtf(ratio) + 2e-7f * ratio + 1e-5f;
}

__global__ void __launch_bounds__(32) chip_spectrum_kernel(const float* chips, int n_chips, float2* cspec) {
  using PI = PlanInfo<CF_N>;
  __shared__ __align__(16) float2 slot[PI::SLOT];
  const int t = threadIdx.x;
  float2 v[PI::P];
  fft_forward<CF_N>(v, slot, t, [&](int i) { return make_float2(i < n_chips ? chips[i] : 0.0f, 0.0f); },
                    [] { __syncwarp(); });
#pragma unroll
  for (int i = 0; i < PI::P; ++i) cspec[reg_bin<CF_N>(i, t)] = v[i];
}

#ifndef OFDMRX_CF_MINB
#define OFDMRX_CF_MINB 2  // 16 warps/SM at 128 registers (some spill) beat 8 warps at 253 (A/B: 12.9 vs 14.6 us/frame)
#endif
__global__ void __launch_bounds__(32 * CF_LANES, OFDMRX_CF_MINB) corr_fft_kernel(const SyncParams p, const float2* __restrict__ cspec,
                                                                    long long blocks_per_row, int bound_mode) {
  using PI = PlanInfo<CF_N>;
  constexpr int P = PI::P;  // 32 points per thread, 32-thread lane
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int lane = threadIdx.x >> 5, t = threadIdx.x & 31;
  float2* slot = reinterpret_cast<float2*>(smem_raw) + (size_t)lane * PI::SLOT;
  float* epre = reinterpret_cast<float*>(reinterpret_cast<float2*>(smem_raw) + (size_t)CF_LANES * PI::SLOT) +
                (size_t)lane * (CF_N + 4);
  auto lsync = [] { __syncwarp(); };
  // chip spectrum staged once per CTA (LDS in the product, not hoisted LDGs)
  float2* cs = reinterpret_cast<float2*>(epre + (size_t)(CF_LANES - lane) * (CF_N + 4));
  for (int i = threadIdx.x; i < CF_N; i += blockDim.x) cs[i] = __ldg(cspec + i);
  __syncthreads();
  const int Pc = p.n_chips;
  const int L = CF_N - Pc + 1;
  const long long total = (long long)p.n_frames * p.n_ant * blocks_per_row;
  float cn2 = 0.0f;
  for (int i = t; i < Pc; i += 32) cn2 = fmaf(p.chips[i], p.chips[i], cn2);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cn2 += __shfl_xor_sync(0xffffffffu, cn2, o);
  const float cn = sqrtf(cn2);
  unsigned long long key = 0ull;
  long long key_row = -1;
  for (long long blk = (long long)blockIdx.x * CF_LANES + lane; blk < total; blk += (long long)gridDim.x * CF_LANES) {
    const long long row = blk / blocks_per_row;
    const long long base = (blk - row * blocks_per_row) * L;
    if (row != key_row) {  // flush the key of the previous row
      if (key_row >= 0 && p.keys != nullptr) {
        unsigned long long k2 = key;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const unsigned long long ok = __shfl_xor_sync(0xffffffffu, k2, o);
          k2 = ok > k2 ? ok : k2;
        }
        if (t == 0 && k2 != 0ull) atomicMax(p.keys + key_row, k2);
      }
      key = 0ull;
      key_row = row;
    }
    const float2* src = row_ptr(p, row);
    // the thread's samples x[t + 32q] (exactly its pass-0 FFT inputs): all
    // loads in flight at once, then fp32 prefix energies by warp scans
    float2 xs[CF_N / 32];
#pragma unroll
    for (int q = 0; q < CF_N / 32; ++q) {
      const long long g = base + t + 32 * q;
      xs[q] = g < p.n_samples ? __ldg(src + g) : make_float2(0.0f, 0.0f);
    }
    float run = 0.0f;
#pragma unroll
    for (int q = 0; q < CF_N / 32; ++q) {
      float e = fmaf(xs[q].x, xs[q].x, xs[q].y * xs[q].y);
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const float y = __shfl_up_sync(0xffffffffu, e, o);
        if (t >= o) e += y;
      }
      epre[1 + t + 32 * q] = run + e;
      run += __shfl_sync(0xffffffffu, e, 31);
    }
    if (t == 0) epre[0] = 0.0f;
    float2 v[P];
    fft_forward<CF_N>(v, slot, t, [&](int idx) { return xs[(idx - t) >> 5]; }, lsync);
    lsync();  // last pass read the slot: free for the product
#pragma unroll
    for (int i = 0; i < P; ++i) {
      const int k = reg_bin<CF_N>(i, t);
      const float2 c = cs[k];
      // conj(S conj(C)) = conj(S) C, the input of IFFT = conj(FFT(conj(.)))
      const float2 sv = v[i];
      slot[k] = make_float2(fmaf(sv.x, c.x, sv.y * c.y), fmaf(sv.x, c.y, -sv.y * c.x));
    }
    lsync();
    fft_forward<CF_N>(v, slot, t, [&](int idx) { return slot[idx]; }, lsync);
    const float eblock = epre[CF_N];
    const float inv = 1.0f / ((float)CF_N * cn);
#pragma unroll
    for (int i = 0; i < P; ++i) {
      const int n = reg_bin<CF_N>(i, t);
      const long long w = base + n;
      if (n < L && w < p.wins) {
        const float e = fmaxf(epre[n + Pc] - epre[n], 0.0f);
        const float den = sqrtf(e);
        const float m = den * cn > 1e-30f ? sqrtf(fmaf(v[i].x, v[i].x, v[i].y * v[i].y)) * inv / den : 0.0f;
        float out = m;
        float lo = m;
        if (bound_mode) {
          const float dw = cf_delta(eblock, e);
          out = m + dw;
          lo = fmaxf(m - dw, 0.0f);
        }
        p.metrics[row * p.wins + w] = out;
        if (lo == lo) {  // NaN never wins
          const unsigned long long k2 = peak_key(lo, w);
          key = k2 > key ? k2 : key;
        }
      }
    }
    lsync();  // slot / epre reuse by the next block
  }
  if (key_row >= 0 && p.keys != nullptr) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long ok = __shfl_xor_sync(0xffffffffu, key, o);
      key = ok > key ? ok : key;
    }
    if (t == 0 && key != 0ull) atomicMax(p.keys + key_row, key);
  }
}

}  // namespace

bool sync_use_fft(int n_chips) { return n_chips >= 64 && n_chips <= CF_N - 64; }

size_t sync_fft_scratch_bytes() { return (size_t)CF_N * sizeof(float2); }

cudaError_t launch_corr_fft(const SyncParams& p, float2* cspec, int bound_mode, cudaStream_t s) {
  if ((long long)p.n_frames * p.n_ant == 0 || p.wins <= 0) return cudaSuccess;
  using PI = PlanInfo<CF_N>;
  const size_t smem = (size_t)CF_LANES * (PI::SLOT * sizeof(float2) + (CF_N + 4) * sizeof(float)) +
                      CF_N * sizeof(float2);
  static unsigned attr_done = 0;
  if (cudaError_t e = ensure_smem_attr(corr_fft_kernel, (int)smem, attr_done); e != cudaSuccess) return e;
  if (p.keys != nullptr) {
    cudaError_t e = cudaMemsetAsync(p.keys, 0, (size_t)p.n_frames * p.n_ant * sizeof(unsigned long long), s);
    if (e != cudaSuccess) return e;
  }
  chip_spectrum_kernel<<<1, 32, 0, s>>>(p.chips, p.n_chips, cspec);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const int L = CF_N - p.n_chips + 1;
  const long long bpr = (p.wins + L - 1) / L;
  const long long total = (long long)p.n_frames * p.n_ant * bpr;
  long long grid = (total + CF_LANES - 1) / CF_LANES;
  if (grid > (long long)device_sm_count() * 2 * 8) grid = (long long)device_sm_count() * 2 * 8;  // persistent-ish: blocks of a row stay on one lane
  corr_fft_kernel<<<(unsigned)grid, 32 * CF_LANES, smem, s>>>(p, cspec, bpr, bound_mode);
  return cudaGetLastError();
}

size_t sync_smem_bytes(int n_chips) { return (size_t)(2 * n_chips - 1 + SYNC_TW + SYNC_K) * sizeof(float2); }

cudaError_t launch_corr(const SyncParams& p, cudaStream_t s) {
  if ((long long)p.n_frames * p.n_ant == 0 || p.wins <= 0) return cudaSuccess;
  const size_t smem = sync_smem_bytes(p.n_chips);
  static unsigned attr_done = 0;  // enough for the largest PN the ABI accepts (8192 chips)
  if (cudaError_t e = ensure_smem_attr(corr_kernel, (int)sync_smem_bytes(8192), attr_done); e != cudaSuccess)
    return e;
  if (p.keys != nullptr) {
    cudaError_t e = cudaMemsetAsync(p.keys, 0, (size_t)p.n_frames * p.n_ant * sizeof(unsigned long long), s);
    if (e != cudaSuccess) return e;
  }
  const dim3 grid((unsigned)((long long)p.n_frames * p.n_ant), (unsigned)((p.wins + SYNC_TW - 1) / SYNC_TW));
  corr_kernel<<<grid, SYNC_THREADS, smem, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_refine(const SyncParams& p, int32_t* peak_idx, double* peak_metric, int bound_mode,
                          cudaStream_t s) {
  const long long rows = (long long)p.n_frames * p.n_ant;
  if (rows == 0) return cudaSuccess;
  refine_kernel<<<(unsigned)rows, REFINE_THREADS, 0, s>>>(p, peak_idx, peak_metric, bound_mode);
  return cudaGetLastError();
}

}  // namespace ofdmrx
