// GPU frame synthesizer: the reference transmitter and
// channel simulator as device kernels, so long runs and large batches need
// no host-side generation.
//
// Restates waveform.build_frame (waveform.py:260-286: PN preamble | pilot
// symbol | data symbols, qam_map 164-176 with the Gray table of 133-151,
// ofdm_modulate 248-257: un-shift, inverse FFT, x sqrt(M), cyclic prefix) and
// channel.apply_channel (channel.py:72-108: per-antenna response - identity,
// fixed gains, flat Rayleigh or a multipath FIR truncated to the frame - plus
// complex AWGN at snr_db relative to that antenna's mean signal power, with
// `timing_offset` noise-only samples in front).
//
// Kernels:
//   bits_kernel    payload bits from a counter-based hash of (seed, frame, bit)
//   gains_kernel   flat-Rayleigh gains (CN(0,1)) per (frame, antenna)
//   tx_kernel<M>   one FFT lane per (frame, symbol): map bits/pilot, inverse
//                  FFT via conj(FFT(conj(.))) on the receive path's FFT,
//                  write body + CP
//   sigpow_kernel  per (frame, antenna) signal energy partials (fixed order)
//   channel_kernel response (FIR) + AWGN + timing offset -> rx [F, N, S]
// Random numbers are counter-based (splitmix64 finaliser of (seed, stream,
// index)), so a batch is reproducible and any frame can be generated alone;
// they are NOT numpy's PCG64 streams, so device-synthesised captures are
// distributionally, not bitwise, equal to the reference's (the deterministic
// stages are bit-for-bit the reference's up to fp32 rounding: tests compare
// noiseless captures against the oracle).
#include <cstdint>

#include "ofdmrx_fft.cuh"
#include "ofdmrx_internal.h"

namespace ofdmrx {

namespace {

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
// SplitMix64 per (seed, stream): key once per stream, one finaliser per draw
__device__ __forceinline__ uint64_t rng_key(uint64_t seed, uint64_t stream) {
  return mix64(seed ^ mix64(stream * 0xD1B54A32D192ED03ull));
}
__device__ __forceinline__ uint64_t rng_draw(uint64_t key, uint64_t index) {
  return mix64(key + index * 0x9E3779B97F4A7C15ull);
}
__device__ __forceinline__ uint64_t rng64(uint64_t seed, uint64_t stream, uint64_t index) {
  return rng_draw(rng_key(seed, stream), index);
}
// two independent N(0,1) from one 64-bit draw (Box-Muller, 2 x 32-bit uniforms in (0,1))
__device__ __forceinline__ float2 normal2(uint64_t h) {
  const float u1 = ((float)(uint32_t)(h >> 40) + 0.5f) * (1.0f / 16777216.0f);
  const float u2 = ((float)(uint32_t)(h & 0xffffffu) + 0.5f) * (1.0f / 16777216.0f);
  // fast intrinsics: ~2 ulp log / sin / cos on (0,1) x [0, 2pi) are far
  // below what a noise generator needs
  const float r = sqrtf(-2.0f * __logf(u1));
  float s, c;
  __sincosf(6.283185307179586f * u2, &s, &c);
  return make_float2(r * c, r * s);
}

constexpr uint64_t kStreamBits = 1, kStreamGains = 2, kStreamNoise = 3;

__global__ void bits_kernel(uint8_t* bits, long long n_per_frame, int n_frames, uint64_t seed) {
  const long long total = n_per_frame * n_frames;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long f = i / n_per_frame, j = i - f * n_per_frame;
    bits[i] = (uint8_t)(rng64(seed, kStreamBits + 16 * (uint64_t)f, (uint64_t)j) >> 63);
  }
}

__global__ void gains_kernel(float2* resp, int rows, uint64_t seed) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rows) return;
  const float2 z = normal2(rng64(seed, kStreamGains, (uint64_t)i));
  resp[i] = make_float2(z.x * 0.70710678118654752f, z.y * 0.70710678118654752f);  // (a + ib)/sqrt(2)
}

// waveform._build_constellation point of a b-bit value (MSB-first bits)
__device__ __forceinline__ float2 qam_point(uint32_t value, int axis_bits, int levels, float scale) {
  uint32_t gi = value >> axis_bits, gq = value & (uint32_t)(levels - 1);
  // gray decode: i = g ^ (g >> 1) ^ (g >> 2) ...
  for (int s = 1; s < 8; s <<= 1) {
    gi ^= gi >> s;
    gq ^= gq >> s;
  }
  return make_float2((float)((levels - 1) - 2 * (int)gi) * scale, (float)((levels - 1) - 2 * (int)gq) * scale);
}

template <int M>
__global__ void __launch_bounds__(256) tx_kernel(const SynthParams p, int lanes_per_cta) {
  using PI = PlanInfo<M>;
  constexpr int P = PI::P, G = PI::G;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int lane = threadIdx.x / G;
  const int t = threadIdx.x & (G - 1);
  float2* slot = reinterpret_cast<float2*>(smem_raw) + (size_t)lane * PI::SLOT;
  const LaneSync<G> lsync{1 + lane};
  const long long rows = (long long)p.n_frames * (1 + p.n_data);
  const long long row = (long long)blockIdx.x * lanes_per_cta + lane;
  const bool ok = row < rows;
  const long long f = ok ? row / (1 + p.n_data) : 0;
  const int s = ok ? (int)(row - f * (1 + p.n_data)) : 0;
  const int axis_bits = p.qb >> 1;
  const uint8_t* bsym = p.bits + (f * p.n_data + (s - 1)) * (long long)M * p.qb;
  // IFFT input at natural index j is the fftshift-ed subcarrier k = (j + M/2) mod M
  // (waveform.py:252), conjugated for IFFT = conj(FFT(conj(.)))
  auto load = [&](int j) -> float2 {
    if (!ok) return make_float2(0.f, 0.f);
    const int k = (j + M / 2) & (M - 1);
    float2 x;
    if (s == 0) {
      x = __ldg(p.pilot + k);
    } else {
      uint32_t v = 0;
      for (int b = 0; b < p.qb; ++b) v = (v << 1) | bsym[(long long)k * p.qb + b];
      x = qam_point(v, axis_bits, p.levels, p.qscale);
    }
    return make_float2(x.x, -x.y);
  };
  float2 v[P];
  fft_forward<M>(v, slot, t, load, lsync);
  const float norm = rsqrtf((float)M);  // ifft's 1/M times sqrt(M)
  if (ok) {
    float2* dst = p.tx + f * p.tx_len + (long long)s * (M + p.cp);
#pragma unroll
    for (int i = 0; i < P; ++i) {
      const int n = reg_bin<M>(i, t);  // time index
      const float2 y = make_float2(v[i].x * norm, -v[i].y * norm);
      dst[p.cp + n] = y;
      if (n >= M - p.cp) dst[n - (M - p.cp)] = y;  // cyclic prefix = last cp samples
    }
  }
}

// per (frame, antenna, block) partial signal energy sum_j |(h * x)[j]|^2
constexpr int SIG_BLOCK = 256, SIG_SPAN = 4096;

__device__ __forceinline__ float2 tx_sample(const SynthParams& p, long long f, long long j) {
  if (j < 0) return make_float2(0.f, 0.f);
  if (j < p.pn_len) return make_float2(p.chips[j], 0.f);
  return p.tx[f * p.tx_len + (j - p.pn_len)];
}

__device__ __forceinline__ float2 signal_at(const SynthParams& p, long long f, int n, long long j) {
  const float2* h = p.resp + ((p.resp_per_frame ? f * p.n_ant : 0) + n) * p.n_taps;
  float2 acc = make_float2(0.f, 0.f);
  for (int k = 0; k < p.n_taps; ++k) {
    const float2 x = tx_sample(p, f, j - k);
    const float2 hk = __ldg(h + k);
    acc.x = fmaf(hk.x, x.x, fmaf(-hk.y, x.y, acc.x));
    acc.y = fmaf(hk.x, x.y, fmaf(hk.y, x.x, acc.y));
  }
  return acc;
}

// rows: (frame, antenna) with the channel response applied, or, for flat
// channels (FLAT), frames only: |h|^2 * sum |tx|^2 is applied in channel_kernel
template <bool FLAT>
__global__ void __launch_bounds__(SIG_BLOCK) sigpow_kernel(const SynthParams p, int nblk) {
  const long long rowb = blockIdx.x;
  const long long row = rowb / nblk;
  const int b = (int)(rowb - row * nblk);
  const long long f = FLAT ? row : row / p.n_ant;
  const int n = FLAT ? 0 : (int)(row - f * p.n_ant);
  const long long L = p.pn_len + p.tx_len;
  double e = 0.0;
  for (long long j = (long long)b * SIG_SPAN + threadIdx.x; j < L && j < (long long)(b + 1) * SIG_SPAN;
       j += SIG_BLOCK) {
    const float2 y = FLAT ? tx_sample(p, f, j) : signal_at(p, f, n, j);
    e += (double)y.x * y.x + (double)y.y * y.y;
  }
  __shared__ double red[SIG_BLOCK];
  red[threadIdx.x] = e;
  __syncthreads();
  for (int w = SIG_BLOCK / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) p.sig_part[rowb] = red[0];
}

constexpr int CH_SPAN = 2048;  // samples of one row per channel_kernel block

template <bool FLAT>
__global__ void __launch_bounds__(256) channel_kernel(const SynthParams p, int nblk, int spans) {
  const long long row = blockIdx.x / spans;  // (frame, antenna)
  const long long i0 = (long long)(blockIdx.x - row * spans) * CH_SPAN;
  const long long f = row / p.n_ant;
  const int n = (int)(row - f * p.n_ant);
  const long long L = p.pn_len + p.tx_len;
  const float2 h0 = FLAT ? __ldg(p.resp + (p.resp_per_frame ? f * p.n_ant : 0) + n) : make_float2(1.f, 0.f);
  float sigma = 0.0f;
  if (p.noisy) {
    double e = 0.0;
    const long long prow = FLAT ? f : row;
    for (int b = 0; b < nblk; ++b) e += p.sig_part[prow * nblk + b];
    if (FLAT) e *= (double)h0.x * h0.x + (double)h0.y * h0.y;  // mean |h tx|^2 = |h|^2 mean |tx|^2
    const double noise_power = (e / (double)L) / pow(10.0, (double)p.snr_db / 10.0);
    sigma = (float)sqrt(noise_power / 2.0);
  }
  const uint64_t key = rng_key(p.seed, kStreamNoise + 16 * (uint64_t)row);
  float2* out = p.rx + row * p.n_samples;
  const long long i1 = i0 + CH_SPAN < p.n_samples ? i0 + CH_SPAN : p.n_samples;
  for (long long i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
    const long long j = i - p.offset;
    float2 y = make_float2(0.f, 0.f);
    if (j >= 0 && j < L) {
      if constexpr (FLAT) {
        const float2 x = tx_sample(p, f, j);
        y = make_float2(fmaf(h0.x, x.x, -h0.y * x.y), fmaf(h0.x, x.y, h0.y * x.x));
      } else {
        y = signal_at(p, f, n, j);
      }
    }
    if (sigma > 0.0f) {
      const float2 z = normal2(rng_draw(key, (uint64_t)i));
      y.x = fmaf(sigma, z.x, y.x);
      y.y = fmaf(sigma, z.y, y.y);
    }
    out[i] = y;
  }
}

template <int M>
cudaError_t tx_impl(const SynthParams& p, cudaStream_t s) {
  using PI = PlanInfo<M>;
  constexpr int G = PI::G;
  const int lanes = G >= 256 ? 1 : 256 / G;
  const size_t smem = (size_t)lanes * PI::SLOT * sizeof(float2);
  static unsigned attr_done = 0;
  if (cudaError_t e = ensure_smem_attr(tx_kernel<M>, 227 * 1024, attr_done); e != cudaSuccess) return e;
  const long long rows = (long long)p.n_frames * (1 + p.n_data);
  tx_kernel<M><<<(unsigned)((rows + lanes - 1) / lanes), lanes * G, smem, s>>>(p, lanes);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_synth_bits(uint8_t* bits, long long n_per_frame, int n_frames, uint64_t seed, cudaStream_t s) {
  const long long total = n_per_frame * n_frames;
  if (total == 0) return cudaSuccess;
  long long blocks = (total + 255) / 256;
  if (blocks > device_sm_count() * 64) blocks = device_sm_count() * 64;
  bits_kernel<<<(unsigned)blocks, 256, 0, s>>>(bits, n_per_frame, n_frames, seed);
  return cudaGetLastError();
}

cudaError_t launch_synth_gains(float2* resp, int rows, uint64_t seed, cudaStream_t s) {
  if (rows == 0) return cudaSuccess;
  gains_kernel<<<(rows + 255) / 256, 256, 0, s>>>(resp, rows, seed);
  return cudaGetLastError();
}

cudaError_t launch_synth(const SynthParams& p, cudaStream_t s) {
  if (p.n_frames == 0) return cudaSuccess;
  cudaError_t e;
  switch (p.M) {
#define X(m)                  \
  case m:                     \
    e = tx_impl<m>(p, s);     \
    break;
    X(2) X(4) X(8) X(16) X(32) X(64) X(128) X(256) X(512) X(1024) X(2048) X(4096)
#undef X
    default:
      return cudaErrorInvalidValue;
  }
  if (e != cudaSuccess) return e;
  const long long L = p.pn_len + p.tx_len;
  const int nblk = (int)((L + SIG_SPAN - 1) / SIG_SPAN);
  const long long rows = (long long)p.n_frames * p.n_ant;
  const bool flat = p.n_taps == 1;
  if (p.noisy) {
    if (flat) sigpow_kernel<true><<<(unsigned)((long long)p.n_frames * nblk), SIG_BLOCK, 0, s>>>(p, nblk);
    else sigpow_kernel<false><<<(unsigned)(rows * nblk), SIG_BLOCK, 0, s>>>(p, nblk);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  const int spans = (int)((p.n_samples + CH_SPAN - 1) / CH_SPAN);
  if (flat) channel_kernel<true><<<(unsigned)(rows * spans), 256, 0, s>>>(p, nblk, spans);
  else channel_kernel<false><<<(unsigned)(rows * spans), 256, 0, s>>>(p, nblk, spans);
  return cudaGetLastError();
}

size_t synth_sig_parts(long long pn_len, long long tx_len) {
  return (size_t)((pn_len + tx_len + SIG_SPAN - 1) / SIG_SPAN);
}

}  // namespace ofdmrx
