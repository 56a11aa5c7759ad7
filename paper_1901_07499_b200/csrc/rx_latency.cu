// Row-parallel receive for single frames and small batches (the paper's
// per-symbol latency regime; OFDMRX_OPT_LATENCY).
//
// The fused kernels give each frame a fixed group of lanes that stream its
// rows in sequence, so one frame alone keeps ~1-8 SMs busy.  Here every FFT
// row of the batch is an independent lane spread over the whole GPU, in
// three stream-ordered launches:
//   1. pilot rows:  CP drop + FFT + fftshift, H_n = Y_n conj(P) -> H
//      (receiver.py:196-218)
//   2. data rows:   CP drop + FFT + fftshift, conj(H_n) Y_n -> per-antenna
//      products in scratch [F, D, N, M] (+ the per-antenna ZF output)
//   3. combine:     per (frame, subcarrier): den = sum_n |H_n|^2, then per
//      data symbol num = sum_n products, in ascending antenna order
//      (mrc_seq, numba_backend.py:143-162), s_hat = num / max(den, eps),
//      demap (waveform.py:179-197), weights, flags.
// The products round-trip through L2 (5 MB per C3 frame).  The antenna-sum
// order is fixed (ascending n), so results never depend on the batch.
#include "ofdmrx_fft.cuh"
#include "ofdmrx_internal.h"

namespace ofdmrx {

namespace {

constexpr int kLatThreads = 256;

// one FFT lane per row; PILOT: rows (f, n) of symbol 0, else rows (f, d, n)
template <int M, bool PILOT, bool BPSK, bool ZF, bool PROF>
__global__ void __launch_bounds__(kLatThreads) lat_rows_kernel(const FusedParams p, float2* prod) {
  using PI = PlanInfo<M>;
  constexpr int P = PI::P, G = PI::G, SLOT = PI::SLOT;
  constexpr int LPC = G >= kLatThreads ? 1 : kLatThreads / G;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int lane = threadIdx.x / G;
  const int t = threadIdx.x & (G - 1);
  float2* slot = reinterpret_cast<float2*>(smem_raw) + (size_t)lane * SLOT;
  const LaneSync<G> lsync{1 + lane};
  const int N = p.n_ant, D = p.n_data;
  const long long rows = PILOT ? (long long)p.n_frames * N : (long long)p.n_frames * D * N;
  const long long row = (long long)blockIdx.x * LPC + lane;
  const bool ok = row < rows;
  const long long r = ok ? row : 0;
  const int n = (int)(r % N);
  const long long fd = r / N;
  const int d = PILOT ? 0 : (int)(fd % D);
  const int f = PILOT ? (int)fd : (int)(fd / D);
  const uint32_t c0 = PROF ? sm_clock() : 0u;
  const float2* src = p.rx + (long long)f * p.frame_stride + (long long)n * p.row_stride + p.sym0 + p.cp +
                      (long long)(PILOT ? 0 : 1 + d) * (M + p.cp);
  float2 y[P];
  fft_forward<M>(y, slot, t, [&](int idx) { return ok ? __ldg(src + idx) : make_float2(0.f, 0.f); }, lsync);
  const uint32_t c1 = PROF ? sm_clock() : 0u;
  if (ok) {
    float2* Hn = p.H + ((long long)f * N + n) * M + t;
    if constexpr (PILOT) {
#pragma unroll
      for (int i = 0; i < P; ++i) {
        const float2 yy = y[i];
        float2 h;
        const float2 pc = __ldg(p.pilot + shifted_bin<M>(i, t));
        if constexpr (BPSK) {
          h = pc.x < 0.0f ? make_float2(-yy.x, -yy.y) : yy;
        } else {
          h = make_float2(fmaf(yy.y, pc.y, yy.x * pc.x), fmaf(-yy.x, pc.y, yy.y * pc.x));
        }
        Hn[shifted_bin<M>(i, 0)] = h;
      }
    } else {
      float2* pr = prod + (((long long)f * D + d) * N + n) * M + t;
#pragma unroll
      for (int i = 0; i < P; ++i) {
        const int j = shifted_bin<M>(i, 0);
        const float2 h = __ldcg(Hn + j), yy = y[i];
        // conj(H) * Y = h.x * (y.x, y.y) + h.y * (y.y, -y.x)  (numba_backend.py:149-150)
        pr[j] = upk(fma2(bc(h.y), pk(yy.y, -yy.x), mul2(bc(h.x), pk(yy))));
        if constexpr (ZF) {
          const float dd = fmaxf(fmaf(h.x, h.x, h.y * h.y), p.eps);
          p.zf[(((long long)f * D + d) * N + n) * M + t + j] =
              make_float2(fmaf(h.x, yy.x, h.y * yy.y) / dd, fmaf(h.x, yy.y, -h.y * yy.x) / dd);
        }
      }
    }
    if (PROF && t == 0) {
      unsigned long long* sc = p.stage_cycles + (long long)f * kStages;
      atomicAdd(sc + (PILOT ? kStagePilotFft : kStageDataFft), (unsigned long long)(c1 - c0));
      atomicAdd(sc + (PILOT ? kStageLs : kStageMrc), (unsigned long long)(sm_clock() - c1));
    }
  }
}

// CTA = (frame, 32 subcarriers) x (nw + 1) warps: warps 0..nw-1 sum the
// products of data symbols d = w, w + nw, ... over the antennas while warp
// nw sums den (both in ascending antenna order, 32 loads in flight per
// thread), so the L2 round trips of num and den overlap; then divide, demap.
constexpr int kCombWarps = 16;
__device__ __forceinline__ float2 sum_rows(const float2* src, int N, int M, bool ok) {
  float2 acc = make_float2(0.f, 0.f);
  for (int n0 = 0; n0 < N; n0 += 32) {
    float2 v[32];
#pragma unroll
    for (int e = 0; e < 32; ++e) v[e] = ok && n0 + e < N ? __ldcg(src + (long long)(n0 + e) * M) : make_float2(0.f, 0.f);
#pragma unroll
    for (int e = 0; e < 32; ++e)
      if (n0 + e < N) acc = upk(add2(pk(acc), pk(v[e])));
  }
  return acc;
}

template <bool PROF>
__global__ void __launch_bounds__(32 * (kCombWarps + 1)) lat_combine_kernel(const FusedParams p, const float2* prod,
                                                                             int M) {
  __shared__ float den_s[32];
  const int N = p.n_ant, D = p.n_data;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x >> 5) - 1;
  const int f = blockIdx.x, k = blockIdx.y * 32 + lane;
  const bool ok = k < M;
  const uint32_t c0 = PROF ? sm_clock() : 0u;
  uint32_t flag = 0;
  const QamParams qp{p.qb, p.levels, p.qscale};
  auto finish = [&](int d, float2 num, float dd) {
    const float2 sh = make_float2(num.x / dd, num.y / dd);
    if (!isfinite(sh.x) || !isfinite(sh.y)) flag |= 1u;
    const long long sym = ((long long)f * D + d) * M + k;
    p.s_hat[sym] = sh;
    demap_store(sh, qp, p.bits + sym * p.qb);
  };
  float2 num0 = make_float2(0.f, 0.f);
  if (w == nw) {  // den warp
    const float2* H = p.H + (long long)f * N * M + k;
    float den = 0.0f;
    for (int n0 = 0; n0 < N; n0 += 32) {
      float2 h[32];
#pragma unroll
      for (int e = 0; e < 32; ++e) h[e] = ok && n0 + e < N ? __ldcg(H + (long long)(n0 + e) * M) : make_float2(0.f, 0.f);
#pragma unroll
      for (int e = 0; e < 32; ++e)
        if (n0 + e < N) den = fmaf(h[e].x, h[e].x, fmaf(h[e].y, h[e].y, den));
    }
    den_s[lane] = den;
    if (ok) {
      if (!isfinite(den)) flag |= 1u;
      if (den < p.eps) flag |= 2u;
      if (p.weights != nullptr) p.weights[(long long)f * M + k] = den;
    }
  } else if (w < D) {  // this warp's first symbol, concurrently with den
    num0 = sum_rows(prod + ((long long)f * D + w) * N * M + k, N, M, ok);
  }
  __syncthreads();
  const float dd = fmaxf(den_s[lane], p.eps);  // np.maximum(den, eps)
  if (w < nw && ok) {
    if (w < D) finish(w, num0, dd);
    for (int d = w + nw; d < D; d += nw) finish(d, sum_rows(prod + ((long long)f * D + d) * N * M + k, N, M, ok), dd);
  }
  if (flag != 0u && p.flags != nullptr) atomicOr(&p.flags[f], flag);
  if (PROF && lane == 0)  // per warp, like the row kernels' per-lane attribution
    atomicAdd(p.stage_cycles + (long long)f * kStages + kStageDemap, (unsigned long long)(sm_clock() - c0));
}

template <int M, bool PILOT, bool BPSK, bool ZF, bool PROF>
cudaError_t launch_rows(const FusedParams& p, float2* prod, cudaStream_t s) {
  using PI = PlanInfo<M>;
  constexpr int G = PI::G, LPC = G >= kLatThreads ? 1 : kLatThreads / G;
  static unsigned done = 0;
  auto kern = lat_rows_kernel<M, PILOT, BPSK, ZF, PROF>;
  const size_t smem = (size_t)LPC * PI::SLOT * sizeof(float2);
  if (cudaError_t e = ensure_smem_attr(kern, (int)smem, done); e != cudaSuccess) return e;
  const long long rows = PILOT ? (long long)p.n_frames * p.n_ant : (long long)p.n_frames * p.n_data * p.n_ant;
  if (rows == 0) return cudaSuccess;
  kern<<<(unsigned)((rows + LPC - 1) / LPC), LPC * G, smem, s>>>(p, prod);
  return cudaGetLastError();
}

template <int M, bool BPSK, bool ZF, bool PROF>
cudaError_t launch_all(const FusedParams& p, float2* prod, cudaStream_t s) {
  if (cudaError_t e = launch_rows<M, true, BPSK, false, PROF>(p, prod, s); e != cudaSuccess) return e;
  if (cudaError_t e = launch_rows<M, false, BPSK, ZF, PROF>(p, prod, s); e != cudaSuccess) return e;
  const int nw = p.n_data < 1 ? 1 : (p.n_data < kCombWarps ? p.n_data : kCombWarps);
  lat_combine_kernel<PROF><<<dim3((unsigned)p.n_frames, (unsigned)((M + 31) / 32)), 32 * (nw + 1), 0, s>>>(p, prod,
                                                                                                          M);
  return cudaGetLastError();
}

template <int M>
cudaError_t launch_m(const FusedParams& p, float2* prod, cudaStream_t s) {
  const bool zf = p.zf != nullptr, prof = p.stage_cycles != nullptr;
#define OFDMRX_LAT(B, Z, PR) \
  if (p.pilot_bpsk == B && zf == Z && prof == PR) return launch_all<M, B, Z, PR>(p, prod, s);
  OFDMRX_LAT(true, false, false)
  OFDMRX_LAT(true, false, true)
  OFDMRX_LAT(true, true, false)
  OFDMRX_LAT(true, true, true)
  OFDMRX_LAT(false, false, false)
  OFDMRX_LAT(false, false, true)
  OFDMRX_LAT(false, true, false)
  OFDMRX_LAT(false, true, true)
#undef OFDMRX_LAT
  return cudaErrorInvalidValue;
}

}  // namespace

size_t latency_scratch_bytes(int n_frames, int n_ant, int n_data, int M) {
  return (size_t)n_frames * n_data * n_ant * M * sizeof(float2);
}

cudaError_t launch_latency(int M, const FusedParams& p, float2* prod, cudaStream_t s) {
  if (p.n_frames == 0) return cudaSuccess;
  switch (M) {
#define X(m) \
  case m:    \
    return launch_m<m>(p, prod, s);
    X(2) X(4) X(8) X(16) X(32) X(64) X(128) X(256) X(512) X(1024) X(2048) X(4096)
#undef X
    default:
      return cudaErrorInvalidValue;
  }
}

}  // namespace ofdmrx
