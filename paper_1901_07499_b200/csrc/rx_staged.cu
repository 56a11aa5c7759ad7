// Staged (unfused) kernels: one kernel per reference stage, used by the
// engine protocol (freq_transform / ls_divide / mrc) and for per-stage timing.
//   fft_rows_kernel  <- SequentialEngine.freq_transform (receiver.py:92-93):
//                       kernels.fft_rows (numba_backend.py:15-52) + fftshift
//   ls_kernel        <- ls_divide (receiver.py:95-96)
//   mrc_kernel       <- mrc_seq (numba_backend.py:143-162) / mrc_tree (109-140)
//   demap_kernel     <- waveform.qam_demap (waveform.py:179-197)
//   finish_kernel    <- the divide+demap tail of mrc_combine/process_symbol after
//                       the antenna-sharded partial sums were exchanged
#include "ofdmrx_fft.cuh"
#include "ofdmrx_internal.h"

namespace ofdmrx {

// ---------------------------------------------------------------------------
// batched CP-drop + FFT + fftshift over rows (frame, symbol, antenna)
// ---------------------------------------------------------------------------
template <int M>
__global__ void __launch_bounds__(256) fft_rows_kernel(const FftRowsParams p, int lanes_per_cta, int iters) {
  using PI = PlanInfo<M>;
  constexpr int P = PI::P, G = PI::G, SLOT = PI::SLOT;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int lane = threadIdx.x / G;
  const int t = threadIdx.x & (G - 1);
  float2* slot = reinterpret_cast<float2*>(smem_raw) + (size_t)lane * SLOT;
  const LaneSync<G> lsync{1 + lane};
  const long long rows = (long long)p.n_frames * p.n_sym * p.n_ant;
  float2 v[P];
  for (int it = 0; it < iters; ++it) {
    const long long row = ((long long)it * gridDim.x + blockIdx.x) * lanes_per_cta + lane;
    const bool ok = row < rows;
    const long long r = ok ? row : 0;
    const int n = (int)(r % p.n_ant);
    const long long fs = r / p.n_ant;
    const int s = (int)(fs % p.n_sym);
    const long long f = fs / p.n_sym;
    const float2* src = p.src + f * p.frame_stride + (long long)n * p.row_stride + p.sym0 + (long long)s * p.sym_stride;
    fft_forward<M>(v, slot, t, [&](int idx) { return ok ? __ldg(src + idx) : make_float2(0.f, 0.f); }, lsync);
    if (ok) {
      float2* dst = p.out + row * M;
#pragma unroll
      for (int i = 0; i < P; ++i) dst[shifted_bin<M>(i, t)] = v[i];
    }
    lsync();  // slot reuse across iterations
  }
}

template <int M>
static cudaError_t fft_rows_impl(const FftRowsParams& p, cudaStream_t s) {
  using PI = PlanInfo<M>;
  constexpr int G = PI::G;
  const int lanes = G >= 256 ? 1 : 256 / G;
  const int threads = lanes * G;
  const size_t smem = (size_t)lanes * PI::SLOT * sizeof(float2);
  static unsigned attr_done = 0;
  if (cudaError_t e = ensure_smem_attr(fft_rows_kernel<M>, 227 * 1024, attr_done); e != cudaSuccess) return e;
  const long long rows = (long long)p.n_frames * p.n_sym * p.n_ant;
  if (rows == 0) return cudaSuccess;
  long long blocks = (rows + lanes - 1) / lanes;
  const long long cap = (long long)device_sm_count() * 16;
  const int grid = (int)(blocks < cap ? blocks : cap);
  const int iters = (int)((blocks + grid - 1) / grid);
  fft_rows_kernel<M><<<grid, threads, smem, s>>>(p, lanes, iters);
  return cudaGetLastError();
}

#define OFDMRX_FOR_EACH_M(X) X(2) X(4) X(8) X(16) X(32) X(64) X(128) X(256) X(512) X(1024) X(2048) X(4096)

cudaError_t launch_fft_rows(int M, const FftRowsParams& p, cudaStream_t s) {
  switch (M) {
#define X(m) \
  case m:    \
    return fft_rows_impl<m>(p, s);
    OFDMRX_FOR_EACH_M(X)
#undef X
    default:
      return cudaErrorInvalidValue;
  }
}

// ---------------------------------------------------------------------------
// LS: H[f, n, k] = Y[f, pilot, n, k] * conj(P[k])
// ---------------------------------------------------------------------------
__global__ void ls_kernel(const float2* __restrict__ Y, long long y_fs, int n_frames, int n_ant, int M,
                          const float2* __restrict__ pilot, float2* __restrict__ H) {
  const long long total = (long long)n_frames * n_ant * M;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int k = (int)(i % M);
    const long long fn = i / M;
    const long long f = fn / n_ant;
    const int n = (int)(fn % n_ant);
    const float2 y = Y[f * y_fs + (long long)n * M + k];
    const float2 pc = __ldg(pilot + k);
    H[i] = make_float2(fmaf(y.y, pc.y, y.x * pc.x), fmaf(-y.x, pc.y, y.y * pc.x));
  }
}

cudaError_t launch_ls(const float2* Y, long long y_fs, int n_frames, int n_ant, int M, const float2* pilot,
                      float2* H, cudaStream_t s) {
  const long long total = (long long)n_frames * n_ant * M;
  if (total == 0) return cudaSuccess;
  long long blocks = (total + 255) / 256;
  if (blocks > device_sm_count() * 32) blocks = device_sm_count() * 32;
  ls_kernel<<<(int)blocks, 256, 0, s>>>(Y, y_fs, n_frames, n_ant, M, pilot, H);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// MRC over antennas for every (frame, data symbol, subcarrier).
// tree=0: ascending antenna order (mrc_seq).  tree=1: the reference pairwise
// tree (numerics.ReductionPlan, numerics.py:85-106) via a binary-counter stack:
// pairs are merged as soon as they complete, the remainder right-to-left,
// which reproduces pairs (2i, 2i+1) with the odd element carried.
// ---------------------------------------------------------------------------
__global__ void mrc_kernel(const MrcParams p) {
  const long long total = (long long)p.n_frames * p.n_data * p.M;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int k = (int)(i % p.M);
    const long long fd = i / p.M;
    const int d = (int)(fd % p.n_data);
    const long long f = fd / p.n_data;
    const float2* y = p.Y + f * p.y_fs + (long long)d * p.y_ss + k;
    const float2* h = p.H + f * (long long)p.n_ant * p.M + k;
    float nr = 0.f, ni = 0.f, dn = 0.f;
    if (!p.tree) {
      for (int n = 0; n < p.n_ant; ++n) {
        const float2 hv = h[(long long)n * p.M], yv = y[(long long)n * p.M];
        nr += fmaf(hv.x, yv.x, hv.y * yv.y);
        ni += fmaf(hv.x, yv.y, -hv.y * yv.x);
        dn += fmaf(hv.x, hv.x, hv.y * hv.y);
        if (p.zf) {
          const float dd = fmaxf(fmaf(hv.x, hv.x, hv.y * hv.y), p.eps);
          p.zf[(fd * p.n_ant + n) * p.M + k] =
              make_float2(fmaf(hv.x, yv.x, hv.y * yv.y) / dd, fmaf(hv.x, yv.y, -hv.y * yv.x) / dd);
        }
      }
    } else {
      float sr[32], si[32], sd[32];
      int top = 0;
      for (int n = 0; n < p.n_ant; ++n) {
        const float2 hv = h[(long long)n * p.M], yv = y[(long long)n * p.M];
        sr[top] = fmaf(hv.x, yv.x, hv.y * yv.y);
        si[top] = fmaf(hv.x, yv.y, -hv.y * yv.x);
        sd[top] = fmaf(hv.x, hv.x, hv.y * hv.y);
        ++top;
        if (p.zf) {
          const float dd = fmaxf(sd[top - 1], p.eps);
          p.zf[(fd * p.n_ant + n) * p.M + k] = make_float2(sr[top - 1] / dd, si[top - 1] / dd);
        }
        for (unsigned c = (unsigned)(n + 1); (c & 1u) == 0u; c >>= 1) {
          --top;
          sr[top - 1] += sr[top];
          si[top - 1] += si[top];
          sd[top - 1] += sd[top];
        }
      }
      while (top > 1) {
        --top;
        sr[top - 1] += sr[top];
        si[top - 1] += si[top];
        sd[top - 1] += sd[top];
      }
      nr = sr[0];
      ni = si[0];
      dn = sd[0];
    }
    const float dd = fmaxf(dn, p.eps);
    p.s_hat[i] = make_float2(nr / dd, ni / dd);
    if (p.weights) p.weights[i] = dn;
  }
}

cudaError_t launch_mrc(const MrcParams& p, cudaStream_t s) {
  const long long total = (long long)p.n_frames * p.n_data * p.M;
  if (total == 0) return cudaSuccess;
  long long blocks = (total + 255) / 256;
  if (blocks > device_sm_count() * 32) blocks = device_sm_count() * 32;
  mrc_kernel<<<(int)blocks, 256, 0, s>>>(p);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// hard demap of a flat symbol vector
// ---------------------------------------------------------------------------
__global__ void demap_kernel(const float2* __restrict__ sym, long long n, QamParams q, uint8_t* __restrict__ bits) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    demap_store(sym[i], q, bits + i * q.qb);
}

cudaError_t launch_demap(const float2* sym, long long n, int qb, int levels, float scale, uint8_t* bits,
                         cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  long long blocks = (n + 255) / 256;
  if (blocks > device_sm_count() * 32) blocks = device_sm_count() * 32;
  demap_kernel<<<(int)blocks, 256, 0, s>>>(sym, n, QamParams{qb, levels, scale}, bits);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// finish after the partial-sum exchange: reduce `parts` partials in the
// reference pairwise-tree order over parts, divide by max(den, eps), demap.
// ---------------------------------------------------------------------------
__global__ void finish_kernel(const FinishParams p) {
  const long long total = (long long)p.n_frames * p.n_data * p.M;
  const long long part_num = total, part_den = (long long)p.n_frames * p.M;
  const QamParams q{p.qb, p.levels, p.qscale};
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int k = (int)(i % p.M);
    const long long f = i / ((long long)p.n_data * p.M);
    const long long di = f * p.M + k;
    // frames a detection rejected (NOT_DETECTED / OUT_OF_RANGE) carry no partials
    if (p.flags != nullptr && (p.flags[f] & 12u) != 0u) continue;
    float sr[32], si[32], sd[32];
    int top = 0;
    for (int g = 0; g < p.parts; ++g) {
      const float2 nv = p.num[g * part_num + i];
      sr[top] = nv.x;
      si[top] = nv.y;
      sd[top] = p.den[g * part_den + di];
      ++top;
      for (unsigned c = (unsigned)(g + 1); (c & 1u) == 0u; c >>= 1) {
        --top;
        sr[top - 1] += sr[top];
        si[top - 1] += si[top];
        sd[top - 1] += sd[top];
      }
    }
    while (top > 1) {
      --top;
      sr[top - 1] += sr[top];
      si[top - 1] += si[top];
      sd[top - 1] += sd[top];
    }
    const float dd = fmaxf(sd[0], p.eps);
    const float2 sh = make_float2(sr[0] / dd, si[0] / dd);
    p.s_hat[i] = sh;
    demap_store(sh, q, p.bits + i * p.qb);
    const bool first_sym = (i / p.M) % p.n_data == 0;
    if (first_sym && p.weights) p.weights[di] = sd[0];
    if (p.flags) {
      uint32_t fl = 0;
      if (!isfinite(sh.x) || !isfinite(sh.y)) fl |= 1u;
      if (first_sym && sd[0] < p.eps) fl |= 2u;
      if (fl) atomicOr(&p.flags[f], fl);
    }
  }
}

cudaError_t launch_finish(const FinishParams& p, cudaStream_t s) {
  const long long total = (long long)p.n_frames * p.n_data * p.M;
  if (total == 0) return cudaSuccess;
  long long blocks = (total + 255) / 256;
  if (blocks > device_sm_count() * 32) blocks = device_sm_count() * 32;
  finish_kernel<<<(int)blocks, 256, 0, s>>>(p);
  return cudaGetLastError();
}

}  // namespace ofdmrx
