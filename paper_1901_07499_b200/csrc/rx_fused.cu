// Fused uplink receive kernel: CP drop + FFT + fftshift -> LS estimate (pilot)
// -> MRC combine across antennas -> divide -> hard QAM demap, one pass over HBM.
//
// Restates, per frame, the reference's run_ring_pipeline/process_symbol chain
// (receiver.py:238-267,308-348): cp_drop (186-193), to_freq (196-204) ->
// SequentialEngine.freq_transform (92-93), ls_estimate/ls_divide (207-218,
// 95-96), mrc_combine/mrc_seq (221-235; kernels/numba_backend.py:143-162) with
// MRC_WEIGHT_FLOOR (33), and waveform.qam_demap (waveform.py:179-197).
//
// Work decomposition:
//   CTA          = FPB work items, work item = (frame, chunk of DC data symbols)
//   symbol lane  = G threads holding one OFDM symbol's M-point FFT (P points each)
//   lane 0/item  = pilot lane (LS estimate, sum |H|^2), lanes 1..DC = data lanes
//   time loop    = antennas n = 0..N-1; each lane's row (frame, n, symbol) is
//                  TMA bulk-copied into a double-buffered smem slot one antenna
//                  ahead; the pilot lane publishes H_n in its slot; data lanes
//                  accumulate sum_n conj(H_n) Y_n in registers (ascending n =
//                  the SequentialEngine order).
// HBM traffic per frame = the rx samples of 1+D symbols x N antennas (CP never
// read) + H + s_hat + bits (+ weights): the algorithmic minimum.
#include "ofdmrx_fft.cuh"
#include "ofdmrx_internal.h"

namespace ofdmrx {

template <int M>
__global__ void __launch_bounds__(PlanInfo<M>::MAX_THREADS, 1) rx_fused_kernel(const FusedParams p) {
  using PI = PlanInfo<M>;
  constexpr int P = PI::P, G = PI::G, SLOT = PI::SLOT;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int lanes = p.lanes;
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem_raw);
  float2* slots = reinterpret_cast<float2*>(smem_raw + ((2 * lanes * 8 + 127) & ~127));

  const int lane = threadIdx.x / G;
  const int t = threadIdx.x & (G - 1);
  const int per_item = 1 + p.dc;
  const int item = lane / per_item;
  const int sl = lane - item * per_item;
  const bool phantom = lane >= p.fpb * per_item;  // pads the CTA to whole warps
  const int work = blockIdx.x * p.fpb + item;
  const bool item_ok = !phantom && work < p.n_work;
  const int f = item_ok ? work / p.n_chunks : 0;
  const int chunk = item_ok ? work - f * p.n_chunks : 0;
  const bool is_pilot = !phantom && sl == 0;
  const int d = is_pilot ? 0 : chunk * p.dc + (sl - 1);  // data-symbol index (0-based)
  const bool active = item_ok && (is_pilot || d < p.n_data);
  const int pilot_lane = item * per_item;
  const int s = is_pilot ? 0 : d + 1;  // symbol index within the frame
  const LaneSync<G> lsync{1 + lane};

  const float2* row0 = p.rx + (long long)f * p.frame_stride + p.sym0 + (long long)s * (M + p.cp) + p.cp;

  if (threadIdx.x == 0) {
    for (int i = 0; i < 2 * lanes; ++i) mbar_init(&mbar[i], 1);
    fence_mbar_init();
  }
  __syncthreads();

  const bool leader = active && t == 0;
  uint64_t pol = 0;
  if (leader) pol = l2_evict_first_policy();
  auto issue = [&](int n, int st) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(row0 + (long long)n * p.row_stride);
    const uintptr_t start = a & ~uintptr_t(15);
    const uint32_t bytes = (uint32_t)(((a + (uintptr_t)M * 8u + 15u) & ~uintptr_t(15)) - start);
    uint64_t* bar = &mbar[st * lanes + lane];
    mbar_arrive_expect_tx(bar, bytes);
    tma_bulk_g2s(slots + (size_t)(st * lanes + lane) * SLOT, reinterpret_cast<const void*>(start), bytes, bar,
                 pol);
  };
  if (leader) issue(0, 0);

  const bool write_h = is_pilot && active && chunk == 0 && p.H != nullptr;
  const bool write_zf = !is_pilot && active && p.zf != nullptr;
  float2 v[P];
  float2 acc[P];
#pragma unroll
  for (int i = 0; i < P; ++i) acc[i] = make_float2(0.0f, 0.0f);

  for (int n = 0; n < p.n_ant; ++n) {
    const int st = n & 1;
    if (leader && n + 1 < p.n_ant) issue(n + 1, st ^ 1);  // slot freed by the previous step's barrier
    float2* slot = slots + (size_t)(st * lanes + lane) * SLOT;
    if (active) mbar_wait_parity(&mbar[st * lanes + lane], (n >> 1) & 1);
    const int sh = (int)((reinterpret_cast<uintptr_t>(row0 + (long long)n * p.row_stride) >> 3) & 1);
    const float2* src = slot + sh;
    fft_forward<M>(v, slot, t, [&](int idx) { return src[idx]; }, lsync);
    lsync();  // last pass has read the slot; the pilot lane overwrites it with H_n
    if (is_pilot) {
#pragma unroll
      for (int i = 0; i < P; ++i) {
        const int j = shifted_bin<M>(i, t);
        const float2 pc = __ldg(p.pilot + j);
        const float2 y = v[i];
        // H = Y / P for unit-modulus P == Y * conj(P) (bit-exact for BPSK +-1)
        const float2 h = make_float2(fmaf(y.y, pc.y, y.x * pc.x), fmaf(-y.x, pc.y, y.y * pc.x));
        slot[i * G + t] = h;
        acc[i].x += fmaf(h.x, h.x, h.y * h.y);
        if (write_h) p.H[((long long)f * p.n_ant + n) * M + j] = h;
      }
    }
    __syncthreads();  // H_n visible to the data lanes
    if (!is_pilot && active) {
      const float2* hs = slots + (size_t)(st * lanes + pilot_lane) * SLOT;
#pragma unroll
      for (int i = 0; i < P; ++i) {
        const float2 h = hs[i * G + t];
        const float2 y = v[i];
        // conj(H) * Y, expanded as in numba_backend.py:149-150
        acc[i].x += fmaf(h.x, y.x, h.y * y.y);
        acc[i].y += fmaf(h.x, y.y, -h.y * y.x);
        if (write_zf) {
          const float dn = fmaxf(fmaf(h.x, h.x, h.y * h.y), p.eps);
          const float zr = fmaf(h.x, y.x, h.y * y.y), zi = fmaf(h.x, y.y, -h.y * y.x);
          const int j = shifted_bin<M>(i, t);
          p.zf[(((long long)f * p.n_data + d) * p.n_ant + n) * M + j] = make_float2(zr / dn, zi / dn);
        }
      }
    }
    fence_proxy_async_smem();  // generic-proxy smem writes ordered before the next TMA into this stage
    __syncthreads();
  }

  // ---- epilogue: share den, divide, demap ---------------------------------
  uint32_t flag = 0;
  if (is_pilot) {
    float* dslot = reinterpret_cast<float*>(slots + (size_t)lane * SLOT);
#pragma unroll
    for (int i = 0; i < P; ++i) {
      dslot[i * G + t] = acc[i].x;
      if (active) {
        if (!isfinite(acc[i].x)) flag |= 1u;
        if (acc[i].x < p.eps) flag |= 2u;
      }
    }
    if (active && chunk == 0) {
      float* wdst = p.mode == 0 ? p.weights : p.part_den;
      if (wdst != nullptr) {
#pragma unroll
        for (int i = 0; i < P; ++i) wdst[(long long)f * M + shifted_bin<M>(i, t)] = acc[i].x;
      }
    }
  }
  __syncthreads();
  if (!is_pilot && active) {
    const float* dslot = reinterpret_cast<const float*>(slots + (size_t)pilot_lane * SLOT);
    const long long sym_base = ((long long)f * p.n_data + d) * M;
    if (p.mode == 0) {
      const QamParams q{p.qb, p.levels, p.qscale};
#pragma unroll
      for (int i = 0; i < P; ++i) {
        const float den = dslot[i * G + t];
        const float dd = fmaxf(den, p.eps);  // np.maximum(den, eps)
        const float2 sh = make_float2(acc[i].x / dd, acc[i].y / dd);
        if (!isfinite(sh.x) || !isfinite(sh.y)) flag |= 1u;
        const int j = shifted_bin<M>(i, t);
        p.s_hat[sym_base + j] = sh;
        demap_store(sh, q, p.bits + (sym_base + j) * p.qb);
      }
    } else {
#pragma unroll
      for (int i = 0; i < P; ++i) {
        if (!isfinite(acc[i].x) || !isfinite(acc[i].y)) flag |= 1u;
        p.part_num[sym_base + shifted_bin<M>(i, t)] = acc[i];
      }
    }
  }
  if (flag != 0u && p.flags != nullptr) atomicOr(&p.flags[f], flag);
}

template <int M>
static cudaError_t plan_impl(int n_frames, int n_data, FusedLaunch* l) {
  using PI = PlanInfo<M>;
  constexpr int G = PI::G;
  const int lanes_max = PI::MAX_THREADS / G;
  int dc = 0, chunks = 1;
  if (n_data > 0) {
    dc = n_data;
    if (dc > lanes_max - 1) dc = lanes_max - 1;
    if (dc > 15) dc = 15;
    chunks = (n_data + dc - 1) / dc;
    dc = (n_data + chunks - 1) / chunks;
  }
  const int per_item = 1 + dc;
  const size_t slot_bytes = (size_t)PI::SLOT * sizeof(float2);
  const size_t smem_cap = 227 * 1024;
  auto smem_for = [&](int lanes) { return (size_t)((2 * lanes * 8 + 127) & ~127) + 2 * (size_t)lanes * slot_bytes; };
  if (smem_for(per_item) > smem_cap) return cudaErrorInvalidValue;
  int fpb = lanes_max / per_item;
  if (fpb < 1) fpb = 1;
  const long long n_work = (long long)n_frames * chunks;
  const long long want = (n_work + 147) / 148;  // spread items over the 148 SMs first
  if (fpb > want) fpb = (int)(want < 1 ? 1 : want);
  int lanes = fpb * per_item;
  while (true) {
    int padded = lanes;
    if (G < 32) padded = ((lanes * G + 31) / 32 * 32) / G;
    if (smem_for(padded) <= smem_cap || fpb == 1) { lanes = padded; break; }
    --fpb;
    lanes = fpb * per_item;
  }
  if (smem_for(lanes) > smem_cap) return cudaErrorInvalidValue;
  l->dc = dc;
  l->n_chunks = chunks;
  l->fpb = fpb;
  l->lanes = lanes;
  l->threads = lanes * G;
  l->grid = (int)((n_work + fpb - 1) / fpb);
  l->smem = smem_for(lanes);
  return cudaSuccess;
}

template <int M>
static cudaError_t launch_impl(const FusedParams& p, const FusedLaunch& l, cudaStream_t s) {
  static bool attr_set = false;  // benign race: idempotent attribute write
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(rx_fused_kernel<M>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         227 * 1024);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  if (l.grid == 0) return cudaSuccess;
  rx_fused_kernel<M><<<l.grid, l.threads, l.smem, s>>>(p);
  return cudaGetLastError();
}

#define OFDMRX_FOR_EACH_M(X) X(2) X(4) X(8) X(16) X(32) X(64) X(128) X(256) X(512) X(1024) X(2048) X(4096)

cudaError_t fused_plan(int M, int n_frames, int n_data, FusedLaunch* out) {
  switch (M) {
#define X(m) \
  case m:    \
    return plan_impl<m>(n_frames, n_data, out);
    OFDMRX_FOR_EACH_M(X)
#undef X
    default:
      return cudaErrorInvalidValue;
  }
}

cudaError_t launch_fused(int M, const FusedParams& p, const FusedLaunch& l, cudaStream_t s) {
  switch (M) {
#define X(m) \
  case m:    \
    return launch_impl<m>(p, l, s);
    OFDMRX_FOR_EACH_M(X)
#undef X
    default:
      return cudaErrorInvalidValue;
  }
}

}  // namespace ofdmrx
