// Balanced fused receive for M = 1024 (one 32-thread FFT lane per warp),
// D <= 12 data symbols: the same stages as rx_fused_kernel (CP drop + FFT +
// fftshift -> LS -> MRC -> divide -> demap, receiver.py:238-267,308-348) with
// a different work split.
//
// rx_fused_kernel gives each warp one OFDM symbol for all N antennas, so the
// data warps walk the antennas in lockstep behind the pilot units' H ring and
// every scheduler carries whole symbols: with 1 + 10 symbols on 12 warps, two
// schedulers run three full data warps while the other two carry half-busy
// pilot warps (profiles/experiments_r01_C3.md).  Here:
//   phase A  every warp FFTs pilot rows n = w, w + 12, ...: H_n = Y_n conj(P)
//            is written to the H output (global, L2-resident), |H_n|^2 is
//            accumulated into a per-warp den partial;
//   barrier  (+ generic -> async proxy fence for the H stores)
//   phase B  the D x N data rows, symbol-major (antennas ascending inside a
//            symbol), are cut into 12 equal contiguous ranges.  A warp walks
//            its range with the rx row of step k+1 TMA-prefetched; after the
//            FFT's last pass has read the slot, H_n is TMA-loaded from L2 into
//            that slot for the MAC.  Accumulators (<= 2 symbols per warp: its
//            range is at most N rows) live in TMEM.  No warp waits for another
//            inside the loop.
//   epilogue the owner of each symbol (the warp holding its first row) adds
//            the partial of the warps continuing it (fixed order), den is the
//            fixed-order sum of the 12 warp partials; divide, demap, store.
// Every scheduler gets 3 warps x (704 / 12) rows of the same mix of work.
#include "ofdmrx_fft.cuh"
#include "ofdmrx_internal.h"

namespace ofdmrx {

namespace {

constexpr int BW = 12;     // warps = FFT lanes per CTA
constexpr int BM = 1024;
using BPI = PlanInfo<BM>;
constexpr int BP = BPI::P;  // 32 points per thread
constexpr int BSS = BPI::SLOT;
constexpr int BACC = 2 * BP;             // floats per accumulator set
constexpr int BCOLS = 2 * BACC + BP;     // 2 sets + den partial
constexpr size_t BBAR = 512;             // mbarriers + TMEM address word

__device__ __forceinline__ int range_lo(int w, int total) { return (int)((long long)total * w / BW); }

__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

template <bool BPSK>
__global__ void __launch_bounds__(BW * 32, 1) rx_balanced_kernel(const FusedParams p) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int w = threadIdx.x >> 5, t = threadIdx.x & 31;
  const int f = blockIdx.x;
  const int N = p.n_ant, D = p.n_data;
  uint32_t reject = 0u;
  const long long sym0 = frame_sym0(p, f, BM, &reject);
  if (reject != 0u) {  // not detected / out of range: flagged, no traffic, no outputs
    if (threadIdx.x == 0 && p.flags != nullptr) atomicOr(&p.flags[f], reject);
    return;
  }
  uint64_t* rx_bar = reinterpret_cast<uint64_t*>(smem_raw);  // [BW][2]
  uint64_t* h_bar = rx_bar + 2 * BW;                          // [BW]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(h_bar + BW);
  float2* slot_base = reinterpret_cast<float2*>(smem_raw + BBAR) + (size_t)w * 2 * BSS;
  const bool leader = t == 0;

  if (threadIdx.x < 3 * BW) mbar_init(&rx_bar[threadIdx.x], 1);
  fence_mbar_init();
  if (w == 0) tmem_alloc(tmem_slot, 512);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t tbase = *tmem_slot + ((uint32_t)(32 * (w & 3)) << 16) + (uint32_t)((w >> 2) * BCOLS);
  const uint32_t t_den = tbase + 2 * BACC;

  const float2* frame = p.rx + (long long)f * p.frame_stride + sym0 + p.cp;
  float2* Hf = p.H + (long long)f * N * BM;
  // rx row (symbol s, antenna n): TMA into stage st of this warp
  auto row_addr = [&](int s, int n) { return frame + (long long)n * p.row_stride + (long long)s * (BM + p.cp); };
  auto issue_rx = [&](const float2* src, int st) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(src);
    const uintptr_t start = a & ~uintptr_t(15);
    const uint32_t bytes = (uint32_t)(((a + (uintptr_t)BM * 8u + 15u) & ~uintptr_t(15)) - start);
    uint64_t* bar = &rx_bar[2 * w + st];
    mbar_arrive_expect_tx(bar, bytes);
    // policy made at the issue (1 instruction) rather than held in 2 registers
    tma_bulk_g2s(slot_base + (size_t)st * BSS, reinterpret_cast<const void*>(start), bytes, bar,
                 l2_evict_first_policy());
  };
#ifdef OFDMRX_BAL_H_TMA
  uint32_t h_phase = 0u;
#endif
  // stage st = k & 1 is used at every other step, so its phase is (k >> 1) & 1
  // (a per-stage phase array indexed by st would live in local memory)
  auto wait_rx = [&](int kk) { mbar_wait_parity(&rx_bar[2 * w + (kk & 1)], (uint32_t)(kk >> 1) & 1u); };

  // ---------------- phase A: pilot rows --------------------------------------
  uint32_t pmask = 0;
  if constexpr (BPSK) {
#pragma unroll
    for (int i = 0; i < BP; ++i) pmask |= (__ldg(p.pilot + shifted_bin<BM>(i, t)).x < 0.0f ? 1u : 0u) << i;
  }
  {  // zero the den partial and both accumulator sets (TMEM)
    float z[BACC];
#pragma unroll
    for (int i = 0; i < BACC; ++i) z[i] = 0.0f;
    tmem_st<BP>(t_den, z);
    tmem_st<BACC>(tbase, z);
    tmem_st<BACC>(tbase + BACC, z);
  }
  const int total = D * N;
  const int r0 = range_lo(w, total), r1 = range_lo(w + 1, total);
  int k = 0;  // stage counter across both phases
  if (leader && w < N) issue_rx(row_addr(0, w), 0);
  float2 v[BP];
  for (int n = w; n < N; n += BW, ++k) {
    const int st = k & 1;
    float2* slot = slot_base + (size_t)st * BSS;
    if (leader) {
      if (n + BW < N) issue_rx(row_addr(0, n + BW), st ^ 1);
      else if (r0 < r1) issue_rx(row_addr(1 + r0 / N, r0 % N), st ^ 1);  // first data row of phase B
    }
    wait_rx(k);
    const int sh = (int)((reinterpret_cast<uintptr_t>(row_addr(0, n)) >> 3) & 1);
    const float2* src = slot + sh;
    fft_forward<BM>(v, slot, t, [&](int idx) { return src[idx]; }, [] { __syncwarp(); });
    fence_proxy_async_smem();
    __syncwarp();
    float2* hdst = Hf + (long long)n * BM + t;
    float dp[BP];
    tmem_wait_st();
    tmem_ld<BP>(t_den, dp);
    tmem_wait_ld();
#pragma unroll
    for (int i = 0; i < BP; ++i) {
      const float2 y = v[i];
      float2 h;
      if constexpr (BPSK) {
        const uint32_t sgn = (pmask << (31 - i)) & 0x80000000u;
        h = make_float2(__uint_as_float(__float_as_uint(y.x) ^ sgn), __uint_as_float(__float_as_uint(y.y) ^ sgn));
      } else {
        const float2 pc = __ldg(p.pilot + shifted_bin<BM>(i, t));
        h = make_float2(fmaf(y.y, pc.y, y.x * pc.x), fmaf(-y.x, pc.y, y.y * pc.x));
      }
      dp[i] = fmaf(h.x, h.x, fmaf(h.y, h.y, dp[i]));
      hdst[shifted_bin<BM>(i, 0)] = h;
    }
    tmem_st<BP>(t_den, dp);
  }
  if (leader && w >= N && r0 < r1) issue_rx(row_addr(1 + r0 / N, r0 % N), k & 1);  // no pilot rows
  tmem_wait_st();
  // H rows (generic stores of all warps) -> phase B loads (the TMA variant
  // also needs the generic -> async proxy fences).  A per-antenna mbarrier
  // instead of this barrier measured 0.4 % slower.
  fence_proxy_async_global();
  __syncthreads();
  fence_proxy_async_global();

  // ---------------- phase B: this warp's data rows -----------------------
  const int d_first = r0 < r1 ? r0 / N : 0;
  int d = d_first, n = r0 - d_first * N;   // current row (symbol-major)
  int dn = d, nn = n + 1;                  // next row
  if (nn == N) nn = 0, ++dn;
  for (int r = r0; r < r1; ++r, ++k) {
    const int st = k & 1;
    float2* slot = slot_base + (size_t)st * BSS;
    if (leader && r + 1 < r1) issue_rx(row_addr(1 + dn, nn), st ^ 1);
    wait_rx(k);
    const int sh = (int)((reinterpret_cast<uintptr_t>(row_addr(1 + d, n)) >> 3) & 1);
    const float2* src = slot + sh;
#ifdef OFDMRX_BAL_H_TMA
    fft_forward<BM>(v, slot, t, [&](int idx) { return src[idx]; }, [] { __syncwarp(); },
                    [&] {  // slot consumed: bring H_n from L2 into it while the last pass runs
                      fence_proxy_async_smem();
                      __syncwarp();
                      if (leader) {
                        mbar_arrive_expect_tx(&h_bar[w], BM * 8u);
                        tma_bulk_g2s(slot, Hf + (long long)n * BM, BM * 8u, &h_bar[w], l2_evict_first_policy());
                      }
                    });
    const uint32_t tacc = tbase + (uint32_t)((d - d_first) * BACC);
    float a[BACC];
    tmem_wait_st();
    tmem_ld<BACC>(tacc, a);
    tmem_wait_ld();
    mbar_wait_parity(&h_bar[w], h_phase);
    h_phase ^= 1u;
    auto h_at = [&](int i) { return slot[shifted_bin<BM>(i, t)]; };
#else
    // H_n straight from L2 into registers (ld.global.cg: coherent with the
    // phase-A stores of the other warps), issued once the last FFT pass has
    // its inputs so the latency hides under that pass's butterflies
    float2 hreg[BP];
    const float2* hsrc = Hf + (long long)n * BM + t;
    fft_forward<BM>(v, slot, t, [&](int idx) { return src[idx]; }, [] { __syncwarp(); }, [&] {
#pragma unroll
      for (int i = 0; i < BP; ++i) hreg[i] = __ldcg(hsrc + shifted_bin<BM>(i, 0));
    });
    const uint32_t tacc = tbase + (uint32_t)((d - d_first) * BACC);
    tmem_wait_st();
    // MAC in 16-column TMEM chunks: keeps v + hreg + one chunk in registers
    static_for<BACC / 16>([&](auto ci) {
      constexpr int c = decltype(ci)::value;
      float a[16];
      tmem_ld16(tacc + 16 * c, a);
      tmem_wait_ld();
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int i = 8 * c + q;
        const float2 h = hreg[i];
        const float2 y = v[i];
        // conj(H) * Y = h.x * (y.x, y.y) + h.y * (y.y, -y.x)  (numba_backend.py:149-150)
        const float2 m = upk(fma2(bc(h.y), pk(y.y, -y.x), fma2(bc(h.x), pk(y), pk(a[2 * q], a[2 * q + 1]))));
        a[2 * q] = m.x;
        a[2 * q + 1] = m.y;
      }
      tmem_st16(tacc + 16 * c, a);
    });
#endif
#ifdef OFDMRX_BAL_H_TMA
#pragma unroll
    for (int i = 0; i < BP; ++i) {
      const float2 h = h_at(i);
      const float2 y = v[i];
      const float2 m = upk(fma2(bc(h.y), pk(y.y, -y.x), fma2(bc(h.x), pk(y), pk(a[2 * i], a[2 * i + 1]))));
      a[2 * i] = m.x;
      a[2 * i + 1] = m.y;
    }
    tmem_st<BACC>(tacc, a);
#endif
    fence_proxy_async_smem();  // reads of this slot before its next TMA refill
    __syncwarp();
    d = dn, n = nn;
    if (++nn == N) nn = 0, ++dn;
  }

  // ---------------- epilogue -------------------------------------------------
  tmem_wait_st();
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  float* denbuf = reinterpret_cast<float*>(smem_raw + BBAR);                       // [BW][BM]
  float2* partbuf = reinterpret_cast<float2*>(smem_raw + BBAR + (size_t)BW * BM * 4);  // [BW][BM]
  const bool has_rows = r0 < r1;
  const bool continues = has_rows && (r0 % N) != 0;  // set 0 continues a symbol owned by an earlier warp
  {
    float dp[BP];
    tmem_ld<BP>(t_den, dp);
    tmem_wait_ld();
#pragma unroll
    for (int i = 0; i < BP; ++i) denbuf[w * BM + i * 32 + t] = dp[i];
    if (continues) {
      float a[BACC];
      tmem_ld<BACC>(tbase, a);
      tmem_wait_ld();
#pragma unroll
      for (int i = 0; i < BP; ++i) partbuf[w * BM + i * 32 + t] = make_float2(a[2 * i], a[2 * i + 1]);
    }
  }
  __syncthreads();
  uint32_t flag = 0;
  float den[BP];
#pragma unroll
  for (int i = 0; i < BP; ++i) {
    float s = 0.0f;
    for (int q = 0; q < BW; ++q) s += denbuf[q * BM + i * 32 + t];
    den[i] = s;
  }
  if (w == 0) {
    if (p.weights != nullptr) {
      float* wd = p.weights + (long long)f * BM + t;
#pragma unroll
      for (int i = 0; i < BP; ++i) wd[shifted_bin<BM>(i, 0)] = den[i];
    }
#pragma unroll
    for (int i = 0; i < BP; ++i) {
      if (!isfinite(den[i])) flag |= 1u;
      if (den[i] < p.eps) flag |= 2u;
    }
  }
  // the symbol owned by this warp: its first row lies in [r0, r1)
  const int d_own = has_rows ? (r0 + N - 1) / N : D;
  if (has_rows && d_own * N < r1 && d_own < D) {
    float a[BACC];
    tmem_ld<BACC>(tbase + (uint32_t)((d_own - d_first) * BACC), a);
    tmem_wait_ld();
    // add the partials of the following warps that continue this symbol
    for (int q = w + 1; q < BW; ++q) {
      const int q0 = range_lo(q, total), q1 = range_lo(q + 1, total);
      if (q0 >= q1 || q0 / N != d_own || q0 % N == 0) break;
#pragma unroll
      for (int i = 0; i < BP; ++i) {
        const float2 pv = partbuf[q * BM + i * 32 + t];
        a[2 * i] += pv.x;
        a[2 * i + 1] += pv.y;
      }
    }
    const QamParams qp{p.qb, p.levels, p.qscale};
    const long long sym_base = ((long long)f * D + d_own) * BM;
    float2* sdst = p.s_hat + sym_base + t;
    uint8_t* bdst = p.bits + (sym_base + t) * p.qb;
#pragma unroll
    for (int i = 0; i < BP; ++i) {
      const float dd = fmaxf(den[i], p.eps);
      const float2 shv = make_float2(a[2 * i] / dd, a[2 * i + 1] / dd);
      if (!isfinite(shv.x) || !isfinite(shv.y)) flag |= 1u;
      const int j = shifted_bin<BM>(i, 0);
      sdst[j] = shv;
      demap_store(shv, qp, bdst + (long long)j * p.qb);
    }
  }
  if (flag != 0u && p.flags != nullptr) atomicOr(&p.flags[f], flag);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  if (w == 0) tmem_dealloc(*tmem_slot, 512);
}

}  // namespace

bool balanced_eligible(int M, int n_ant, int n_data, int mode, bool zf, int shards) {
#ifdef OFDMRX_NO_BALANCED
  return false;
#else
  return M == BM && mode == 0 && !zf && shards == 1 && n_data >= 1 && n_data <= BW && n_ant >= 1;
#endif
}

size_t balanced_smem_bytes() { return BBAR + (size_t)BW * 2 * BSS * sizeof(float2); }

cudaError_t launch_balanced(const FusedParams& p, cudaStream_t s) {
  if (p.n_frames == 0) return cudaSuccess;
  static unsigned done_t = 0, done_f = 0;
  const size_t smem = balanced_smem_bytes();
  cudaError_t e = ensure_smem_attr(rx_balanced_kernel<true>, (int)smem, done_t);
  if (e == cudaSuccess) e = ensure_smem_attr(rx_balanced_kernel<false>, (int)smem, done_f);
  if (e != cudaSuccess) return e;
  if (p.pilot_bpsk) rx_balanced_kernel<true><<<p.n_frames, BW * 32, smem, s>>>(p);
  else rx_balanced_kernel<false><<<p.n_frames, BW * 32, smem, s>>>(p);
  return cudaGetLastError();
}

}  // namespace ofdmrx
