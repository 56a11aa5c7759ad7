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
//   work item   = (frame, chunk of DC data symbols)
//   symbol lane = G threads computing one OFDM symbol's M-point FFT
//                 (P points per thread, Stockham passes through a smem slot)
//   role unit   = max(32, G) threads = GI lanes of the same symbol slot for the
//                 GI items of a group; unit 0 of a group is the pilot unit.
//   CTA         = NGROUPS groups x (1 + DC) units.
// Every lane loops over the antennas n = 0..N-1 on its own: its row (frame,
// n, symbol) is TMA bulk-copied into a private double-buffered slot one antenna
// ahead.  The pilot unit publishes H_n = Y_n conj(P) into a RING-deep smem ring
// (mbarrier full/empty protocol, no CTA-wide barrier in the loop); data units
// accumulate sum_n conj(H_n) Y_n in registers (ascending n = SequentialEngine
// order).  HBM traffic per frame = rx samples of 1+D symbols x N antennas (CP
// never read) + H + s_hat + bits + weights: the algorithmic minimum.
#include "ofdmrx_fft.cuh"
#include "ofdmrx_internal.h"

namespace ofdmrx {

template <int M>
struct FusedCfg {
  using PI = PlanInfo<M>;
  static constexpr int G = PI::G;
  static constexpr int UT = G < 32 ? 32 : G;  // threads per role unit
  static constexpr int GI = UT / G;           // lanes (items) per unit
  static constexpr int SLOT_STRIDE = PI::SLOT + (G == 1 ? 2 : (G == 8 ? 8 : 0));  // bank skew between lanes
  static constexpr int HSTRIDE = M + 2;       // one item's H block in a ring slot (float2)
  static constexpr int RING = 2;  // must be a multiple of the pilot-unit count (1 or 2)
  static constexpr int NSTAGE = M >= 4096 ? 1 : 2;
  // mbarriers + the TMEM base-address word, rounded up to 128 B
  __host__ __device__ static size_t bar_bytes(int lanes, int ngroups) {
    return ((size_t)(NSTAGE * lanes + 2 * ngroups * RING + 1) * 8 + 127) & ~size_t(127);
  }
  static size_t smem_bytes(int ngroups, int per_group) {
    const int units = ngroups * per_group, lanes = units * GI;
    return bar_bytes(lanes, ngroups) + (size_t)NSTAGE * lanes * SLOT_STRIDE * 8 +
           (size_t)ngroups * RING * GI * HSTRIDE * 8 + (size_t)ngroups * GI * M * 4;  // + den per item
  }
  // TMEM columns: warps of a lane quarter (warp % 4) stack 2P columns each
  __host__ __device__ static uint32_t tmem_cols(int nwarps) {
    const uint32_t need = (uint32_t)((nwarps + 3) / 4) * 2 * PI::P;
    uint32_t c = 32;
    while (c < need) c <<= 1;
    return c;
  }
};

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

template <int M, bool ZF, bool BPSK>
__global__ void __launch_bounds__(PlanInfo<M>::MAX_THREADS, PlanInfo<M>::MIN_CTAS) rx_fused_kernel(const FusedParams p) {
  using PI = PlanInfo<M>;
  using FC = FusedCfg<M>;
  constexpr int P = PI::P, G = PI::G, UT = FC::UT, GI = FC::GI, RING = FC::RING, NSTAGE = FC::NSTAGE;
  constexpr int SS = FC::SLOT_STRIDE, HS = FC::HSTRIDE;
  // MRC accumulators (re, im per point; den for pilots) live in TMEM between
  // antenna steps, keeping the FFT's register budget free for twiddle prefetch
#ifdef OFDMRX_EXP_NOTMEM
  constexpr bool USE_TMEM = false;  // experiment: accumulators in registers (spills at P = 32)
#else
  constexpr bool USE_TMEM = P >= 8;
#endif
  constexpr int NACC = 2 * P;
  extern __shared__ __align__(128) unsigned char smem_raw[];

  const int npilot = p.npilot;          // pilot units per group (the plan uses 1: the epilogue takes den from it)
  const int per_group = npilot + p.dc;  // units per group
  const int ngroups = p.ngroups;
  const int lanes = ngroups * per_group * GI;
  uint64_t* tma_bar = reinterpret_cast<uint64_t*>(smem_raw);  // [NSTAGE][lanes]
  uint64_t* full_bar = tma_bar + NSTAGE * lanes;               // [ngroups][RING]
  uint64_t* empty_bar = full_bar + ngroups * RING;             // [ngroups][RING]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(empty_bar + ngroups * RING);
  const size_t bar_bytes = FC::bar_bytes(lanes, ngroups);
  float2* slots = reinterpret_cast<float2*>(smem_raw + bar_bytes);  // [NSTAGE][lanes][SS]
  float2* ring = slots + (size_t)NSTAGE * lanes * SS;               // [ngroups][RING][GI][HS]
  float* den_sh = reinterpret_cast<float*>(ring + (size_t)ngroups * RING * GI * HS);  // [ngroups][GI][M]

  const int unit = threadIdx.x / UT;
  const int u = threadIdx.x - unit * UT;
  const int grp = unit / per_group;
  const int sl = unit - grp * per_group;
  const int sub = u / G;
  const int t = u - sub * G;
  const int lane = unit * GI + sub;
  const int warp = threadIdx.x >> 5;
  const int work = blockIdx.x * p.fpb + grp * GI + sub;
  bool item_ok = work < p.n_work;
  // work = (frame, chunk, antenna shard), shards innermost
  const int shard = item_ok ? work % p.n_shards : 0;
  const int fc = item_ok ? work / p.n_shards : 0;
  const int f = fc / p.n_chunks;
  const int chunk = fc - f * p.n_chunks;
  const int ant0 = shard * p.n_ant;  // first antenna of this shard (global index)
  uint32_t reject = 0u;
  const long long sym0 = item_ok ? frame_sym0(p, f, M, &reject) : p.sym0;
  if (reject != 0u) {  // not detected / out of range: flagged, no traffic, no outputs
    if (sl == 0 && t == 0 && chunk == 0 && shard == 0 && p.flags != nullptr) atomicOr(&p.flags[f], reject);
    item_ok = false;
  }
  const bool is_pilot = sl < npilot;
  const int d = is_pilot ? 0 : chunk * p.dc + (sl - npilot);  // data-symbol index (0-based)
  const bool active = item_ok && (is_pilot || d < p.n_data);
  const int s = is_pilot ? 0 : d + 1;                          // symbol index within the frame
  // antennas visited by this unit: pilots take every npilot-th antenna
  const int n_first = is_pilot ? sl : 0;
  const int n_step = is_pilot ? npilot : 1;

  // unit == lane group of whole warps: one warp (G <= 32) or G/32 warps
  auto unit_sync = [&]() {
    if constexpr (UT == 32) __syncwarp();
    else named_bar_sync(1 + unit, UT);
  };

  const float2* row0 = p.rx + (long long)f * p.frame_stride + (long long)ant0 * p.row_stride + sym0 +
                       (long long)s * (M + p.cp) + p.cp;

  if (threadIdx.x == 0) {
    for (int i = 0; i < NSTAGE * lanes; ++i) mbar_init(&tma_bar[i], 1);
    for (int i = 0; i < ngroups * RING; ++i) {
      // every thread of the producing / consuming units arrives (each
      // thread's release covers its own ring accesses)
      mbar_init(&full_bar[i], UT);
      mbar_init(&empty_bar[i], (p.dc > 0 ? p.dc : 1) * UT);
    }
    fence_mbar_init();
  }
  const int nwarps = blockDim.x >> 5;
  const uint32_t tmem_cols = FC::tmem_cols(nwarps);
  if constexpr (USE_TMEM) {
    if (warp == 0) tmem_alloc(tmem_slot, tmem_cols);
    tmem_fence_before();
  }
  __syncthreads();
  uint32_t tacc = 0;
  if constexpr (USE_TMEM) {
    tmem_fence_after();
    tacc = *tmem_slot + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * NACC);
  }

  const bool leader = active && t == 0;
  uint64_t pol = 0;
  if (leader) pol = l2_evict_first_policy();
  auto issue_lane = [&](int n, int st) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(row0 + (long long)n * p.row_stride);
    const uintptr_t start = a & ~uintptr_t(15);
    const uint32_t bytes = (uint32_t)(((a + (uintptr_t)M * 8u + 15u) & ~uintptr_t(15)) - start);
    uint64_t* bar = &tma_bar[st * lanes + lane];
    mbar_arrive_expect_tx(bar, bytes);
    tma_bulk_g2s(slots + (size_t)(st * lanes + lane) * SS, reinterpret_cast<const void*>(start), bytes, bar, pol);
  };
  // Row n of every lane of this unit into stage st (called by the whole unit;
  // n is unit-uniform): each lane's leader issues its own copy.  With lanes
  // narrower than a warp (GI > 1) the GI leaders issue converged, and the
  // lanes wait converged on GI different mbarriers -- correct, but
  // compute-sanitizer's racecheck tracks one barrier per warp-level wait and
  // reports "invalid async operation synchronization".  The
  // OFDMRX_RACECHECK_SERIAL build (scripts/sanitize.sh) issues and waits one
  // lane at a time, and is hazard-free under racecheck.
  auto issue = [&](int n, int st) {
#ifdef OFDMRX_RACECHECK_SERIAL
    for (int s2 = 0; s2 < GI; ++s2) {
      if (sub == s2 && leader) issue_lane(n, st);
      __syncwarp();
    }
#else
    if (leader) issue_lane(n, st);
#endif
  };
  auto wait_rx = [&](int st, uint32_t parity) {
#ifdef OFDMRX_RACECHECK_SERIAL
    for (int s2 = 0; s2 < GI; ++s2) {
      if (sub == s2 && active) mbar_wait_parity(&tma_bar[st * lanes + lane], parity);
      __syncwarp();
    }
#else
    if (active) mbar_wait_parity(&tma_bar[st * lanes + lane], parity);
#endif
  };
  if (n_first < p.n_ant) issue(n_first, 0);
#ifdef OFDMRX_EXP_NOLOAD
  constexpr bool kLoadEvery = false;  // experiment: compute-only (first antenna's row reused)
#else
  constexpr bool kLoadEvery = true;
#endif

  // pilot units: BPSK (+-1 real) pilots reduce H = Y conj(P) to a sign flip; the
  // sign bits of this thread's P subcarriers are loaded once.
  uint32_t pmask = 0;
  if (BPSK && is_pilot) {
#pragma unroll
    for (int i = 0; i < P; ++i) pmask |= (__ldg(p.pilot + shifted_bin<M>(i, t)).x < 0.0f ? 1u : 0u) << i;
  }

  // accumulator storage: TMEM columns of this warp, or registers for tiny P
  float accr[USE_TMEM ? 1 : NACC];
  auto acc_load = [&](float* a) {
    if constexpr (USE_TMEM) {
      tmem_wait_st();
      tmem_ld<NACC>(tacc, a);
      tmem_wait_ld();
    } else {
#pragma unroll
      for (int i = 0; i < NACC; ++i) a[i] = accr[i];
    }
  };
  auto acc_store = [&](const float* a) {
    if constexpr (USE_TMEM) tmem_st<NACC>(tacc, a);
    else {
#pragma unroll
      for (int i = 0; i < NACC; ++i) accr[i] = a[i];
    }
  };
  {
    float z[NACC];
#pragma unroll
    for (int i = 0; i < NACC; ++i) z[i] = 0.0f;
    acc_store(z);
  }

  const bool write_h = is_pilot && active && chunk == 0 && p.H != nullptr;
  const bool prof = p.stage_cycles != nullptr;
  uint32_t c_fft = 0u, c_comb = 0u;  // this lane's stage cycles (per-stage attribution)
  float2 v[P];
  float2* hring_grp = ring + (size_t)grp * RING * GI * HS + (size_t)sub * HS;

  for (int k = 0, n = n_first; n < p.n_ant; ++k, n += n_step) {
    const int st = NSTAGE == 2 ? (k & 1) : 0;
    if (kLoadEvery && NSTAGE == 2 && n + n_step < p.n_ant) issue(n + n_step, st ^ 1);  // freed at the end of step k-1
    float2* slot = slots + (size_t)(st * lanes + lane) * SS;
    uint32_t tc = prof ? sm_clock() : 0u;
    if (kLoadEvery || k == 0) wait_rx(st, NSTAGE == 2 ? ((k >> 1) & 1) : (k & 1));
    const int sh = (int)((reinterpret_cast<uintptr_t>(row0 + (long long)n * p.row_stride) >> 3) & 1);
    const float2* src = slot + sh;
#ifdef OFDMRX_EXP_NOFFT
#pragma unroll
    for (int i = 0; i < P; ++i) v[i] = src[i * G + t];  // experiment: skeleton without the FFT
#else
    fft_forward<M>(v, slot, t, [&](int idx) { return src[idx]; }, unit_sync);
#endif
    fence_proxy_async_smem();  // this thread's generic smem writes before the async-proxy refill
    unit_sync();               // every read of the slot done: it may be refilled
    if (kLoadEvery && NSTAGE == 1 && n + n_step < p.n_ant) issue(n + n_step, 0);
    if (prof) {
      const uint32_t t1 = sm_clock();
      c_fft += t1 - tc;
      tc = t1;
    }

    const int r = n % RING;
    const int j = n / RING;
    float2* hb = hring_grp + (size_t)r * GI * HS;
    float a[NACC];
    if (is_pilot) {
      if constexpr (BPSK) asm volatile("" : "+r"(pmask));  // keep the per-bit sign words out of registers
      if (p.dc > 0) mbar_wait_parity(&empty_bar[grp * RING + r], (j + 1) & 1);  // data units done with H_{n-RING}
#pragma unroll
      for (int i = 0; i < P; ++i) {
        const float2 y = v[i];
        float2 h;
        if constexpr (BPSK) {
          const uint32_t sgn = (pmask << (31 - i)) & 0x80000000u;
          h = make_float2(__uint_as_float(__float_as_uint(y.x) ^ sgn), __uint_as_float(__float_as_uint(y.y) ^ sgn));
        } else {
          // H = Y / P for unit-modulus P == Y * conj(P)
          const float2 pc = __ldg(p.pilot + shifted_bin<M>(i, t));
          h = make_float2(fmaf(y.y, pc.y, y.x * pc.x), fmaf(-y.x, pc.y, y.y * pc.x));
        }
        v[i] = h;
      }
#pragma unroll
      for (int i = 0; i < P; i += 2)
        *reinterpret_cast<float4*>(hb + (i >> 1) * 2 * G + 2 * t) = make_float4(v[i].x, v[i].y, v[i + 1].x, v[i + 1].y);
      mbar_arrive(&full_bar[grp * RING + r]);
      acc_load(a);
#pragma unroll
      for (int i = 0; i < P; ++i) {  // (sum h.x^2, sum h.y^2) per subcarrier, added at the end
        const float2 d2 = upk(fma2(pk(v[i]), pk(v[i]), pk(a[2 * i], a[2 * i + 1])));
        a[2 * i] = d2.x;
        a[2 * i + 1] = d2.y;
      }
      acc_store(a);
      if (write_h) {  // off the critical path: the data units already have H_n
        float2* hdst = p.H + ((long long)f * p.ant_total + ant0 + n) * M + t;
#pragma unroll
        for (int i = 0; i < P; ++i) hdst[shifted_bin<M>(i, 0)] = v[i];
      }
    } else {
      mbar_wait_parity(&full_bar[grp * RING + r], j & 1);
      acc_load(a);
#pragma unroll
      for (int i = 0; i < P; i += 2) {
        const float4 hh = *reinterpret_cast<const float4*>(hb + (i >> 1) * 2 * G + 2 * t);
        const float2 h[2] = {make_float2(hh.x, hh.y), make_float2(hh.z, hh.w)};
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const float2 y = v[i + e];
          // conj(H) * Y = h.x * (y.x, y.y) + h.y * (y.y, -y.x)  (numba_backend.py:149-150)
          const float2 m = upk(fma2(bc(h[e].y), pk(y.y, -y.x),
                                    fma2(bc(h[e].x), pk(y), pk(a[2 * (i + e)], a[2 * (i + e) + 1]))));
          a[2 * (i + e)] = m.x;
          a[2 * (i + e) + 1] = m.y;
          if constexpr (ZF) {
            if (active) {
              const float dn = fmaxf(fmaf(h[e].x, h[e].x, h[e].y * h[e].y), p.eps);
              const float zr = fmaf(h[e].x, y.x, h[e].y * y.y), zi = fmaf(h[e].x, y.y, -h[e].y * y.x);
              p.zf[(((long long)f * p.n_data + d) * p.ant_total + ant0 + n) * M + shifted_bin<M>(i + e, t)] =
                  make_float2(zr / dn, zi / dn);
            }
          }
        }
      }
      mbar_arrive(&empty_bar[grp * RING + r]);
      acc_store(a);
    }
    if (prof) c_comb += sm_clock() - tc;
  }
  const uint32_t t_epi = prof ? sm_clock() : 0u;

  // ---- epilogue: den from the pilot unit, divide, demap --------------------
  // The pilot unit publishes den = sum_n |H_n|^2 (its (h.x^2, h.y^2) sums)
  // into the item's den buffer; ONE barrier then covers the den hand-off,
  // the end of the ring traffic and the TMEM reads before the dealloc.
  float a[NACC];
  acc_load(a);  // every unit: its accumulators back to registers
  float* dsh = den_sh + (size_t)(grp * GI + sub) * M;
  if (is_pilot) {
#pragma unroll
    for (int i = 0; i < P; ++i) dsh[i * G + t] = a[2 * i] + a[2 * i + 1];
  }
  if constexpr (USE_TMEM) tmem_fence_before();
  __syncthreads();
  if constexpr (USE_TMEM) {
    tmem_fence_after();
    if (warp == 0) tmem_dealloc(*tmem_slot, tmem_cols);
  }
  uint32_t flag = 0;
  if (is_pilot && active) {
#pragma unroll
    for (int i = 0; i < P; ++i) {
      const float dn = a[2 * i] + a[2 * i + 1];
      if (!isfinite(dn)) flag |= 1u;
      if (p.mode == 0 && dn < p.eps) flag |= 2u;  // partial sums: erasure is decided after the combine
    }
    if (chunk == 0) {
      float* wdst = p.mode == 0 ? p.weights : p.part_den;
      long long wrow = (long long)shard * p.n_frames + f;
      if (p.mode == 1 && p.den_dst != nullptr) {  // routed to the frame's owner
        const int o = f / p.fpo;
        wdst = p.den_dst[o];
        wrow = (long long)p.slot * p.fpo + (f - o * p.fpo);
      }
      if (wdst != nullptr) {
        float* w = wdst + wrow * M + t;
#pragma unroll
        for (int i = 0; i < P; ++i) w[shifted_bin<M>(i, 0)] = a[2 * i] + a[2 * i + 1];
      }
    }
  }
  float* dslot = dsh;
  if (!is_pilot && active) {
    const long long sym_base = (((long long)shard * p.n_frames + f) * p.n_data + d) * M;
    if (p.mode == 0) {
      float2* sdst = p.s_hat + sym_base + t;
      uint8_t* bdst = p.bits + (sym_base + t) * p.qb;
#ifdef OFDMRX_EPI_PLAIN
      const QamParams q{p.qb, p.levels, p.qscale};
#pragma unroll
      for (int i = 0; i < P; ++i) {
        const int j = shifted_bin<M>(i, 0);
        flag |= finish_subcarrier(a[2 * i], a[2 * i + 1], dslot[i * G + t], p.eps, sdst + j, bdst + (long long)j * p.qb, q);
      }
#else
      flag |= finish_points<P>(
          a, [&](int i) { return dslot[i * G + t]; }, p.eps, p.qb, p.levels, p.qscale, sdst, bdst,
          [](int i) { return shifted_bin<M>(i, 0); }, [](int) { return true; });
#endif
    } else {
      float2* ndst = p.part_num + sym_base + t;
      if (p.num_dst != nullptr) {
        const int o = f / p.fpo;
        ndst = p.num_dst[o] + (((long long)p.slot * p.fpo + (f - o * p.fpo)) * p.n_data + d) * M + t;
      }
#pragma unroll
      for (int i = 0; i < P; ++i) {
        if (!isfinite(a[2 * i]) || !isfinite(a[2 * i + 1])) flag |= 1u;
        ndst[shifted_bin<M>(i, 0)] = make_float2(a[2 * i], a[2 * i + 1]);
      }
    }
  }
  if (flag != 0u && p.flags != nullptr) atomicOr(&p.flags[f], flag);
  if (prof && active && t == 0) {
    unsigned long long* sc = p.stage_cycles + (long long)f * kStages;
    atomicAdd(sc + (is_pilot ? kStagePilotFft : kStageDataFft), (unsigned long long)c_fft);
    atomicAdd(sc + (is_pilot ? kStageLs : kStageMrc), (unsigned long long)c_comb);
    atomicAdd(sc + kStageDemap, (unsigned long long)(sm_clock() - t_epi));
  }
  if (p.num_dst != nullptr) {  // peer stores before the exchange flags: the CTA's
    __syncthreads();            // stores happen-before thread 0's (cumulative) system fence
    if (threadIdx.x == 0) __threadfence_system();
  }
}

template <int M>
static cudaError_t plan_impl(int n_frames, int n_data, FusedLaunch* l) {
  using PI = PlanInfo<M>;
  using FC = FusedCfg<M>;
  constexpr int UT = FC::UT, GI = FC::GI;
  const size_t smem_cap = 227 * 1024;
  const int units_max = PI::MAX_THREADS / UT;
  if (FC::smem_bytes(1, 1 + (n_data > 0 ? 1 : 0)) > smem_cap) return cudaErrorInvalidValue;
  // two pilot units (alternating antennas) keep the LS estimate off the critical
  // path when there are enough data units to feed
  // one pilot unit: it is as busy as a data unit (one antenna row per step)
  // and the 2-deep H ring keeps it ahead (A/B on one B200: two alternating
  // pilot units were 1.6 points slower at C1 and equal at C2)
  const int npilot = 1;
  int dc_cap = units_max - npilot;
  if (dc_cap > 15) dc_cap = 15;
  while (dc_cap > 1 && FC::smem_bytes(1, npilot + dc_cap) > smem_cap) --dc_cap;
  int dc = 0, chunks = 1;
  if (n_data > 0) {
    dc = n_data < dc_cap ? n_data : dc_cap;
    chunks = (n_data + dc - 1) / dc;
    dc = (n_data + chunks - 1) / chunks;
  }
  const int per_group = npilot + dc;
  int ngroups = units_max / per_group;
  if (ngroups < 1) ngroups = 1;
  while (ngroups > 1 && FC::smem_bytes(ngroups, per_group) > smem_cap) --ngroups;
  const long long n_work = (long long)n_frames * chunks;
  const long long want = (n_work + (long long)device_sm_count() * GI - 1) / ((long long)device_sm_count() * GI);  // spread groups over the SMs first
  if (ngroups > want) ngroups = (int)(want < 1 ? 1 : want);
  l->dc = dc;
  l->npilot = npilot;
  l->n_chunks = chunks;
  l->ngroups = ngroups;
  l->fpb = ngroups * GI;
  l->lanes = ngroups * per_group * GI;
  l->threads = ngroups * per_group * UT;
  l->grid = (int)((n_work + l->fpb - 1) / l->fpb);
  l->smem = FC::smem_bytes(ngroups, per_group);
  return cudaSuccess;
}

template <int M, bool ZF, bool BPSK>
static cudaError_t launch_one(const FusedParams& p, const FusedLaunch& l, cudaStream_t s) {
  static unsigned attr_done = 0;
  if (cudaError_t e = ensure_smem_attr(rx_fused_kernel<M, ZF, BPSK>, 227 * 1024, attr_done); e != cudaSuccess)
    return e;
  if (l.grid == 0) return cudaSuccess;
  rx_fused_kernel<M, ZF, BPSK><<<l.grid, l.threads, l.smem, s>>>(p);
  return cudaGetLastError();
}

template <int M>
static cudaError_t launch_impl(const FusedParams& p, const FusedLaunch& l, cudaStream_t s) {
  if (p.pilot_bpsk)
    return p.zf != nullptr ? launch_one<M, true, true>(p, l, s) : launch_one<M, false, true>(p, l, s);
  return p.zf != nullptr ? launch_one<M, true, false>(p, l, s) : launch_one<M, false, false>(p, l, s);
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
