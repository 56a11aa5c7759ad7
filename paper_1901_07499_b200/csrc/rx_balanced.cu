// Balanced fused receive for M in {1024, 2048, 4096} (FFT lanes of G = 32,
// 64, 128 threads, P = 32 points per thread; lanes narrower than a warp run
// in pairs in the OFDMRX_BAL_PAIRED experiment build): CP drop + FFT + fftshift -> LS
// -> MRC -> divide -> demap (receiver.py:238-267,308-348) with the work of a
// frame cut into V "virtual lanes" whose arithmetic does not depend on how
// the lanes are mapped onto CTAs.
//
// Per frame (V fixed by the frame shape, never by the batch size):
//   phase A  lane v FFTs pilot rows n = v, v + V, ...: H_n = Y_n conj(P) is
//            written to the H output (global, L2-resident), |H_n|^2 is
//            accumulated into the lane's den partial (TMEM);
//            cluster barrier ARRIVE (release: H rows published)
//   phase B  the D x N data rows, symbol-major (antennas ascending inside a
//            symbol), are cut into V contiguous ranges that even out the
//            lanes' pilot + data rows (<= N rows each, so a lane touches at
//            most 2 symbols).  A lane streams its range:
//            the next rx row is TMA-prefetched, and once the FFT's last pass
//            has its inputs the lane loads H_n from L2 into registers
//            (ld.global.cg) so the latency hides under that pass.  The first
//            of these loads is preceded by the cluster barrier WAIT (acquire;
//            an mbarrier when the frame has one CTA), so a lane that finished
//            its pilot rows early runs its first data FFT instead of idling.  MRC accumulators (<= 2 symbols) in TMEM.
//   epilogue den = sum of the V lane partials in lane order; the owner of
//            each symbol (the lane holding its first row) adds the partials
//            of the lanes continuing it, in lane order, then divides, demaps
//            and stores (mode 0) or stores the un-normalised sums (mode 1).
//
// Mapping: a CTA runs LPC lanes; a thread-block cluster of CL = V / LPC CTAs
// runs one frame.  Partials of lanes in other CTAs of the cluster are read
// through distributed shared memory (mapa + ld.shared::cluster), so a small
// batch spreads each frame over several SMs with results bit-identical to
// the one-CTA-per-frame launch a large batch uses.
#include "ofdmrx_fft.cuh"
#include "ofdmrx_internal.h"

namespace ofdmrx {

namespace {

constexpr int BMAXW = 12;       // warps per CTA at most (register budget 168 x 384)
constexpr size_t BBAR = 1024;   // mbarriers, TMEM address word, range table
constexpr int BMAX_V = 96;      // workers per frame at most (8 CTAs x 12 lanes)
constexpr int BMAX_CLUSTER = 8; // portable cluster size

// A virtual lane is a whole number of warps.  FFT plans whose lanes are
// narrower than a warp (G < 32: M = 64, 128, 256, 512) run RB = 32 / G FFTs
// side by side in one warp: the warp streams "super-rows" of RB consecutive
// antennas of one symbol (part b of the warp FFTs antenna n' RB + b), and the
// RB per-part partial sums are combined in part order before the epilogue.
template <int M>
struct BalCfg {
  using PI = PlanInfo<M>;
  static constexpr int P = PI::P, G = PI::G, SLOT = PI::SLOT;
  static constexpr int RB = G < 32 ? 32 / G : 1;  // rows per lane iteration
  static constexpr int WT = G < 32 ? 32 : G;      // threads per virtual lane
  static constexpr int LW = WT / 32;              // warps per virtual lane
  static constexpr int ACC = 2 * P;               // floats per accumulator set
  static constexpr int COLS = (2 * ACC + P + 15) / 16 * 16;  // 2 sets + den partial, per warp (16-aligned)
  static constexpr int LPC_MAX = BMAXW / LW;      // lanes per CTA at most
  // register-lean lanes: two CTAs per SM (24 warps) hide more latency
#ifdef OFDMRX_BAL_MINCTAS16
  static constexpr int MIN_CTAS = P <= 16 ? 2 : 1;  // experiment: 85 registers at P = 16 (spills)
#else
  static constexpr int MIN_CTAS = P <= 8 ? 2 : 1;
#endif
  static_assert((P == 32 || P == 16 || P == 8) && G * RB == WT, "balanced kernel: 8..32 points per thread");
  static size_t smem_bytes(int lpc) { return BBAR + (size_t)lpc * 2 * RB * SLOT * sizeof(float2); }
};

// sum over the RB parts of a warp of value x in part order (identical result
// in every part: each part adds the same RB values in the same order)
template <int RB, int G>
__device__ __forceinline__ float parts_sum(float x) {
  if constexpr (RB == 1) {
    return x;
  } else {
    const int t = threadIdx.x & (G - 1);
    float s = __shfl_sync(0xffffffffu, x, t);
#pragma unroll
    for (int b = 1; b < RB; ++b) s += __shfl_sync(0xffffffffu, x, t + b * G);
    return s;
  }
}

// sum_{a=0}^{x} floor(a / V) (0 for x < 0)
__device__ __forceinline__ long long floor_sum(long long x, int V) {
  if (x < 0) return 0;
  const long long k = x / V, r = x - k * V;
  return V * k * (k - 1) / 2 + k * (r + 1);
}

// Data-row range table lo[0..V] of a frame: lane v streams data rows
// [lo[v], lo[v+1]).  The N(1+D) rows are split evenly over the V lanes
// counting each lane's pilot rows (n = q, q + V, ... < N), so the lanes that
// FFT one pilot row more get one data row less; the boundaries are the
// prefix maximum of that split (monotone even when a lane's pilot share
// exceeds its total, N < V).  A range is at most ceil(N(1+D)/V) <= N rows
// when V > D.  Built once per CTA by warp 0 (closed-form pilot counts and a
// shuffle max-scan), so the hot loop and epilogue only read smem.
__device__ void build_range_table(int* lo, int N, int D, int V) {
  const int lane = threadIdx.x & 31;
  const long long rows = (long long)N * (1 + D);
  const int total = D * N;
  int carry = 0;
  for (int base = 0; base <= V; base += 32) {
    const int q = base + lane;
    int g = 0;
    if (q <= V) {
      const int c = q < N ? q : N;  // lanes before q that own pilot rows
      // pilots before q: sum_{q' < c} (floor((N-1-q')/V) + 1)
      const long long pc = c + floor_sum(N - 1, V) - floor_sum((long long)N - 1 - c, V);
      g = (int)(rows * q / V - pc);
      if (q == V) g = total;
    }
    g = g > carry ? g : carry;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, g, o);
      if (lane >= o && u > g) g = u;
    }
    if (q <= V) lo[q] = g < total ? g : total;
    carry = __shfl_sync(0xffffffffu, g, 31);
  }
}

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_nctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_id_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
// split cluster barrier: every thread of every CTA of the cluster arrives
// once, then waits once (release / acquire at cluster scope)
__device__ __forceinline__ void cluster_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }
__device__ __forceinline__ uint32_t dsmem_addr(const void* local, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(local)), "r"(rank));
  return r;
}
__device__ __forceinline__ float ld_dsmem(uint32_t a) {
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ float2 ld_dsmem2(uint32_t a) {
  float2 v;
  asm volatile("ld.shared::cluster.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a) : "memory");
  return v;
}

template <int M, bool BPSK, bool ZF, bool PROF>
__global__ void __launch_bounds__(BMAXW * 32, BalCfg<M>::MIN_CTAS) rx_balanced_kernel(const FusedParams p) {
  using BC = BalCfg<M>;
  constexpr int P = BC::P, G = BC::G, LW = BC::LW, SS = BC::SLOT, ACC = BC::ACC, COLS = BC::COLS;
  constexpr int RB = BC::RB, WT = BC::WT;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int lpc = blockDim.x / WT;
  const int l = threadIdx.x / WT, t = threadIdx.x % G, w = threadIdx.x >> 5;
  const int part = (threadIdx.x % WT) / G;  // which of the RB FFTs of the lane (0 for whole-warp lanes)
  const uint32_t crank = cluster_ctarank();
  const int V = lpc * (int)cluster_nctarank();
  const int v = (int)crank * lpc + l;  // virtual lane of this thread
  const int f = (int)cluster_id_x();   // one cluster per frame
  const int N = p.n_ant, D = p.n_data;
  const int Nr = N / RB;  // super-antennas (the plan requires RB | N)
  uint32_t reject = 0u;
  const long long sym0 = frame_sym0(p, f, M, &reject);
  if (reject != 0u) {  // not detected / out of range: the whole cluster leaves; flagged, no traffic
    if (threadIdx.x == 0 && crank == 0 && p.flags != nullptr) atomicOr(&p.flags[f], reject);
    return;
  }
  uint64_t* rx_bar = reinterpret_cast<uint64_t*>(smem_raw);  // [lpc][2]
  uint64_t* h_bar = rx_bar + 2 * BC::LPC_MAX;                 // H rows published (one-CTA frames)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(h_bar + 1);
  int* lo_tab = reinterpret_cast<int*>(smem_raw + 256);  // [V + 1]
  uint32_t* cyc = reinterpret_cast<uint32_t*>(smem_raw + 768) + l * kStages;  // this lane's stage cycles
  constexpr bool prof = PROF;  // per-stage attribution build (ofdmrx_rx_frames_profiled)
#ifdef OFDMRX_BAL_CLUSTER_BAR
  const bool one_cta = false;  // experiment: the cluster barrier even for one-CTA frames
#else
  const bool one_cta = V == lpc;
#endif
  float2* slot_base = reinterpret_cast<float2*>(smem_raw + BBAR) + (size_t)l * 2 * RB * SS;
  const bool leader = (threadIdx.x % WT) == 0;  // issues the lane's copies, keeps its stage cycles
  auto lane_sync = [&]() {
    if constexpr (LW == 1) __syncwarp();
    else named_bar_sync(1 + l, WT);
  };

  if (threadIdx.x < 2 * lpc) mbar_init(&rx_bar[threadIdx.x], RB);
  if (prof && leader) {
#pragma unroll
    for (int s = 0; s < kStages; ++s) cyc[s] = 0u;
  }
  if (threadIdx.x == 0) mbar_init(h_bar, blockDim.x);
  fence_mbar_init();
  if (w == 0) build_range_table(lo_tab, Nr, D, V);
  const int nw = lpc * LW;
  uint32_t cols = 32;
  while (cols < (uint32_t)(((nw + 3) / 4) * COLS)) cols <<= 1;
  if (w == 0) tmem_alloc(tmem_slot, cols);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t tbase = *tmem_slot + ((uint32_t)(32 * (w & 3)) << 16) + (uint32_t)((w >> 2) * COLS);
  const uint32_t t_den = tbase + 2 * ACC;

  const float2* frame = p.rx + (long long)f * p.frame_stride + sym0 + p.cp;
  float2* Hf = p.H + (long long)f * N * M;
  auto row_addr = [&](int s, int n) { return frame + (long long)n * p.row_stride + (long long)s * (M + p.cp); };
  // super-row (symbol s, super-antenna nr): RB copies into the stage's RB sub-slots
  auto issue_rx = [&](int s, int nr, int st) {
#pragma unroll
    for (int b = 0; b < RB; ++b) {
      const uintptr_t a = reinterpret_cast<uintptr_t>(row_addr(s, nr * RB + b));
      const uintptr_t start = a & ~uintptr_t(15);
      const uint32_t bytes = (uint32_t)(((a + (uintptr_t)M * 8u + 15u) & ~uintptr_t(15)) - start);
      uint64_t* bar = &rx_bar[2 * l + st];
      mbar_arrive_expect_tx(bar, bytes);
      tma_bulk_g2s(slot_base + (size_t)(st * RB + b) * SS, reinterpret_cast<const void*>(start), bytes, bar,
                   l2_evict_first_policy());
    }
  };
  // stage st = k & 1 is used at every other step, so its phase is (k >> 1) & 1
  auto wait_rx = [&](int kk) { mbar_wait_parity(&rx_bar[2 * l + (kk & 1)], (uint32_t)(kk >> 1) & 1u); };

  // ---------------- phase A: pilot rows --------------------------------------
  uint32_t pmask = 0;
  if constexpr (BPSK) {
#pragma unroll
    for (int i = 0; i < P; ++i) pmask |= (__ldg(p.pilot + shifted_bin<M>(i, t)).x < 0.0f ? 1u : 0u) << i;
  }
  {  // zero the den partial and both accumulator sets (TMEM)
    float z[ACC];
#pragma unroll
    for (int i = 0; i < ACC; ++i) z[i] = 0.0f;
    tmem_st<P>(t_den, z);
    tmem_st<ACC>(tbase, z);
    tmem_st<ACC>(tbase + ACC, z);
  }
#ifdef OFDMRX_BAL_EVEN_SPLIT
  const int total = D * N;
  const int r0 = (int)((long long)total * v / V), r1 = (int)((long long)total * (v + 1) / V);  // experiment
#else
  const int r0 = lo_tab[v], r1 = lo_tab[v + 1];
#endif
  // Phase-B row order.  The lane's rows are symbol d_first from antenna nA
  // on (set A) and, when the range spans a symbol boundary, symbol
  // d_first + 1 up to antenna nB (set B).  They are streamed by ascending
  // ANTENNA, not symbol-major: B-only rows (n < nA), then pairs (d_first, n),
  // (d_first + 1, n) for n in [nA, nB], then A-only rows.  All V lanes of a
  // frame thus sweep the antennas together, so each H row is re-read D times
  // within a short window and stays in L2 even when the H rows of all frames
  // in flight exceed it (C4: 148 x 4 MB).  Each accumulator set still sees
  // its antennas in ascending order: the arithmetic is that of the
  // symbol-major order.
  const int d_first = r0 < r1 ? r0 / Nr : 0;
  const int nA = r0 - d_first * Nr;
  const bool two = r0 < r1 && r1 - 1 >= (d_first + 1) * Nr;
  const int nB = two ? r1 - 1 - (d_first + 1) * Nr : -1;
  // first row: antenna 0 of set B if the lane has one, else antenna nA of A;
  // next row after (n, set): (n, B) if the current is A and n <= nB, else
  // antenna n + 1 (skipping the gap nB < n < nA), set A from nA on
  auto first_row = [&](int& dd, int& nn) {
    nn = two ? 0 : nA;
    dd = d_first + (nn < nA ? 1 : 0);
  };
  auto next_row = [&](int& dd, int& nn) {
    if (dd == d_first && nn <= nB) {
      dd = d_first + 1;
    } else {
      ++nn;
      if (nn > nB && nn < nA) nn = nA;
      dd = d_first + (nn < nA ? 1 : 0);
    }
  };
  const int nrows = r1 - r0;
  int k = 0;  // stage counter across both phases
  // this lane's pilot super-rows v, v + V, ... (pcount of them)
  const int pcount = v < Nr ? (Nr - 1 - v) / V + 1 : 0;
  const int pstart = v, pstep = V;
  if (leader && pcount > 0) issue_rx(0, pstart, 0);
  float2 y[P];
  for (int j = 0; j < pcount; ++j, ++k) {
    const int nr = pstart + j * pstep;
    const int st = k & 1;
    const int n = nr * RB + part;  // this part's antenna
    float2* slot = slot_base + (size_t)(st * RB + part) * SS;
    if (leader) {
      if (j + 1 < pcount) issue_rx(0, nr + pstep, st ^ 1);
      else if (nrows > 0) {  // first data row of phase B
        int d0, n0;
        first_row(d0, n0);
        issue_rx(1 + d0, n0, st ^ 1);
      }
    }
    uint32_t tc = prof ? sm_clock() : 0u;
    wait_rx(k);
    const int sh = (int)((reinterpret_cast<uintptr_t>(row_addr(0, n)) >> 3) & 1);
    const float2* src = slot + sh;
    fft_forward<M>(y, slot, t, [&](int idx) { return src[idx]; }, lane_sync);
    fence_proxy_async_smem();
    lane_sync();
    if (prof) {
      const uint32_t t1 = sm_clock();
      if (leader) cyc[kStagePilotFft] += t1 - tc;
      tc = t1;
    }
    float2* hdst = Hf + (long long)n * M + t;
    float dp[P];
    tmem_wait_st();
    tmem_ld<P>(t_den, dp);
    tmem_wait_ld();
#pragma unroll
    for (int i = 0; i < P; ++i) {
      const float2 yy = y[i];
      float2 h;
      if constexpr (BPSK) {
        const uint32_t sgn = (pmask << (31 - i)) & 0x80000000u;
        h = make_float2(__uint_as_float(__float_as_uint(yy.x) ^ sgn), __uint_as_float(__float_as_uint(yy.y) ^ sgn));
      } else {
        const float2 pc = __ldg(p.pilot + shifted_bin<M>(i, t));
        h = make_float2(fmaf(yy.y, pc.y, yy.x * pc.x), fmaf(-yy.x, pc.y, yy.y * pc.x));
      }
      dp[i] = fmaf(h.x, h.x, fmaf(h.y, h.y, dp[i]));
      hdst[shifted_bin<M>(i, 0)] = h;
    }
    tmem_st<P>(t_den, dp);
    if (prof && leader) cyc[kStageLs] += sm_clock() - tc;
  }
  if (leader && pcount == 0 && nrows > 0) {  // no pilot rows
    int d0, n0;
    first_row(d0, n0);
    issue_rx(1 + d0, n0, k & 1);
  }
  tmem_wait_st();
  // H rows of this lane are published; lanes of the frame acquire them
  // before their first H load (wait inside the first data FFT, below).  One
  // CTA: an mbarrier (release / acquire at CTA scope); a cluster: the split
  // cluster barrier.
  auto h_publish = [&] {
    if (one_cta) mbar_arrive_cta(h_bar);
    else cluster_arrive();
  };
  auto h_acquire = [&] {
    if (one_cta) mbar_wait_parity(h_bar, 0u);
    else cluster_wait();
  };
  h_publish();
  bool h_acquired = false;

  // ---------------- phase B: this lane's data rows -------------------------
  int d, nr;  // current super-row
  first_row(d, nr);
  for (int q = 0; q < nrows; ++q, ++k) {
    const int st = k & 1;
    const int n = nr * RB + part;  // this part's antenna
    float2* slot = slot_base + (size_t)(st * RB + part) * SS;
    int dn = d, nn = nr;  // next super-row
    next_row(dn, nn);
    if (leader && q + 1 < nrows) issue_rx(1 + dn, nn, st ^ 1);
    uint32_t tc = prof ? sm_clock() : 0u;
    wait_rx(k);
    const int sh = (int)((reinterpret_cast<uintptr_t>(row_addr(1 + d, n)) >> 3) & 1);
    const float2* src = slot + sh;
    // H_n straight from L2 into registers (ld.global.cg: coherent with the
    // phase-A stores of the other lanes), issued once the last FFT pass has
    // its inputs so the latency hides under that pass's butterflies
    float2 hreg[P];
    const float2* hsrc = Hf + (long long)n * M + t;
    fft_forward<M>(y, slot, t, [&](int idx) { return src[idx]; }, lane_sync, [&] {
      if (!h_acquired) {
        h_acquire();
        h_acquired = true;
      }
#pragma unroll
      for (int i = 0; i < P; ++i) hreg[i] = __ldcg(hsrc + shifted_bin<M>(i, 0));
    });
    const uint32_t tacc = tbase + (uint32_t)((d - d_first) * ACC);
    if (prof) {
      const uint32_t t1 = sm_clock();
      if (leader) cyc[kStageDataFft] += t1 - tc;
      tc = t1;
    }
    tmem_wait_st();
    // MAC in 16-column TMEM chunks: keeps y + hreg + one chunk in registers
    auto mac_chunk = [&](auto ci, float (&a)[16]) {
      constexpr int c = decltype(ci)::value;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int i = 8 * c + e;
        const float2 h = hreg[i];
        const float2 yy = y[i];
        // conj(H) * Y = h.x * (y.x, y.y) + h.y * (y.y, -y.x)  (numba_backend.py:149-150)
        const float2 m = upk(fma2(bc(h.y), pk(yy.y, -yy.x), fma2(bc(h.x), pk(yy), pk(a[2 * e], a[2 * e + 1]))));
        a[2 * e] = m.x;
        a[2 * e + 1] = m.y;
      }
    };
    // chunk c+1's TMEM load is in flight while chunk c is computed
    {
      constexpr int NCH = ACC / 16;
      float a0[16], a1[16];
      tmem_ld16(tacc, a0);
      tmem_wait_ld();
      static_for<NCH>([&](auto ci) {
        constexpr int c = decltype(ci)::value;
        float(&cur)[16] = (c & 1) ? a1 : a0;
        float(&nxt)[16] = (c & 1) ? a0 : a1;
        if constexpr (c + 1 < NCH) tmem_ld16(tacc + 16 * (c + 1), nxt);
        mac_chunk(ci, cur);
        tmem_st16(tacc + 16 * c, cur);
        if constexpr (c + 1 < NCH) tmem_wait_ld();
      });
    }

    if constexpr (ZF) {  // per-antenna ZF output conj(H) Y / max(|H|^2, eps) (1-row mrc_combine)
      float2* zdst = p.zf + (((long long)f * D + d) * N + n) * M + t;
#pragma unroll
      for (int i = 0; i < P; ++i) {
        const float2 h = hreg[i], yy = y[i];
        const float dd = fmaxf(fmaf(h.x, h.x, h.y * h.y), p.eps);
        zdst[shifted_bin<M>(i, 0)] = make_float2(fmaf(h.x, yy.x, h.y * yy.y) / dd, fmaf(h.x, yy.y, -h.y * yy.x) / dd);
      }
    }
    fence_proxy_async_smem();  // reads of this slot before its next TMA refill
    lane_sync();
    if (prof && leader) cyc[kStageMrc] += sm_clock() - tc;
    d = dn, nr = nn;
  }
  if (!h_acquired) h_acquire();

  // ---------------- epilogue -------------------------------------------------
  const uint32_t t_epi = prof ? sm_clock() : 0u;
  // every lane parks its den partial (and the partial of a symbol it
  // continues) in the now idle TMA slots of its CTA; the cluster reads them
  tmem_wait_st();
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  float* denbuf = reinterpret_cast<float*>(smem_raw + BBAR);                          // [lpc][M]
  float2* partbuf = reinterpret_cast<float2*>(smem_raw + BBAR + (size_t)lpc * M * 4);  // [lpc][M]
  const bool has_rows = r0 < r1;
  const bool continues = has_rows && (r0 % Nr) != 0;  // set 0 continues a symbol owned by an earlier lane
  // a point of the lane's RB parts is stored by part (i mod RB)
  auto mine = [&](int i) { return RB == 1 || (i % RB) == part; };
  {
    float dp[P];
    tmem_ld<P>(t_den, dp);
    tmem_wait_ld();
#pragma unroll
    for (int i = 0; i < P; ++i) {
      const float x = parts_sum<RB, G>(dp[i]);
      if (mine(i)) denbuf[l * M + i * G + t] = x;
    }
    if (continues) {
      float a[ACC];
      tmem_ld<ACC>(tbase, a);
      tmem_wait_ld();
#pragma unroll
      for (int i = 0; i < P; ++i) {
        const float2 x = make_float2(parts_sum<RB, G>(a[2 * i]), parts_sum<RB, G>(a[2 * i + 1]));
        if (mine(i)) partbuf[l * M + i * G + t] = x;
      }
    }
  }
  auto frame_sync = [&] {  // all lanes of the frame (CTA or cluster)
    if (one_cta) {
      __syncthreads();
    } else {
      cluster_arrive();
      cluster_wait();
    }
  };
  frame_sync();

  // den = sum of the V lane partials in a fixed order.  V = NG groups of
  // LPC_MAX consecutive lanes (fixed by the shape and plan, not by the CTA
  // mapping): den = sum over groups (in group order) of the group's lane
  // partials (in lane order).  With NG = 1 every owner sums the lanes itself;
  // with NG > 1 (wide plans, spread over a cluster) the first lane of each
  // group sums its group into gdenbuf first, so owners read NG group sums
  // instead of V partials (distributed shared memory is slow to chase).
  constexpr int GL = BC::LPC_MAX;
  const int NG = V / GL;
  float* gdenbuf = reinterpret_cast<float*>(smem_raw + BBAR + (size_t)lpc * M * 12);  // [M], one group per CTA
  auto lane_den = [&](int q, float (&acc)[P]) {  // acc += lane q's partial (lane q lives in CTA q / lpc)
    const uint32_t rk = (uint32_t)(q / lpc);
    const float* src = denbuf + (q - (int)rk * lpc) * M + t;
    if (rk == crank) {
#pragma unroll
      for (int i = 0; i < P; ++i) acc[i] += src[i * G];
    } else {
      const uint32_t ra = dsmem_addr(src, rk);
#pragma unroll
      for (int i = 0; i < P; ++i) acc[i] += ld_dsmem(ra + 4u * (uint32_t)(i * G));
    }
  };
  // one-CTA frames: the whole CTA sums den once (each thread a strided set of
  // subcarriers, lanes in order), instead of every owner summing all V
  // partials itself
  const bool coop_den = one_cta && NG == 1;
  if (coop_den) {
    for (int k2 = threadIdx.x; k2 < M; k2 += blockDim.x) {
      float acc = 0.0f;
      for (int q = 0; q < V; ++q) acc += denbuf[q * M + k2];
      gdenbuf[k2] = acc;
    }
    __syncthreads();
  }
  if (NG > 1) {
    if (v % GL == 0) {
      float gs[P];
#pragma unroll
      for (int i = 0; i < P; ++i) gs[i] = 0.0f;
      for (int q = v; q < v + GL; ++q) lane_den(q, gs);
#pragma unroll
      for (int i = 0; i < P; ++i)
        if (mine(i)) gdenbuf[i * G + t] = gs[i];
    }
    frame_sync();
  }

  // the symbol owned by this lane: its first row lies in [r0, r1)
  const int d_own = has_rows ? (r0 + Nr - 1) / Nr : D;
  const bool owns = has_rows && d_own < D && d_own * Nr < r1;
  uint32_t flag = 0;
  if (owns || v == 0) {
    float den[P];
#pragma unroll
    for (int i = 0; i < P; ++i) den[i] = 0.0f;
    if (coop_den) {
#pragma unroll
      for (int i = 0; i < P; ++i) den[i] = gdenbuf[i * G + t];
    } else if (NG == 1) {
      for (int q = 0; q < V; ++q) lane_den(q, den);
    } else {
      for (int c = 0; c < NG; ++c) {  // group c's sum lives in the CTA of its first lane
        const uint32_t rk = (uint32_t)(c * GL / lpc);
        const float* src = gdenbuf + t;
        if (rk == crank) {
#pragma unroll
          for (int i = 0; i < P; ++i) den[i] += src[i * G];
        } else {
          const uint32_t ra = dsmem_addr(src, rk);
#pragma unroll
          for (int i = 0; i < P; ++i) den[i] += ld_dsmem(ra + 4u * (uint32_t)(i * G));
        }
      }
    }
    if (v == 0) {
      float* wdst = p.mode == 0 ? p.weights : p.part_den;
      long long wrow = f;
      if (p.mode == 1 && p.den_dst != nullptr) {  // routed to the frame's owner (peer exchange)
        const int o = f / p.fpo;
        wdst = p.den_dst[o];
        wrow = (long long)p.slot * p.fpo + (f - o * p.fpo);
      }
      if (wdst != nullptr) {
        float* wd = wdst + wrow * M + t;
#pragma unroll
        for (int i = 0; i < P; ++i)
          if (mine(i)) wd[shifted_bin<M>(i, 0)] = den[i];
      }
#pragma unroll
      for (int i = 0; i < P; ++i) {
        if (!isfinite(den[i])) flag |= 1u;
        if (p.mode == 0 && den[i] < p.eps) flag |= 2u;  // partial sums: erasure is decided after the combine
      }
    }
    if (owns) {
      float a[ACC];
      tmem_ld<ACC>(tbase + (uint32_t)((d_own - d_first) * ACC), a);
      tmem_wait_ld();
#pragma unroll
      for (int j = 0; j < ACC; ++j) a[j] = parts_sum<RB, G>(a[j]);  // the lane's RB antenna parts, in order
      // add the partials of the following lanes that continue this symbol, in
      // lane order; lanes without rows are skipped (N < V leaves some empty)
      for (int q = v + 1; q < V; ++q) {
#ifdef OFDMRX_BAL_EVEN_SPLIT
        const int q0 = (int)((long long)total * q / V), q1 = (int)((long long)total * (q + 1) / V);
#else
        const int q0 = lo_tab[q], q1 = lo_tab[q + 1];
#endif
        if (q0 >= q1) continue;
        if (q0 / Nr != d_own || q0 % Nr == 0) break;
        const uint32_t rk = (uint32_t)(q / lpc);
        const float2* src = partbuf + (q - (int)rk * lpc) * M + t;
        if (rk == crank) {
#pragma unroll
          for (int i = 0; i < P; ++i) {
            const float2 pv = src[i * G];
            a[2 * i] += pv.x;
            a[2 * i + 1] += pv.y;
          }
        } else {
          const uint32_t ra = dsmem_addr(src, rk);
#pragma unroll
          for (int i = 0; i < P; ++i) {
            const float2 pv = ld_dsmem2(ra + 8u * (uint32_t)(i * G));
            a[2 * i] += pv.x;
            a[2 * i + 1] += pv.y;
          }
        }
      }
      const long long sym_base = ((long long)f * D + d_own) * M;
      if (p.mode == 0) {
        float2* sdst = p.s_hat + sym_base + t;
        uint8_t* bdst = p.bits + (sym_base + t) * p.qb;
#ifdef OFDMRX_EPI_PLAIN
        const QamParams qp{p.qb, p.levels, p.qscale};
#pragma unroll
        for (int i = 0; i < P; ++i) {
          if (!mine(i)) continue;
          const int j = shifted_bin<M>(i, 0);
          flag |= finish_subcarrier(a[2 * i], a[2 * i + 1], den[i], p.eps, sdst + j, bdst + (long long)j * p.qb, qp);
        }
#else
        flag |= finish_points<P>(
            a, [&](int i) { return den[i]; }, p.eps, p.qb, p.levels, p.qscale, sdst, bdst,
            [](int i) { return shifted_bin<M>(i, 0); }, mine);
#endif
      } else {
        float2* ndst = p.part_num + sym_base + t;
        if (p.num_dst != nullptr) {
          const int o = f / p.fpo;
          ndst = p.num_dst[o] + (((long long)p.slot * p.fpo + (f - o * p.fpo)) * D + d_own) * M + t;
        }
#pragma unroll
        for (int i = 0; i < P; ++i) {
          if (!mine(i)) continue;
          if (!isfinite(a[2 * i]) || !isfinite(a[2 * i + 1])) flag |= 1u;
          ndst[shifted_bin<M>(i, 0)] = make_float2(a[2 * i], a[2 * i + 1]);
        }
      }
    }
  }
  if (flag != 0u && p.flags != nullptr) atomicOr(&p.flags[f], flag);
  if (prof && leader) {
    cyc[kStageDemap] += sm_clock() - t_epi;
#pragma unroll
    for (int s = 0; s < kStages; ++s) atomicAdd(&p.stage_cycles[(long long)f * kStages + s], (unsigned long long)cyc[s]);
  }
  // remote readers of this CTA's partials are done before it exits
  tmem_fence_before();
  frame_sync();
  tmem_fence_after();
  if (w == 0) tmem_dealloc(*tmem_slot, cols);
  if (p.num_dst != nullptr && threadIdx.x == 0) __threadfence_system();  // peer stores before the exchange flags
}

template <int M, bool BPSK, bool ZF, bool PROF>
cudaError_t launch_t(const FusedParams& p, const BalancedPlan& bp, cudaStream_t s) {
  using BC = BalCfg<M>;
  static unsigned done = 0;
  auto kern = rx_balanced_kernel<M, BPSK, ZF, PROF>;
  // the launch pads the request (TMEM residency, below): allow the full 227 KB
  if (cudaError_t e = ensure_smem_attr(kern, 227 * 1024, done); e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)p.n_frames * (unsigned)bp.cluster, 1, 1);
  cfg.blockDim = dim3((unsigned)(bp.lanes_per_cta * BC::WT), 1, 1);
  // CTAs of one cluster may share an SM; every CTA allocates TMEM (blocking
  // tcgen05.alloc), so more co-resident CTAs than the SM's 512 columns hold
  // could wait forever on cluster-mates parked at a cluster barrier.  Pad the
  // shared memory request so that at most 512 / cols CTAs fit on an SM.
  const int nw = bp.lanes_per_cta * BC::LW;
  unsigned cols = 32;
  while (cols < (unsigned)(((nw + 3) / 4) * BC::COLS)) cols <<= 1;
  const size_t per_sm = 228 * 1024, fit = 512 / cols;
  size_t smem = BC::smem_bytes(bp.lanes_per_cta);
  if (smem < per_sm / (fit + 1) + 1) smem = per_sm / (fit + 1) + 1;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)bp.cluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, p);
}

template <int M, bool PROF>
cudaError_t launch_mp(const FusedParams& p, const BalancedPlan& bp, cudaStream_t s) {
  const bool zf = p.zf != nullptr;
  if (p.pilot_bpsk) return zf ? launch_t<M, true, true, PROF>(p, bp, s) : launch_t<M, true, false, PROF>(p, bp, s);
  return zf ? launch_t<M, false, true, PROF>(p, bp, s) : launch_t<M, false, false, PROF>(p, bp, s);
}

template <int M>
cudaError_t launch_m(const FusedParams& p, const BalancedPlan& bp, cudaStream_t s) {
  return p.stage_cycles != nullptr ? launch_mp<M, true>(p, bp, s) : launch_mp<M, false>(p, bp, s);
}

template <int M>
bool plan_m(int n_ant, int n_data, int n_frames, int n_sm, bool latency, BalancedPlan* out) {
  using BC = BalCfg<M>;
  constexpr int LMAX = BC::LPC_MAX;
  // V (virtual lanes per frame) depends on the frame shape only: the fewest
  // CTAs' worth of lanes with V > D, so that a lane's range (<= N(1+D)/V
  // rows) never spans more than two symbols.  Few CTAs per frame keep the
  // cluster small at large batches (a GPC fits fewer 8-CTA clusters than its
  // SM count suggests, and the epilogue waits on every CTA of the frame).
  if (n_ant % BC::RB != 0) return false;  // sub-warp FFT lanes pair up antennas
  int c = (n_data + 1 + LMAX - 1) / LMAX;
  if (latency) {  // OFDMRX_OPT_LATENCY: the widest portable cluster, >= ~4 rows per worker
    const long long rows = (long long)n_ant * (1 + n_data);
    long long cl = (rows + 4LL * LMAX - 1) / (4LL * LMAX);
    if (cl > BMAX_CLUSTER) cl = BMAX_CLUSTER;
    if (cl > c) c = (int)cl;
  }
  if (c > BMAX_CLUSTER || c * LMAX > BMAX_V) return false;
  const int V = c * LMAX;
  // CTA mapping depends on the batch: the fewest CTAs per frame (largest
  // lpc) that still give every SM a CTA, within the portable cluster size
  int best_lpc = LMAX;
  for (int lpc = LMAX; lpc >= 1; --lpc) {
    if (V % lpc != 0 || V / lpc > BMAX_CLUSTER) continue;
    best_lpc = lpc;
    if ((long long)n_frames * (V / lpc) >= n_sm) break;
  }
  out->workers = V;
  out->lanes_per_cta = best_lpc;
  out->cluster = V / best_lpc;
  out->fft_lane_threads = BC::G;
  return true;
}

}  // namespace

bool balanced_plan(int M, int n_ant, int n_data, int n_frames, int n_sm, bool latency, BalancedPlan* out) {
#ifdef OFDMRX_NO_BALANCED
  return false;
#else
  if (n_ant < 1 || n_data < 0) return false;
  switch (M) {
#ifdef OFDMRX_BAL_PAIRED
    // experiment: paired sub-warp FFT lanes (A/B on one B200, C2 at 1000 /
    // 2000 frames: 35 % / 37 % of the roofline vs 42 % / 51 % for rx_fused)
    case 256: return plan_m<256>(n_ant, n_data, n_frames, n_sm, latency, out);
    case 512: return plan_m<512>(n_ant, n_data, n_frames, n_sm, latency, out);
#endif
    case 1024: return plan_m<1024>(n_ant, n_data, n_frames, n_sm, latency, out);
    case 2048: return plan_m<2048>(n_ant, n_data, n_frames, n_sm, latency, out);
    case 4096: return plan_m<4096>(n_ant, n_data, n_frames, n_sm, latency, out);
    default: return false;
  }
#endif
}

size_t balanced_smem_bytes(int M, int lanes_per_cta) {
  switch (M) {
#ifdef OFDMRX_BAL_PAIRED
    case 256: return BalCfg<256>::smem_bytes(lanes_per_cta);
    case 512: return BalCfg<512>::smem_bytes(lanes_per_cta);
#endif
    case 1024: return BalCfg<1024>::smem_bytes(lanes_per_cta);
    case 2048: return BalCfg<2048>::smem_bytes(lanes_per_cta);
    case 4096: return BalCfg<4096>::smem_bytes(lanes_per_cta);
    default: return 0;
  }
}

cudaError_t launch_balanced(int M, const FusedParams& p, const BalancedPlan& bp, cudaStream_t s) {
  if (p.n_frames == 0) return cudaSuccess;
  switch (M) {
#ifdef OFDMRX_BAL_PAIRED
    case 256: return launch_m<256>(p, bp, s);
    case 512: return launch_m<512>(p, bp, s);
#endif
    case 1024: return launch_m<1024>(p, bp, s);
    case 2048: return launch_m<2048>(p, bp, s);
    case 4096: return launch_m<4096>(p, bp, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace ofdmrx
