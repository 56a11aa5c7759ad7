// Internal launch interfaces shared by the kernel TUs and the C-ABI layer.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace ofdmrx {

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per kernel and device;
// `done` is the call site's static bit set of devices already configured
// (idempotent, so a race only repeats the attribute write).
template <typename K>
inline cudaError_t ensure_smem_attr(K kernel, int bytes, unsigned& done) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const unsigned bit = dev < 32 ? 1u << dev : 0u;
  if (bit != 0u && (done & bit) != 0u) return cudaSuccess;
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done |= bit;
  return e;
}

// Fused receive: one CTA processes FPB work items; a work item is one
// (frame, chunk of data symbols) pair and owns 1 + DC "symbol lanes"
// (lane 0 = pilot).  Every lane streams its symbol's antenna rows through
// a double-buffered TMA stage, FFTs them, and the pilot lane hands the LS
// estimate H_n to the data lanes through shared memory.
struct FusedParams {
  const float2* rx;        // capture base (cf32)
  long long frame_stride;  // samples between frames
  long long row_stride;    // samples between antenna rows
  long long sym0;          // offset (samples) of the pilot symbol's CP inside a row
  int n_frames, n_ant, cp, n_data;   // n_ant = antennas per shard
  int n_shards, ant_total;           // antenna shards per frame (mode 1 only when > 1)
  int dc, n_chunks, fpb, n_work, lanes, ngroups, npilot;
  const float2* pilot;     // [M] pilot values, subcarrier (shifted) order
  float eps;
  int qb, levels;
  float qscale;
  int mode;                // 0 = full (divide + demap), 1 = partial sums
  int pilot_bpsk;          // pilot values are exactly +-1 (sign-flip LS)
  // outputs (nullable unless noted)
  float2* H;               // [F, N, M]
  float2* s_hat;           // [F, D, M]            (mode 0, required)
  float* weights;          // [F, M]
  uint8_t* bits;           // [F, D*M*qb]          (mode 0, required)
  float2* zf;              // [F, D, N, M]
  uint32_t* flags;         // [F]
  float2* part_num;        // [S, F, D, M]         (mode 1, required)
  float* part_den;         // [S, F, M]            (mode 1, required)
  // mode 1 routed to peers (antenna-sharded exchange over peer memory):
  // frame f goes to owner o = f / fpo, slot `slot` of its inbox
  // num_dst[o] [G, fpo, D, M] and den_dst[o] [G, fpo, M]
  float2* const* num_dst;
  float* const* den_dst;
  int fpo, slot;
  // per-frame symbol0 from a device-side detection (ofdmrx_rx_frames_detected):
  // sym0_f = det_idx[f * det_stride] + det_add; frames whose antenna-0 peak is
  // below det_threshold, or whose symbols overrun n_samples, are flagged and skipped
  const int32_t* det_idx;
  const double* det_metric;
  int det_stride, det_add;
  double det_threshold;
  long long n_samples;
  // optional per-stage attribution (ofdmrx_rx_frames_profiled): SM clock
  // cycles of every lane, summed per frame and stage (kStage*)
  unsigned long long* stage_cycles;  // [F, kStages]
};

// stages of the per-stage attribution (StageTimings fields, receiver.py:65-79)
constexpr int kStagePilotFft = 0;  // pilot symbol: TMA wait + FFT          -> fft_s  (pilot)
constexpr int kStageLs = 1;        // H = Y conj(P), |H|^2, H store          -> combine_s (pilot, "ls")
constexpr int kStageDataFft = 2;   // data symbols: TMA wait + FFT          -> fft_s  (data)
constexpr int kStageMrc = 3;       // conj(H) Y accumulation (+ ZF output)   -> combine_s (data, "mrc")
constexpr int kStageDemap = 4;     // combine, divide, demap, stores         -> combine_s (data, "mrc")
constexpr int kStages = 5;

__device__ __forceinline__ uint32_t sm_clock() {
  uint32_t c;
  asm volatile("mov.u32 %0, %%clock;" : "=r"(c));
  return c;
}

// per-frame symbol0 (detected or fixed) and the frame's admission flags
__device__ __forceinline__ long long frame_sym0(const FusedParams& p, int f, int M, uint32_t* reject) {
  *reject = 0u;
  if (p.det_idx == nullptr) return p.sym0;
  const long long s0 = (long long)p.det_idx[(long long)f * p.det_stride] + p.det_add;
  if (!(p.det_metric[(long long)f * p.det_stride] >= p.det_threshold)) *reject |= 4u;  // OFDMRX_FLAG_NOT_DETECTED
  if (s0 + (long long)(1 + p.n_data) * (M + p.cp) > p.n_samples) *reject |= 8u;       // OFDMRX_FLAG_OUT_OF_RANGE
  return *reject ? 0 : s0;
}

struct FusedLaunch {
  int dc, n_chunks, fpb, lanes, threads, grid, ngroups, npilot;
  size_t smem;
};

// Balanced variant (rx_balanced.cu), M in {1024, 2048, 4096}: V virtual FFT
// lanes per frame (fixed by the frame shape: the antenna-sum order), mapped
// onto `cluster` CTAs of `lanes_per_cta` lanes each (chosen per batch).
// Needs p.H (caller supplies scratch).
struct BalancedPlan {
  int workers;          // V virtual lanes per frame
  int lanes_per_cta;    // LPC
  int cluster;          // CTAs per frame (thread-block cluster size)
  int fft_lane_threads; // G
};
bool balanced_plan(int M, int n_ant, int n_data, int n_frames, int n_sm, bool latency, BalancedPlan* out);
size_t balanced_smem_bytes(int M, int lanes_per_cta);
cudaError_t launch_balanced(int M, const FusedParams& p, const BalancedPlan& bp, cudaStream_t s);

// Row-parallel latency path (rx_latency.cu, OFDMRX_OPT_LATENCY, mode 0):
// pilot rows -> H, data rows -> conj(H) Y into prod [F, D, N, M], combine.
// Needs p.H (caller supplies scratch).
size_t latency_scratch_bytes(int n_frames, int n_ant, int n_data, int M);
cudaError_t launch_latency(int M, const FusedParams& p, float2* prod, cudaStream_t s);

// multiprocessor count of the current device (cached per device)
int device_sm_count();

// returns cudaErrorInvalidValue for unsupported M
cudaError_t fused_plan(int M, int n_frames, int n_data, FusedLaunch* out);
cudaError_t launch_fused(int M, const FusedParams& p, const FusedLaunch& l, cudaStream_t s);

// Staged kernels (per-stage timing and the engine protocol).
struct FftRowsParams {
  const float2* src;
  long long frame_stride, row_stride, sym0, sym_stride;  // row address = src + f*fs + n*rs + sym0 + s*ss
  int n_frames, n_sym, n_ant;                            // rows = F*S*N, output [F, S, N, M]
  float2* out;
};
cudaError_t launch_fft_rows(int M, const FftRowsParams& p, cudaStream_t s);

cudaError_t launch_ls(const float2* Y, long long y_frame_stride, int n_frames, int n_ant, int M,
                      const float2* pilot, float2* H, cudaStream_t s);

struct MrcParams {
  const float2* Y;         // data symbols: Y + f*y_fs + d*y_ss + n*M + k
  long long y_fs, y_ss;
  const float2* H;         // H + f*N*M + n*M + k
  int n_frames, n_data, n_ant, M;
  float eps;
  int tree;                // 0 = ascending antenna order, 1 = pairwise tree
  float2* s_hat;           // [F, D, M]
  float* weights;          // [F, D, M]
  float2* zf;              // [F, D, N, M] or null
};
cudaError_t launch_mrc(const MrcParams& p, cudaStream_t s);

cudaError_t launch_demap(const float2* sym, long long n, int qb, int levels, float scale, uint8_t* bits,
                         cudaStream_t s);

struct FinishParams {
  const float2* num;       // [parts, F, D, M]
  const float* den;        // [parts, F, M]
  int parts, n_frames, n_data, M;
  float eps;
  int qb, levels;
  float qscale;
  float2* s_hat;           // [F, D, M]
  float* weights;          // [F, M] or null
  uint8_t* bits;           // [F, D*M*qb]
  uint32_t* flags;         // [F] or null
};
cudaError_t launch_finish(const FinishParams& p, cudaStream_t s);

// PN detection (sync.cu): rows = (frame, antenna) streams of n_samples.
struct SyncParams {
  const float2* rx;
  long long frame_stride, row_stride, n_samples;
  int n_frames, n_ant;
  const float* chips;           // [n_chips] real chips (bipolar PN)
  int n_chips;
  long long wins;               // n_samples - n_chips + 1
  float* metrics;               // [F*N, wins] fp32 metrics
  unsigned long long* keys;     // [F*N] per-row (metric, first index) max key, or null
};
size_t sync_smem_bytes(int n_chips);
cudaError_t launch_corr(const SyncParams& p, cudaStream_t s);
cudaError_t launch_refine(const SyncParams& p, int32_t* peak_idx, double* peak_metric, int bound_mode,
                          cudaStream_t s);
// overlap-save FFT correlation for 64 <= n_chips <= 960 (cspec: 1024 cf32 scratch);
// bound_mode 1 writes per-window upper bounds and keys on lower bounds (detect)
bool sync_use_fft(int n_chips);
size_t sync_fft_scratch_bytes();
cudaError_t launch_corr_fft(const SyncParams& p, float2* cspec, int bound_mode, cudaStream_t s);

// Frame synthesizer (synth.cu).
struct SynthParams {
  int n_frames, n_ant, M, cp, n_data, qb, levels;
  float qscale;
  int pn_len;
  long long tx_len;            // (1 + D) * (M + cp) samples after the preamble
  long long n_samples;         // samples per rx row (>= offset + pn_len + tx_len)
  long long offset;            // timing offset: noise-only samples in front
  const float2* pilot;         // [M] subcarrier (shifted) order
  const float* chips;          // [pn_len] bipolar PN
  const uint8_t* bits;         // [F, D*M*qb]
  const float2* resp;          // [F or 1, N, n_taps] channel response
  int n_taps, resp_per_frame;
  int noisy;
  float snr_db;
  unsigned long long seed;
  float2* tx;                  // [F, tx_len] scratch
  double* sig_part;            // [F*N, parts] scratch
  float2* rx;                  // [F, N, n_samples]
};
cudaError_t launch_synth_bits(uint8_t* bits, long long n_per_frame, int n_frames, uint64_t seed, cudaStream_t s);
cudaError_t launch_synth_gains(float2* resp, int rows, uint64_t seed, cudaStream_t s);
cudaError_t launch_synth(const SynthParams& p, cudaStream_t s);
size_t synth_sig_parts(long long pn_len, long long tx_len);

// Peer-memory exchange flags (peer.cu)
cudaError_t launch_peer_signal(unsigned long long* const* dst, int n, unsigned long long value, cudaStream_t s);
cudaError_t launch_peer_wait(const unsigned long long* const* src, int n, unsigned long long value, cudaStream_t s);

}  // namespace ofdmrx
