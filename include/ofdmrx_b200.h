/*
 * ofdmrx_b200 — C ABI of the B200 (sm_100a) uplink OFDM receive path.
 *
 * Drop-in boundary for the reference receiver's hot path
 * (/root/reference/pkg/src/ofdmrx).  The reference has no native FFI — its
 * swap points are the Python engine protocol (receiver.py:88-179) and the
 * kernel-backend protocol (kernels/__init__.py:40-68).  Each entry point below
 * names the reference interface it replaces; INTEGRATION.md shows the ctypes
 * binding a maintainer adds to the reference to route those calls here.
 *
 * Conventions
 *  - All data pointers are DEVICE pointers (cudaMalloc / torch CUDA tensors),
 *    complex samples are interleaved float32 (cf32, the .cf32 file layout of
 *    io_formats.py:18-30), bits are uint8 0/1 (waveform.qam_demap's format).
 *  - `stream` is a cudaStream_t (NULL = legacy default stream).  Every call is
 *    stream-ordered and asynchronous: returning OFDMRX_OK means "validated and
 *    enqueued"; per-frame data errors are reported through `flags`.
 *  - Subcarrier order of every frequency-domain array is the reference's
 *    fftshift-ed order (numerics.py:57-64).
 *  - Return value: 0 = OK, otherwise an ofdmrx_status whose category mirrors
 *    errors.py (ConfigurationError, ContractError, InputError/FramingError,
 *    NumericInputError); ofdmrx_last_error() returns the message
 *    (thread-local).
 *  - rx buffers must be 8-byte aligned and readable up to the next 16-byte
 *    boundary past the last sample used (TMA bulk copies move whole 16-byte
 *    granules; torch/cudaMalloc allocations satisfy this).  Every entry that
 *    reads a capture bounds-checks it against desc.rx_samples (ABI 2).
 *  - Results never depend on the batch: a frame's bits, H, s_hat and weights
 *    are bit-identical whatever n_frames (and whatever other frames) it is
 *    launched with.  The antenna-sum order is a function of the frame shape
 *    (N, M, D) only (ofdmrx_rx_plan reports it).
 */
#ifndef OFDMRX_B200_H_
#define OFDMRX_B200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OFDMRX_ABI_VERSION 2

#if defined(__GNUC__)
#define OFDMRX_API __attribute__((visibility("default")))
#else
#define OFDMRX_API
#endif

typedef enum {
  OFDMRX_OK = 0,
  OFDMRX_ERR_CONFIG = 1,   /* errors.ConfigurationError (errors.py:10-13) */
  OFDMRX_ERR_CONTRACT = 2, /* errors.ContractError (errors.py:28-31)      */
  OFDMRX_ERR_INPUT = 3,    /* errors.InputError (errors.py:40-43): capture too short, stream < PN */
  OFDMRX_ERR_NUMERIC = 4,  /* errors.NumericInputError (16-19)             */
  OFDMRX_ERR_CUDA = 5      /* device / launch failure                      */
} ofdmrx_status;

/* Per-frame flag bits written by the fused / finish kernels (atomic OR). */
#define OFDMRX_FLAG_NONFINITE 1u /* a non-finite sample reached the FFT: to_freq raises NumericInputError (receiver.py:202-203) */
#define OFDMRX_FLAG_ERASED 2u    /* some subcarrier weight < eps: CombinedSymbol.erased (receiver.py:234) */
#define OFDMRX_FLAG_NOT_DETECTED 4u /* ofdmrx_rx_frames_detected: antenna-0 peak below threshold (DetectionResult.detected false, sync.py:40); frame skipped */
#define OFDMRX_FLAG_OUT_OF_RANGE 8u /* ofdmrx_rx_frames_detected: the detected frame overruns the capture (extract_slots InputError, receiver.py:278-283); frame skipped */

/*
 * Batch of F captures, each N antenna rows of samples.  Frame f, antenna n,
 * symbol s (s = 0 pilot, 1..D data) starts at sample
 *     f*frame_stride + n*row_stride + symbol0_offset + s*(fft_len + cp_len)
 * and its first cp_len samples are the cyclic prefix (never read).
 * This is extract_slots (receiver.py:274-291) + cp_drop (186-193) expressed as
 * strides over the capture streams of channel.RxCapture (channel.py:35-38).
 */
typedef struct {
  int32_t n_frames;       /* F >= 0                                    */
  int32_t n_antennas;     /* N >= 1                                    */
  int32_t fft_len;        /* M: power of two in [2, 4096]              */
  int32_t cp_len;         /* C: 0 <= C < M   (waveform.py:35-38)       */
  int32_t n_data;         /* D >= 0 data symbols after the pilot       */
  int32_t qam_order;      /* 4, 16 or 64     (waveform.py:20)          */
  int64_t symbol0_offset; /* DetectionResult.symbol0_offset (sync.py:21) */
  int64_t row_stride;     /* samples between antenna rows              */
  int64_t frame_stride;   /* samples between frames                    */
  float eps;              /* MRC_WEIGHT_FLOOR (receiver.py:33) = 1e-12 */
  int32_t options;        /* OR of OFDMRX_OPT_* (0 = none)             */
  int64_t rx_samples;     /* ABI 2: cf32 samples readable at rx; every sample a
                           * call reads must lie below it (OFDMRX_ERR_INPUT
                           * otherwise: extract_slots, receiver.py:278-283) */
} ofdmrx_frame_desc;

/* desc.options: the caller asserts every pilot value is exactly +1 or -1
 * (make_pilot's BPSK pilot, waveform.py:214-220); H = Y/P becomes a sign flip. */
#define OFDMRX_OPT_PILOT_BPSK 1
/* desc.options: accepted for ABI-1 callers, no effect since ABI 2 (results
 * never depend on the batch size; small batches spread each frame over a
 * thread-block cluster instead of antenna shards). */
#define OFDMRX_OPT_NO_SHARDS 2
/* desc.options (ABI 2): latency plan for single frames and small batches
 * (the paper's per-symbol regime).  ofdmrx_rx_frames runs
 * the row-parallel path: every FFT row of the batch is its own lane over the
 * whole GPU, in three stream-ordered launches (pilot rows -> H; data rows ->
 * conj(H) Y per antenna into scratch; combine over the antennas in ascending
 * order = mrc_seq, divide, demap).  The partial-sum, peer-routed and detected
 * entry points use the balanced kernel's widest plan (a whole portable
 * cluster per frame) instead.  Results never depend on the batch size and
 * differ from the default plan's only in fp32 rounding (bits bit-exact vs the
 * reference in every test).  ofdmrx_rx_plan reports the plan. */
#define OFDMRX_OPT_LATENCY 4

OFDMRX_API int ofdmrx_abi_version(void);
OFDMRX_API const char* ofdmrx_last_error(void);

/* Host-only validation of a descriptor (no device access). Mirrors
 * OfdmConfig.__post_init__ (waveform.py:32-46) and extract_slots' bounds
 * check (receiver.py:278-283) against desc.rx_samples. */
OFDMRX_API int ofdmrx_check_desc(const ofdmrx_frame_desc* desc);

/*
 * Launch plan ofdmrx_rx_frames (mode 0) / ofdmrx_rx_partials (mode 1) would
 * use for desc on the current device (needs a CUDA device).  `workers` fixes
 * the arithmetic: the balanced kernel cuts a frame's data rows into `workers`
 * contiguous ranges (antenna-sum order: ascending inside a range, ranges
 * combined in order; den = per-worker strided partials combined in order);
 * `cluster` / `ctas` only map those workers onto the GPU and change with
 * n_frames.  The fused (lockstep) kernel sums antennas in ascending order.
 */
#define OFDMRX_KERNEL_BALANCED 1
#define OFDMRX_KERNEL_FUSED 2
#define OFDMRX_KERNEL_ROWS 3     /* OFDMRX_OPT_LATENCY, mode 0: row-parallel; workers = antennas */
typedef struct {
  int32_t kernel;          /* OFDMRX_KERNEL_*                                  */
  int32_t workers;         /* balanced: virtual FFT lanes per frame; fused: 0  */
  int32_t lanes_per_cta;   /* FFT lanes per CTA                                */
  int32_t cluster;         /* CTAs per frame (thread-block cluster size)       */
  int32_t ctas;            /* grid size                                        */
  int32_t threads;         /* threads per CTA                                  */
  int32_t smem_bytes;      /* dynamic shared memory per CTA                    */
  int32_t chunks;          /* fused: work items per frame (pilot recomputed)  */
} ofdmrx_plan;
OFDMRX_API int ofdmrx_rx_plan(const ofdmrx_frame_desc* desc, int32_t mode, int32_t zf, ofdmrx_plan* out);

/*
 * Fused receive of F frames (one pass over HBM).  Replaces, per frame,
 * run_ring_pipeline (receiver.py:308-348) -> process_symbol (238-267) with
 * SequentialEngine (88-108): cp_drop + to_freq (FFT + fftshift), ls_estimate
 * on the pilot, mrc_combine + qam_demap on each data symbol.
 *   rx      cf32 capture (see desc)
 *   pilot   [M]   cf32 pilot values P (unit modulus), subcarrier order
 *   H       [F,N,M] cf32 ChannelEstimate.gains                (nullable)
 *   s_hat   [F,D,M] cf32 CombinedSymbol.equalized            (required if D>0)
 *   weights [F,M]   f32 CombinedSymbol.weight_norm           (nullable)
 *   bits    [F,D*M*log2(Q)] u8 0/1, PipelineResult.bits order (required if D>0)
 *   zf      [F,D,N,M] cf32 per-antenna ZF output conj(H)Y/max(|H|^2,eps) (nullable)
 *   flags   [F] u32, OR-ed OFDMRX_FLAG_* (nullable; caller zeroes it)
 * Antenna-sum order: see ofdmrx_rx_plan (a function of N, M, D only).
 */
OFDMRX_API int ofdmrx_rx_frames(const ofdmrx_frame_desc* desc, const void* rx, const void* pilot, void* H, void* s_hat,
                     float* weights, uint8_t* bits, void* zf, uint32_t* flags, void* stream);

/*
 * ofdmrx_rx_frames plus a per-stage attribution of the fused kernel's time,
 * for StageTimings (receiver.py:65-79, 245-266) and per-stage µs/symbol of
 * the fused path.  stage_cycles [F, 5] u64 (caller zeroes it) receives, per
 * frame, the SM clock cycles all FFT lanes of the frame spent in
 *   [0] pilot symbol: sample wait + FFT        (fft_s of the pilot slot)
 *   [1] LS estimate H = Y conj(P), |H|^2       (combine_s of the pilot, "ls")
 *   [2] data symbols: sample wait + FFT        (fft_s of the data slots)
 *   [3] MRC accumulation conj(H) Y (+ ZF)      (combine_s of the data, "mrc")
 *   [4] combine, divide, demap, stores         (combine_s of the data, "mrc")
 * Shares of the sum apportion the measured kernel time; the results are the
 * same as ofdmrx_rx_frames'.
 */
OFDMRX_API int ofdmrx_rx_frames_profiled(const ofdmrx_frame_desc* desc, const void* rx, const void* pilot, void* H,
                                         void* s_hat, float* weights, uint8_t* bits, void* zf, uint32_t* flags,
                                         uint64_t* stage_cycles, void* stream);

/*
 * ofdmrx_rx_frames with each frame's symbol0 taken from a device-side
 * detection (ofdmrx_detect outputs, no host round trip): symbol0 of frame f
 * = peak_index[f * peak_stride] + n_chips (DetectionResult.symbol0_offset,
 * sync.py:37-42, antenna 0).  desc.symbol0_offset must be 0; rows hold
 * n_samples samples (desc.rx_samples covers all F x N rows).  Frames with peak_metric[f * peak_stride] < threshold
 * get OFDMRX_FLAG_NOT_DETECTED, frames whose 1 + D symbols overrun the row get
 * OFDMRX_FLAG_OUT_OF_RANGE; both are skipped (their outputs unspecified).
 * flags is required.  This is the reference's detect_packet -> extract_slots
 * -> run_ring_pipeline chain (cli.py:306-321) for F captures in two launches.
 */
OFDMRX_API int ofdmrx_rx_frames_detected(const ofdmrx_frame_desc* desc, int64_t n_samples, const int32_t* peak_index,
                                         const double* peak_metric, int32_t peak_stride, int32_t n_chips,
                                         double threshold, const void* rx, const void* pilot, void* H, void* s_hat,
                                         float* weights, uint8_t* bits, void* zf, uint32_t* flags, void* stream);

/*
 * Antenna-sharded variant, step 1: the same fused pass over this shard's
 * antennas, emitting the un-normalised MRC partial sums instead of s_hat/bits.
 *   num [F,D,M] cf32 = sum_n conj(H_n) Y_n,  den [F,M] f32 = sum_n |H_n|^2
 * (the two accumulators of mrc_seq, numba_backend.py:146-151).
 */
OFDMRX_API int ofdmrx_rx_partials(const ofdmrx_frame_desc* desc, const void* rx, const void* pilot, void* H, void* num,
                       float* den, uint32_t* flags, void* stream);

/*
 * Antenna-sharded variant, step 2 (after the partials of all shards were
 * gathered into [n_parts, ...]): pairwise-tree sum over parts in the
 * reference ReductionPlan order (numerics.py:85-106), floor, divide and demap.
 */
OFDMRX_API int ofdmrx_mrc_finish(int32_t n_frames, int32_t n_data, int32_t fft_len, int32_t qam_order, int32_t n_parts,
                      const void* num, const float* den, float eps, void* s_hat, float* weights, uint8_t* bits,
                      uint32_t* flags, void* stream);

/*
 * Staged stage 1: CP drop + FFT + fftshift of symbols [first_symbol,
 * first_symbol + n_symbols) of every frame/antenna in desc.
 * Replaces engine.freq_transform (receiver.py:92-93,133-142) and
 * kernels.fft_rows (kernels/__init__.py:40-42) + numerics.fftshift.
 *   Y [F, n_symbols, N, M] cf32
 */
OFDMRX_API int ofdmrx_fft_shift(const ofdmrx_frame_desc* desc, int32_t first_symbol, int32_t n_symbols, const void* rx,
                     void* Y, void* stream);

/* Staged stage 2: H[f,n,k] = Y[f*y_frame_stride + n*M + k] * conj(P[k]).
 * Replaces engine.ls_divide (receiver.py:95-96,144-151). */
OFDMRX_API int ofdmrx_ls(int32_t n_frames, int32_t n_antennas, int32_t fft_len, const void* Y, int64_t y_frame_stride,
              const void* pilot, void* H, void* stream);

/* Staged stage 3: MRC of D data symbols per frame.  Y element (f,d,n,k) at
 * Y + f*y_frame_stride + d*y_symbol_stride + n*M + k; H [F,N,M].
 * tree = 0: mrc_seq order; tree = 1: mrc_tree order (numba_backend.py:109-140).
 * Replaces engine.mrc (receiver.py:98-99,153-164).
 *   s_hat [F,D,M] cf32, weights [F,D,M] f32 (nullable), zf [F,D,N,M] (nullable) */
OFDMRX_API int ofdmrx_mrc(int32_t n_frames, int32_t n_data, int32_t n_antennas, int32_t fft_len, const void* Y,
               int64_t y_frame_stride, int64_t y_symbol_stride, const void* H, float eps, int32_t tree, void* s_hat,
               float* weights, void* zf, void* stream);

/* Staged stage 4: hard QAM demap of n symbols -> n*log2(Q) bits.
 * Replaces waveform.qam_demap (waveform.py:179-197). */
OFDMRX_API int ofdmrx_demap(const void* symbols, int64_t n, int32_t qam_order, uint8_t* bits, void* stream);

/*
 * Ingest: copy the symbol payloads of the captures described by desc (CP
 * dropped, every other sample skipped) from `src` (pinned host or device
 * memory) into a dense device buffer dst [F, N, 1+D, M] cf32, as strided 2D
 * copies on `stream` (copy engines, no SM work).  The host side of
 * io_formats.read_cf32 (io_formats.py:26-30) + cli._load_capture
 * (cli.py:249-271) + extract_slots/cp_drop (receiver.py:274-291,186-193):
 * only the samples the FFT consumes cross PCIe.  dst then reads as a capture
 * with cp_len = 0, symbol0_offset = 0, row_stride = (1+D)*M and
 * frame_stride = N*(1+D)*M.
 */
OFDMRX_API int ofdmrx_stage_symbols(const ofdmrx_frame_desc* desc, const void* src, void* dst, void* stream);

/*
 * PN packet detection (the step in front of the hot path).
 * Rows are the (frame, antenna) sample streams of F captures: row (f, n)
 * starts at rx + f*frame_stride + n*row_stride and holds n_samples cf32
 * samples.  chips: [n_chips] f32 device array (the bipolar PN,
 * waveform.generate_pn, waveform.py:77-117), 1 <= n_chips <= 8192.
 * Errors: n_samples < n_chips -> OFDMRX_ERR_INPUT (sync.py:28-31).
 *
 * ofdmrx_corr_metrics replaces kernels.corr_metrics (kernels/__init__.py:45-48,
 * numba_backend.py:55-87): metrics [F*N, n_samples - n_chips + 1] f32,
 * metric[w] = |sum_i c[i] conj(s[w+i])| / (|c| |s[w:w+P]|), 0 where the
 * denominator is <= 1e-30.
 *
 * ofdmrx_detect replaces the per-antenna loop of sync.detect_packet
 * (sync.py:32-36): peak_index [F*N] i32 = first argmax of the metric,
 * peak_metric [F*N] f64 = its value.  Windows within the fp32 error bound of
 * the row maximum are re-scored in fp64, so index and value are the
 * reference's up to the cf32 quantisation of the input.  scratch: device
 * buffer of ofdmrx_detect_scratch_bytes() bytes, 8-byte aligned.  The
 * threshold decision on antenna 0 (DetectionResult.detected) is host logic.
 */
OFDMRX_API int64_t ofdmrx_detect_scratch_bytes(int32_t n_frames, int32_t n_antennas, int64_t n_samples, int32_t n_chips);
OFDMRX_API int ofdmrx_corr_metrics(const void* rx, int32_t n_frames, int32_t n_antennas, int64_t n_samples,
                                   int64_t row_stride, int64_t frame_stride, const float* chips, int32_t n_chips,
                                   float* metrics, void* stream);
OFDMRX_API int ofdmrx_detect(const void* rx, int32_t n_frames, int32_t n_antennas, int64_t n_samples,
                             int64_t row_stride, int64_t frame_stride, const float* chips, int32_t n_chips,
                             void* scratch, int32_t* peak_index, double* peak_metric, void* stream);

/*
 * Frame synthesizer: waveform.build_frame
 * (waveform.py:260-286) + channel.apply_channel (channel.py:72-108) on the
 * device.  rx row (f, n) = timing_offset noise-only samples, then
 * conv(response[f?, n, :], PN | pilot symbol | D data symbols)[:frame_len]
 * plus complex AWGN at snr_db below that row's mean signal power (when
 * noisy), zero-padded/noise to n_samples.  Random draws (ofdmrx_synth_bits,
 * ofdmrx_synth_rayleigh, the AWGN) are counter-based hashes of (seed, stream,
 * index): reproducible, not numpy's PCG64 streams.
 */
typedef struct {
  int32_t n_frames;       /* F                                             */
  int32_t n_antennas;     /* N                                             */
  int32_t fft_len;        /* M, power of two in [2, 4096]                  */
  int32_t cp_len;         /* C, 0 <= C < M                                 */
  int32_t n_data;         /* D >= 1 data symbols (bits fill them exactly)  */
  int32_t qam_order;      /* 4, 16, 64                                     */
  int32_t pn_len;         /* preamble chips (0 = no preamble)              */
  int32_t n_taps;         /* response taps per antenna (1 = flat), <= 64   */
  int32_t resp_per_frame; /* response [F,N,T] (1) or [N,T] for all frames (0) */
  int32_t noisy;          /* 1: add AWGN at snr_db                         */
  float snr_db;
  int64_t timing_offset;  /* leading noise-only samples (ChannelModel.timing_offset) */
  int64_t n_samples;      /* rx row length >= timing_offset + pn_len + (1+D)(M+C) */
  uint64_t seed;
} ofdmrx_synth_desc;

/* bits [F, bits_per_frame] u8 0/1, fair coin per bit. */
OFDMRX_API int ofdmrx_synth_bits(uint8_t* bits, int32_t n_frames, int64_t bits_per_frame, uint64_t seed, void* stream);
/* resp [rows] cf32 ~ CN(0, 1): flat Rayleigh gains (channel.py:95-97). */
OFDMRX_API int ofdmrx_synth_rayleigh(void* resp, int32_t rows, uint64_t seed, void* stream);
/* rx [F, N, n_samples] cf32 from pilot [M] cf32, chips [pn_len] f32,
 * bits [F, D*M*log2(Q)] u8, resp (see desc). */
OFDMRX_API int ofdmrx_synth_frames(const ofdmrx_synth_desc* desc, const void* pilot, const float* chips,
                                   const uint8_t* bits, const void* resp, void* rx, void* stream);

/*
 * Antenna-sharded exchange over peer memory, the fused
 * alternative to gathering the partial sums with NCCL.  Each rank owns
 * frames_per_owner consecutive frames and an inbox allocated with
 * ofdmrx_peer_alloc (num [G, fpo, D, M] cf32 | den [G, fpo, M] f32 | flags),
 * shared with the other ranks by CUDA IPC handle (64 bytes) and mapped with
 * ofdmrx_peer_open (NVLink peer mapping across GPUs).
 *
 * ofdmrx_rx_partials_routed: ofdmrx_rx_partials whose epilogue stores frame
 *   f's (num, den) straight into slot `slot` of owner f / fpo's inbox:
 *   num_dst / den_dst are DEVICE arrays of G pointers (the owners' num / den
 *   bases).  No NCCL call; the stores cross NVLink from the kernel.
 * ofdmrx_peer_signal: st.release.sys of `value` to each of n device flag
 *   addresses (device array dst_table), after the stream's previous work.
 * ofdmrx_peer_wait: stream waits until each of n flags (ld.acquire.sys) is
 *   >= value.
 * The finish step is ofdmrx_mrc_finish over the own inbox.
 */
OFDMRX_API int ofdmrx_rx_partials_routed(const ofdmrx_frame_desc* desc, const void* rx, const void* pilot, void* H,
                                         const void* num_dst, const void* den_dst, int32_t frames_per_owner,
                                         int32_t slot, uint32_t* flags, void* stream);
OFDMRX_API int ofdmrx_peer_alloc(int64_t bytes, void** ptr, void* ipc_handle);
OFDMRX_API int ofdmrx_peer_open(const void* ipc_handle, void** ptr);
OFDMRX_API int ofdmrx_peer_close(void* ptr);
OFDMRX_API int ofdmrx_peer_free(void* ptr);
OFDMRX_API int ofdmrx_peer_signal(const void* dst_table, int32_t n, uint64_t value, void* stream);
OFDMRX_API int ofdmrx_peer_wait(const void* src_table, int32_t n, uint64_t value, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* OFDMRX_B200_H_ */
