// extern "C" boundary of libofdmrx_b200.so (declared in include/ofdmrx_b200.h).
// Validation mirrors the reference's Python-side checks so the host mirror can
// map status codes 1:1 onto the errors.py taxonomy.
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>

#include "../../include/ofdmrx_b200.h"
#include "ofdmrx_internal.h"

namespace {

thread_local std::string g_last_error;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  // consume the runtime's last-error slot: a reported (non-sticky) launch
  // failure must not resurface as the status of the next call's launch
  (void)cudaGetLastError();
  return fail(OFDMRX_ERR_CUDA, "%s: %s (%s)", where, cudaGetErrorString(e), cudaGetErrorName(e));
}

bool is_pow2(long long x) { return x >= 1 && (x & (x - 1)) == 0; }

int qam_bits(int order) { return order == 4 ? 2 : order == 16 ? 4 : order == 64 ? 6 : 0; }

// waveform._build_constellation (waveform.py:138-151): scale = 1/sqrt(2*mean((L-1-2i)^2))
void qam_consts(int order, int* qb, int* levels, float* scale) {
  *qb = qam_bits(order);
  *levels = 1 << (*qb / 2);
  double acc = 0.0;
  for (int i = 0; i < *levels; ++i) {
    const double a = (*levels - 1) - 2.0 * i;
    acc += a * a;
  }
  *scale = (float)(1.0 / std::sqrt(2.0 * (acc / *levels)));
}

int check_fft_len(long long m) {
  if (m < 2 || !is_pow2(m))
    return fail(OFDMRX_ERR_CONFIG, "fft length must be a power of two >= 2, got %lld", m);
  if (m > 4096) return fail(OFDMRX_ERR_CONFIG, "fft length %lld exceeds the device path limit 4096", m);
  return OFDMRX_OK;
}

int check_qam(int order) {
  if (qam_bits(order) == 0) return fail(OFDMRX_ERR_CONFIG, "qam order must be one of (4, 16, 64), got %d", order);
  return OFDMRX_OK;
}

// rows_len: samples a row must hold (span of the 1 + D symbols, or the
// detected-capture row length); the whole batch must lie inside rx_samples
int check_desc_impl(const ofdmrx_frame_desc* d, long long rows_len = -1) {
  if (d == nullptr) return fail(OFDMRX_ERR_CONTRACT, "descriptor is NULL");
  if ((d->options & ~(OFDMRX_OPT_PILOT_BPSK | OFDMRX_OPT_NO_SHARDS | OFDMRX_OPT_LATENCY)) != 0)
    return fail(OFDMRX_ERR_CONTRACT, "unknown descriptor options 0x%x", d->options);
  if (int rc = check_fft_len(d->fft_len)) return rc;
  if (d->cp_len < 0 || d->cp_len >= d->fft_len)
    return fail(OFDMRX_ERR_CONFIG, "cp_len must satisfy 0 <= cp_len < fft_len, got %d", d->cp_len);
  if (d->n_antennas < 1) return fail(OFDMRX_ERR_CONFIG, "n_antennas must be >= 1, got %d", d->n_antennas);
  if (int rc = check_qam(d->qam_order)) return rc;
  if (d->n_frames < 0) return fail(OFDMRX_ERR_CONTRACT, "n_frames must be >= 0, got %d", d->n_frames);
  if (d->n_data < 0) return fail(OFDMRX_ERR_CONTRACT, "n_data must be >= 0, got %d", d->n_data);
  if (!(d->eps >= 0.0f) || !std::isfinite(d->eps)) return fail(OFDMRX_ERR_CONFIG, "eps must be finite and >= 0");
  if (d->symbol0_offset < 0 || d->row_stride < 0 || d->frame_stride < 0)
    return fail(OFDMRX_ERR_CONTRACT, "offsets and strides must be >= 0");
  const long long span = d->symbol0_offset + (long long)(1 + d->n_data) * (d->fft_len + d->cp_len);
  if (d->n_antennas > 1 && d->row_stride < span && d->row_stride != 0)
    return fail(OFDMRX_ERR_CONTRACT, "row_stride %lld shorter than the %lld samples a row needs",
                (long long)d->row_stride, span);
  if (d->rx_samples < 0) return fail(OFDMRX_ERR_CONTRACT, "rx_samples must be >= 0");
  if (d->n_frames > 0) {
    const long long row = rows_len >= 0 ? rows_len : span;
    const long long last = (long long)(d->n_frames - 1) * d->frame_stride +
                           (long long)(d->n_antennas - 1) * d->row_stride + row;
    if (last > d->rx_samples)
      return fail(OFDMRX_ERR_INPUT, "capture has %lld samples, %lld needed for %d symbols at offset %lld",
                  (long long)d->rx_samples, last, 1 + d->n_data, (long long)d->symbol0_offset);
  }
  return OFDMRX_OK;
}

int check_ptr(const void* p, const char* what) {
  if (p == nullptr) return fail(OFDMRX_ERR_CONTRACT, "%s is NULL", what);
  return OFDMRX_OK;
}

int check_align(const void* p, unsigned a, const char* what) {
  if ((reinterpret_cast<uintptr_t>(p) & (a - 1)) != 0)
    return fail(OFDMRX_ERR_CONTRACT, "%s must be %u-byte aligned", what, a);
  return OFDMRX_OK;
}

// stream-ordered scratch from the device's default pool, kept warm
int scratch_alloc(void** ptr, size_t bytes, cudaStream_t st) {
  // a private pool per device (the process-wide default pool keeps its own
  // release threshold); scratch stays mapped between calls
  static cudaMemPool_t pools[32] = {};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  if (dev < 32 && pools[dev] == nullptr) {
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    cudaMemPool_t pool;
    if (cudaMemPoolCreate(&pool, &props) == cudaSuccess) {
      uint64_t keep = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
      pools[dev] = pool;
    }
  }
  e = dev < 32 && pools[dev] != nullptr ? cudaMallocFromPoolAsync(ptr, bytes, pools[dev], st)
                                        : cudaMallocAsync(ptr, bytes, st);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMallocAsync (scratch)");
  return OFDMRX_OK;
}

struct Detected {  // per-frame symbol0 from ofdmrx_detect outputs
  const int32_t* idx;
  const double* metric;
  int stride, add;
  double threshold;
  long long n_samples;
};

struct Route {  // partial sums routed to the owners' peer inboxes
  const void* num_dst;
  const void* den_dst;
  int fpo, slot;
};

// Kernel choice and launch geometry for one fused call.  Everything that
// fixes the arithmetic (balanced vs fused kernel, the balanced kernel's
// worker count, the fused kernel's chunking) depends on the frame shape only;
// n_frames only changes how the work is mapped onto CTAs.
struct RxPlan {
  bool rows;  // row-parallel latency path
  bool balanced;
  ofdmrx::BalancedPlan bp;
  ofdmrx::FusedLaunch fl;
};

// rows_ok: the call can take the row-parallel path (mode 0, fixed symbol0, no routes)
int make_plan(const ofdmrx_frame_desc* d, RxPlan* pl, bool rows_ok = false) {
  *pl = RxPlan{};
  pl->rows = rows_ok && (d->options & OFDMRX_OPT_LATENCY) != 0;
  if (pl->rows) return OFDMRX_OK;
  pl->balanced = ofdmrx::balanced_plan(d->fft_len, d->n_antennas, d->n_data, d->n_frames,
                                        ofdmrx::device_sm_count(), (d->options & OFDMRX_OPT_LATENCY) != 0,
                                        &pl->bp);
  if (!pl->balanced) {
    if (ofdmrx::fused_plan(d->fft_len, d->n_frames, d->n_data, &pl->fl) != cudaSuccess)
      return fail(OFDMRX_ERR_CONFIG, "no launch plan for fft_len %d", d->fft_len);
  }
  return OFDMRX_OK;
}

int fused_common(const ofdmrx_frame_desc* d, const void* rx, const void* pilot, int mode, void* H, void* s_hat,
                 float* weights, uint8_t* bits, void* zf, uint32_t* flags, void* num, float* den, void* stream,
                 const Route* route = nullptr, const Detected* det = nullptr,
                 unsigned long long* stage_cycles = nullptr) {
  if (int rc = check_desc_impl(d, det != nullptr ? det->n_samples : -1)) return rc;
  if (d->n_frames == 0) return OFDMRX_OK;
  if (int rc = check_ptr(rx, "rx")) return rc;
  if (int rc = check_align(rx, 8, "rx")) return rc;
  if (int rc = check_ptr(pilot, "pilot")) return rc;
  if (mode == 0 && d->n_data > 0) {
    if (int rc = check_ptr(s_hat, "s_hat")) return rc;
    if (int rc = check_ptr(bits, "bits")) return rc;
    if (int rc = check_align(bits, 4, "bits")) return rc;
  }
  if (mode == 1 && route == nullptr) {
    if (d->n_data > 0)
      if (int rc = check_ptr(num, "num")) return rc;
    if (int rc = check_ptr(den, "den")) return rc;
  }
  if (route != nullptr) {
    if (int rc = check_ptr(route->num_dst, "num_dst")) return rc;
    if (int rc = check_ptr(route->den_dst, "den_dst")) return rc;
    if (route->fpo < 1 || d->n_frames % route->fpo != 0)
      return fail(OFDMRX_ERR_CONTRACT, "n_frames %d is not a multiple of frames_per_owner %d", d->n_frames, route->fpo);
    if (route->slot < 0) return fail(OFDMRX_ERR_CONTRACT, "slot must be >= 0");
  }
  RxPlan pl;
  if (int rc = make_plan(d, &pl, mode == 0 && route == nullptr && det == nullptr)) return rc;
  ofdmrx::FusedParams p{};
  p.rx = static_cast<const float2*>(rx);
  p.frame_stride = d->frame_stride;
  p.row_stride = d->row_stride;
  p.sym0 = d->symbol0_offset;
  p.n_frames = d->n_frames;
  p.n_ant = d->n_antennas;
  p.ant_total = d->n_antennas;
  p.n_shards = 1;
  p.cp = d->cp_len;
  p.n_data = d->n_data;
  p.dc = pl.fl.dc;
  p.n_chunks = pl.fl.n_chunks;
  p.fpb = pl.fl.fpb;
  p.n_work = d->n_frames * pl.fl.n_chunks;
  p.lanes = pl.fl.lanes;
  p.ngroups = pl.fl.ngroups;
  p.npilot = pl.fl.npilot;
  p.pilot = static_cast<const float2*>(pilot);
  p.eps = d->eps;
  qam_consts(d->qam_order, &p.qb, &p.levels, &p.qscale);
  p.mode = mode;
  p.pilot_bpsk = (d->options & OFDMRX_OPT_PILOT_BPSK) != 0;
  p.H = static_cast<float2*>(H);
  p.s_hat = static_cast<float2*>(s_hat);
  p.weights = weights;
  p.bits = bits;
  p.zf = static_cast<float2*>(zf);
  p.flags = flags;
  p.part_num = static_cast<float2*>(num);
  p.part_den = den;
  p.stage_cycles = stage_cycles;
  if (det != nullptr) {
    p.det_idx = det->idx;
    p.det_metric = det->metric;
    p.det_stride = det->stride;
    p.det_add = det->add;
    p.det_threshold = det->threshold;
    p.n_samples = det->n_samples;
  }
  if (route != nullptr) {
    p.num_dst = static_cast<float2* const*>(route->num_dst);
    p.den_dst = static_cast<float* const*>(route->den_dst);
    p.fpo = route->fpo;
    p.slot = route->slot;
  }
  const cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e;
  if (pl.rows) {
    void* hscratch = nullptr;
    void* prod = nullptr;
    if (p.H == nullptr) {
      if (int rc = scratch_alloc(&hscratch, (size_t)d->n_frames * d->n_antennas * d->fft_len * 8, st)) return rc;
      p.H = static_cast<float2*>(hscratch);
    }
    // the per-antenna products of at most ~1 GB of frames at a time (the
    // frames are independent: chunking changes no result)
    const size_t per_frame = ofdmrx::latency_scratch_bytes(1, d->n_antennas, d->n_data, d->fft_len);
    int chunk = d->n_frames;
    if (per_frame > 0 && (size_t)chunk * per_frame > (1ull << 30)) {
      chunk = (int)((1ull << 30) / per_frame);
      if (chunk < 1) chunk = 1;
    }
    if (per_frame > 0) {
      if (int rc = scratch_alloc(&prod, (size_t)chunk * per_frame, st)) {
        if (hscratch != nullptr) cudaFreeAsync(hscratch, st);
        return rc;
      }
    }
    e = cudaSuccess;
    for (int f0 = 0; f0 < d->n_frames && e == cudaSuccess; f0 += chunk) {
      ofdmrx::FusedParams q = p;
      const int fc = d->n_frames - f0 < chunk ? d->n_frames - f0 : chunk;
      const long long M = d->fft_len, D = d->n_data, N = d->n_antennas;
      q.n_frames = fc;
      q.rx = p.rx + (long long)f0 * d->frame_stride;
      q.H = p.H + (long long)f0 * N * M;
      q.s_hat = p.s_hat != nullptr ? p.s_hat + (long long)f0 * D * M : nullptr;
      q.weights = p.weights != nullptr ? p.weights + (long long)f0 * M : nullptr;
      q.bits = p.bits != nullptr ? p.bits + (long long)f0 * D * M * p.qb : nullptr;
      q.zf = p.zf != nullptr ? p.zf + (long long)f0 * D * N * M : nullptr;
      q.flags = p.flags != nullptr ? p.flags + f0 : nullptr;
      q.stage_cycles = p.stage_cycles != nullptr ? p.stage_cycles + (long long)f0 * ofdmrx::kStages : nullptr;
      e = ofdmrx::launch_latency(d->fft_len, q, static_cast<float2*>(prod), st);
    }
    cudaError_t e2 = prod != nullptr ? cudaFreeAsync(prod, st) : cudaSuccess;
    cudaError_t e3 = hscratch != nullptr ? cudaFreeAsync(hscratch, st) : cudaSuccess;
    if (e != cudaSuccess) return cuda_fail(e, "row-parallel receive launch");
    if (e2 != cudaSuccess) return cuda_fail(e2, "cudaFreeAsync");
    if (e3 != cudaSuccess) return cuda_fail(e3, "cudaFreeAsync");
    return OFDMRX_OK;
  }
  if (pl.balanced) {
    void* hscratch = nullptr;
    if (p.H == nullptr) {  // H travels through L2 between the phases: scratch when the caller wants none
      if (int rc = scratch_alloc(&hscratch, (size_t)d->n_frames * d->n_antennas * d->fft_len * 8, st)) return rc;
      p.H = static_cast<float2*>(hscratch);
    }
    e = ofdmrx::launch_balanced(d->fft_len, p, pl.bp, st);
    cudaError_t e2 = hscratch != nullptr ? cudaFreeAsync(hscratch, st) : cudaSuccess;
    if (e != cudaSuccess) return cuda_fail(e, "rx_balanced_kernel launch");
    if (e2 != cudaSuccess) return cuda_fail(e2, "cudaFreeAsync");
    return OFDMRX_OK;
  }
  e = ofdmrx::launch_fused(d->fft_len, p, pl.fl, st);
  if (e != cudaSuccess) return cuda_fail(e, "rx_fused_kernel launch");
  return OFDMRX_OK;
}

constexpr int kMaxChips = 8192;

int sync_common(const void* rx, int32_t n_frames, int32_t n_antennas, int64_t n_samples, int64_t row_stride,
                int64_t frame_stride, const float* chips, int32_t n_chips, ofdmrx::SyncParams* p) {
  if (n_frames < 0 || n_antennas < 1) return fail(OFDMRX_ERR_CONTRACT, "n_frames must be >= 0 and n_antennas >= 1");
  if (n_chips < 1 || n_chips > kMaxChips)
    return fail(OFDMRX_ERR_CONFIG, "PN length %d outside the device path's [1, %d]", n_chips, kMaxChips);
  if (n_samples < n_chips)
    return fail(OFDMRX_ERR_INPUT, "stream length %lld shorter than PN length %d", (long long)n_samples, n_chips);
  if (n_samples - n_chips + 1 > 0x7fffffffLL) return fail(OFDMRX_ERR_CONFIG, "stream too long (%lld)", (long long)n_samples);
  if (row_stride < 0 || frame_stride < 0) return fail(OFDMRX_ERR_CONTRACT, "strides must be >= 0");
  if (n_antennas > 1 && row_stride < n_samples && row_stride != 0)
    return fail(OFDMRX_ERR_CONTRACT, "row_stride %lld shorter than n_samples %lld", (long long)row_stride,
                (long long)n_samples);
  if (n_frames > 0) {
    if (int rc = check_ptr(rx, "rx")) return rc;
    if (int rc = check_align(rx, 8, "rx")) return rc;
    if (int rc = check_ptr(chips, "chips")) return rc;
  }
  *p = ofdmrx::SyncParams{};
  p->rx = static_cast<const float2*>(rx);
  p->frame_stride = frame_stride;
  p->row_stride = row_stride;
  p->n_samples = n_samples;
  p->n_frames = n_frames;
  p->n_ant = n_antennas;
  p->chips = chips;
  p->n_chips = n_chips;
  p->wins = n_samples - n_chips + 1;
  return OFDMRX_OK;
}

}  // namespace

namespace ofdmrx {
int device_sm_count() {
  static int counts[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0) return 148;
  if (dev < 64 && counts[dev] > 0) return counts[dev];
  int n = 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) return 148;
  if (dev < 64) counts[dev] = n;
  return n;
}
}  // namespace ofdmrx

extern "C" {

int64_t ofdmrx_detect_scratch_bytes(int32_t n_frames, int32_t n_antennas, int64_t n_samples, int32_t n_chips) {
  if (n_frames < 0 || n_antennas < 1 || n_chips < 1 || n_samples < n_chips) return -1;
  const long long rows = (long long)n_frames * n_antennas;
  // keys [rows] u64 | metrics [rows, wins] f32 | (pad to 16) chip spectrum [1024] cf32
  return ((rows * 8 + rows * (n_samples - n_chips + 1) * 4 + 15) & ~15LL) + (long long)ofdmrx::sync_fft_scratch_bytes();
}

int ofdmrx_corr_metrics(const void* rx, int32_t n_frames, int32_t n_antennas, int64_t n_samples, int64_t row_stride,
                        int64_t frame_stride, const float* chips, int32_t n_chips, float* metrics, void* stream) {
  ofdmrx::SyncParams p;
  if (int rc = sync_common(rx, n_frames, n_antennas, n_samples, row_stride, frame_stride, chips, n_chips, &p))
    return rc;
  if (n_frames == 0) return OFDMRX_OK;
  if (int rc = check_ptr(metrics, "metrics")) return rc;
  p.metrics = metrics;
  // the metric array itself is the product here: the direct fp32 form
  // (error <= 3 P 2^-24) rather than the FFT form detect screens with
  cudaError_t e = ofdmrx::launch_corr(p, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "corr_kernel launch");
  return OFDMRX_OK;
}

int ofdmrx_detect(const void* rx, int32_t n_frames, int32_t n_antennas, int64_t n_samples, int64_t row_stride,
                  int64_t frame_stride, const float* chips, int32_t n_chips, void* scratch, int32_t* peak_index,
                  double* peak_metric, void* stream) {
  ofdmrx::SyncParams p;
  if (int rc = sync_common(rx, n_frames, n_antennas, n_samples, row_stride, frame_stride, chips, n_chips, &p))
    return rc;
  if (n_frames == 0) return OFDMRX_OK;
  if (int rc = check_ptr(scratch, "scratch")) return rc;
  if (int rc = check_align(scratch, 8, "scratch")) return rc;
  if (int rc = check_ptr(peak_index, "peak_index")) return rc;
  if (int rc = check_ptr(peak_metric, "peak_metric")) return rc;
  const long long rows = (long long)n_frames * n_antennas;
  p.keys = static_cast<unsigned long long*>(scratch);
  p.metrics = reinterpret_cast<float*>(static_cast<char*>(scratch) + rows * 8);
  const cudaStream_t s = static_cast<cudaStream_t>(stream);
  const bool fft = ofdmrx::sync_use_fft(n_chips);
  cudaError_t e;
  if (fft) {
    const long long off = (rows * 8 + rows * p.wins * 4 + 15) & ~15LL;
    e = ofdmrx::launch_corr_fft(p, reinterpret_cast<float2*>(static_cast<char*>(scratch) + off), 1, s);
  } else {
    e = ofdmrx::launch_corr(p, s);
  }
  if (e != cudaSuccess) return cuda_fail(e, "corr kernel launch");
  e = ofdmrx::launch_refine(p, peak_index, peak_metric, fft ? 1 : 0, s);
  if (e != cudaSuccess) return cuda_fail(e, "refine_kernel launch");
  return OFDMRX_OK;
}


int ofdmrx_abi_version(void) { return OFDMRX_ABI_VERSION; }

const char* ofdmrx_last_error(void) { return g_last_error.c_str(); }

int ofdmrx_check_desc(const ofdmrx_frame_desc* desc) { return check_desc_impl(desc); }

int ofdmrx_rx_plan(const ofdmrx_frame_desc* desc, int32_t mode, int32_t zf, ofdmrx_plan* out) {
  if (int rc = check_desc_impl(desc)) return rc;
  if (int rc = check_ptr(out, "out")) return rc;
  if (mode != 0 && mode != 1) return fail(OFDMRX_ERR_CONTRACT, "mode must be 0 or 1");
  (void)zf;  // the ZF output changes neither the kernel nor the order
  RxPlan pl;
  if (int rc = make_plan(desc, &pl, mode == 0)) return rc;
  *out = ofdmrx_plan{};
  if (pl.rows) {
    out->kernel = OFDMRX_KERNEL_ROWS;
    out->workers = desc->n_antennas;
    out->lanes_per_cta = 0;
    out->cluster = 1;
    out->ctas = 0;
    out->threads = 256;
    out->smem_bytes = 0;
    out->chunks = 1;
  } else if (pl.balanced) {
    out->kernel = OFDMRX_KERNEL_BALANCED;
    out->workers = pl.bp.workers;
    out->lanes_per_cta = pl.bp.lanes_per_cta;
    out->cluster = pl.bp.cluster;
    out->ctas = desc->n_frames * pl.bp.cluster;
    out->threads = pl.bp.lanes_per_cta * pl.bp.fft_lane_threads;
    out->smem_bytes = (int32_t)ofdmrx::balanced_smem_bytes(desc->fft_len, pl.bp.lanes_per_cta);
    out->chunks = 1;
  } else {
    out->kernel = OFDMRX_KERNEL_FUSED;
    out->workers = 0;
    out->lanes_per_cta = pl.fl.lanes;
    out->cluster = 1;
    out->ctas = pl.fl.grid;
    out->threads = pl.fl.threads;
    out->smem_bytes = (int32_t)pl.fl.smem;
    out->chunks = pl.fl.n_chunks;
  }
  return OFDMRX_OK;
}

int ofdmrx_rx_frames(const ofdmrx_frame_desc* desc, const void* rx, const void* pilot, void* H, void* s_hat,
                     float* weights, uint8_t* bits, void* zf, uint32_t* flags, void* stream) {
  return fused_common(desc, rx, pilot, 0, H, s_hat, weights, bits, zf, flags, nullptr, nullptr, stream);
}

int ofdmrx_rx_frames_profiled(const ofdmrx_frame_desc* desc, const void* rx, const void* pilot, void* H, void* s_hat,
                              float* weights, uint8_t* bits, void* zf, uint32_t* flags, uint64_t* stage_cycles,
                              void* stream) {
  if (desc != nullptr && desc->n_frames > 0)
    if (int rc = check_ptr(stage_cycles, "stage_cycles")) return rc;
  return fused_common(desc, rx, pilot, 0, H, s_hat, weights, bits, zf, flags, nullptr, nullptr, stream, nullptr,
                      nullptr, reinterpret_cast<unsigned long long*>(stage_cycles));
}

int ofdmrx_rx_partials(const ofdmrx_frame_desc* desc, const void* rx, const void* pilot, void* H, void* num,
                       float* den, uint32_t* flags, void* stream) {
  return fused_common(desc, rx, pilot, 1, H, nullptr, nullptr, nullptr, nullptr, flags, num, den, stream);
}

int ofdmrx_rx_frames_detected(const ofdmrx_frame_desc* desc, int64_t n_samples, const int32_t* peak_index,
                              const double* peak_metric, int32_t peak_stride, int32_t n_chips, double threshold,
                              const void* rx, const void* pilot, void* H, void* s_hat, float* weights, uint8_t* bits,
                              void* zf, uint32_t* flags, void* stream) {
  if (desc == nullptr) return fail(OFDMRX_ERR_CONTRACT, "descriptor is NULL");
  if (desc->symbol0_offset != 0)
    return fail(OFDMRX_ERR_CONTRACT, "symbol0_offset must be 0: it comes from peak_index per frame");
  if (n_chips < 0 || peak_stride < 1) return fail(OFDMRX_ERR_CONTRACT, "need n_chips >= 0 and peak_stride >= 1");
  if (n_samples < (long long)(1 + desc->n_data) * (desc->fft_len + desc->cp_len))
    return fail(OFDMRX_ERR_INPUT, "rows of %lld samples cannot hold %d symbols", (long long)n_samples,
                1 + desc->n_data);
  if (desc->n_frames > 0) {
    if (int rc = check_ptr(peak_index, "peak_index")) return rc;
    if (int rc = check_ptr(peak_metric, "peak_metric")) return rc;
    if (int rc = check_ptr(flags, "flags")) return rc;  // rejected frames are only visible here
  }
  const Detected det{peak_index, peak_metric, peak_stride, n_chips, threshold, n_samples};
  return fused_common(desc, rx, pilot, 0, H, s_hat, weights, bits, zf, flags, nullptr, nullptr, stream, nullptr, &det);
}

int ofdmrx_rx_partials_routed(const ofdmrx_frame_desc* desc, const void* rx, const void* pilot, void* H,
                              const void* num_dst, const void* den_dst, int32_t frames_per_owner, int32_t slot,
                              uint32_t* flags, void* stream) {
  const Route r{num_dst, den_dst, frames_per_owner, slot};
  return fused_common(desc, rx, pilot, 1, H, nullptr, nullptr, nullptr, nullptr, flags, nullptr, nullptr, stream, &r);
}

int ofdmrx_peer_alloc(int64_t bytes, void** ptr, void* ipc_handle) {
  if (bytes <= 0) return fail(OFDMRX_ERR_CONTRACT, "bytes must be > 0");
  if (int rc = check_ptr(ptr, "ptr")) return rc;
  if (int rc = check_ptr(ipc_handle, "ipc_handle")) return rc;
  cudaError_t e = cudaMalloc(ptr, (size_t)bytes);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc (peer inbox)");
  if ((e = cudaMemset(*ptr, 0, (size_t)bytes)) != cudaSuccess) return cuda_fail(e, "cudaMemset (peer inbox)");
  cudaIpcMemHandle_t h;
  if ((e = cudaIpcGetMemHandle(&h, *ptr)) != cudaSuccess) return cuda_fail(e, "cudaIpcGetMemHandle");
  memcpy(ipc_handle, &h, sizeof(h));
  return OFDMRX_OK;
}

int ofdmrx_peer_open(const void* ipc_handle, void** ptr) {
  if (int rc = check_ptr(ipc_handle, "ipc_handle")) return rc;
  if (int rc = check_ptr(ptr, "ptr")) return rc;
  cudaIpcMemHandle_t h;
  memcpy(&h, ipc_handle, sizeof(h));
  cudaError_t e = cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return cuda_fail(e, "cudaIpcOpenMemHandle");
  return OFDMRX_OK;
}

int ofdmrx_peer_close(void* ptr) {
  cudaError_t e = cudaIpcCloseMemHandle(ptr);
  return e == cudaSuccess ? OFDMRX_OK : cuda_fail(e, "cudaIpcCloseMemHandle");
}

int ofdmrx_peer_free(void* ptr) {
  cudaError_t e = cudaFree(ptr);
  return e == cudaSuccess ? OFDMRX_OK : cuda_fail(e, "cudaFree (peer inbox)");
}

int ofdmrx_peer_signal(const void* dst_table, int32_t n, uint64_t value, void* stream) {
  if (n < 0) return fail(OFDMRX_ERR_CONTRACT, "n must be >= 0");
  if (n > 0)
    if (int rc = check_ptr(dst_table, "dst_table")) return rc;
  cudaError_t e = ofdmrx::launch_peer_signal(static_cast<unsigned long long* const*>(dst_table), n,
                                             (unsigned long long)value, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? OFDMRX_OK : cuda_fail(e, "peer_signal_kernel launch");
}

int ofdmrx_peer_wait(const void* src_table, int32_t n, uint64_t value, void* stream) {
  if (n < 0) return fail(OFDMRX_ERR_CONTRACT, "n must be >= 0");
  if (n > 0)
    if (int rc = check_ptr(src_table, "src_table")) return rc;
  cudaError_t e = ofdmrx::launch_peer_wait(static_cast<const unsigned long long* const*>(src_table), n,
                                           (unsigned long long)value, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? OFDMRX_OK : cuda_fail(e, "peer_wait_kernel launch");
}

int ofdmrx_mrc_finish(int32_t n_frames, int32_t n_data, int32_t fft_len, int32_t qam_order, int32_t n_parts,
                      const void* num, const float* den, float eps, void* s_hat, float* weights, uint8_t* bits,
                      uint32_t* flags, void* stream) {
  if (int rc = check_fft_len(fft_len)) return rc;
  if (int rc = check_qam(qam_order)) return rc;
  if (n_frames < 0 || n_data < 0) return fail(OFDMRX_ERR_CONTRACT, "n_frames and n_data must be >= 0");
  if (n_parts < 1 || n_parts > 0x7fffffff) return fail(OFDMRX_ERR_CONTRACT, "n_parts must be >= 1");
  if ((long long)n_frames * n_data == 0) return OFDMRX_OK;
  if (int rc = check_ptr(num, "num")) return rc;
  if (int rc = check_ptr(den, "den")) return rc;
  if (int rc = check_ptr(s_hat, "s_hat")) return rc;
  if (int rc = check_ptr(bits, "bits")) return rc;
  ofdmrx::FinishParams p{};
  p.num = static_cast<const float2*>(num);
  p.den = den;
  p.parts = n_parts;
  p.n_frames = n_frames;
  p.n_data = n_data;
  p.M = fft_len;
  p.eps = eps;
  qam_consts(qam_order, &p.qb, &p.levels, &p.qscale);
  p.s_hat = static_cast<float2*>(s_hat);
  p.weights = weights;
  p.bits = bits;
  p.flags = flags;
  cudaError_t e = ofdmrx::launch_finish(p, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "finish_kernel launch");
  return OFDMRX_OK;
}

int ofdmrx_fft_shift(const ofdmrx_frame_desc* desc, int32_t first_symbol, int32_t n_symbols, const void* rx, void* Y,
                     void* stream) {
  if (int rc = check_desc_impl(desc)) return rc;
  if (first_symbol < 0 || n_symbols < 0 || first_symbol + n_symbols > 1 + desc->n_data)
    return fail(OFDMRX_ERR_CONTRACT, "symbol range [%d, %d) outside the frame's %d symbols", first_symbol,
                first_symbol + n_symbols, 1 + desc->n_data);
  if ((long long)desc->n_frames * n_symbols == 0) return OFDMRX_OK;
  if (int rc = check_ptr(rx, "rx")) return rc;
  if (int rc = check_ptr(Y, "Y")) return rc;
  ofdmrx::FftRowsParams p{};
  const long long sym_len = desc->fft_len + desc->cp_len;
  p.src = static_cast<const float2*>(rx);
  p.frame_stride = desc->frame_stride;
  p.row_stride = desc->row_stride;
  p.sym0 = desc->symbol0_offset + (long long)first_symbol * sym_len + desc->cp_len;
  p.sym_stride = sym_len;
  p.n_frames = desc->n_frames;
  p.n_sym = n_symbols;
  p.n_ant = desc->n_antennas;
  p.out = static_cast<float2*>(Y);
  cudaError_t e = ofdmrx::launch_fft_rows(desc->fft_len, p, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "fft_rows_kernel launch");
  return OFDMRX_OK;
}

int ofdmrx_ls(int32_t n_frames, int32_t n_antennas, int32_t fft_len, const void* Y, int64_t y_frame_stride,
              const void* pilot, void* H, void* stream) {
  if (fft_len < 1) return fail(OFDMRX_ERR_CONFIG, "fft_len must be >= 1");
  if (n_frames < 0 || n_antennas < 0) return fail(OFDMRX_ERR_CONTRACT, "negative sizes");
  if ((long long)n_frames * n_antennas == 0) return OFDMRX_OK;
  if (int rc = check_ptr(Y, "Y")) return rc;
  if (int rc = check_ptr(pilot, "pilot")) return rc;
  if (int rc = check_ptr(H, "H")) return rc;
  cudaError_t e = ofdmrx::launch_ls(static_cast<const float2*>(Y), y_frame_stride, n_frames, n_antennas, fft_len,
                                    static_cast<const float2*>(pilot), static_cast<float2*>(H),
                                    static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "ls_kernel launch");
  return OFDMRX_OK;
}

int ofdmrx_mrc(int32_t n_frames, int32_t n_data, int32_t n_antennas, int32_t fft_len, const void* Y,
               int64_t y_frame_stride, int64_t y_symbol_stride, const void* H, float eps, int32_t tree, void* s_hat,
               float* weights, void* zf, void* stream) {
  if (fft_len < 1) return fail(OFDMRX_ERR_CONFIG, "fft_len must be >= 1");
  if (n_frames < 0 || n_data < 0 || n_antennas < 1) return fail(OFDMRX_ERR_CONTRACT, "bad sizes");
  if (tree != 0 && tree != 1) return fail(OFDMRX_ERR_CONFIG, "tree must be 0 or 1");
  if ((long long)n_frames * n_data == 0) return OFDMRX_OK;
  if (int rc = check_ptr(Y, "Y")) return rc;
  if (int rc = check_ptr(H, "H")) return rc;
  if (int rc = check_ptr(s_hat, "s_hat")) return rc;
  ofdmrx::MrcParams p{};
  p.Y = static_cast<const float2*>(Y);
  p.y_fs = y_frame_stride;
  p.y_ss = y_symbol_stride;
  p.H = static_cast<const float2*>(H);
  p.n_frames = n_frames;
  p.n_data = n_data;
  p.n_ant = n_antennas;
  p.M = fft_len;
  p.eps = eps;
  p.tree = tree;
  p.s_hat = static_cast<float2*>(s_hat);
  p.weights = weights;
  p.zf = static_cast<float2*>(zf);
  cudaError_t e = ofdmrx::launch_mrc(p, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "mrc_kernel launch");
  return OFDMRX_OK;
}

int ofdmrx_stage_symbols(const ofdmrx_frame_desc* desc, const void* src, void* dst, void* stream) {
  if (int rc = check_desc_impl(desc)) return rc;
  const long long F = desc->n_frames, N = desc->n_antennas, S = 1 + desc->n_data, M = desc->fft_len;
  if (F == 0) return OFDMRX_OK;
  if (int rc = check_ptr(src, "src")) return rc;
  if (int rc = check_ptr(dst, "dst")) return rc;
  const cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t width = (size_t)M * 8, dpitch = (size_t)S * M * 8;
  const long long sym_len = desc->fft_len + desc->cp_len;
  // one 2D copy per symbol covers every (frame, antenna) row when the rows are
  // uniformly spaced; otherwise one per (frame, symbol)
  long long rows, pitch, groups;
  if (N == 1) {
    rows = F, pitch = desc->frame_stride, groups = 1;
  } else if (F == 1 || desc->frame_stride == N * desc->row_stride) {
    rows = F * N, pitch = desc->row_stride, groups = 1;
  } else {
    rows = N, pitch = desc->row_stride, groups = F;
  }
  if (rows > 1 && pitch < M) rows = 1, groups = F * N;  // overlapping rows: plain copies
  for (long long g = 0; g < groups; ++g) {
    // first row of group g: frame f, antenna a
    const long long f = rows == 1 && groups == F * N ? g / N : (groups == F ? g : 0);
    const long long a = rows == 1 && groups == F * N ? g % N : 0;
    for (long long sy = 0; sy < S; ++sy) {
      const char* sp = static_cast<const char*>(src) +
                       8 * (f * desc->frame_stride + a * desc->row_stride + desc->symbol0_offset + sy * sym_len +
                            desc->cp_len);
      char* dp = static_cast<char*>(dst) + 8 * (((f * N + a) * S + sy) * M);
      cudaError_t e = rows == 1 ? cudaMemcpyAsync(dp, sp, width, cudaMemcpyDefault, s)
                                : cudaMemcpy2DAsync(dp, dpitch, sp, (size_t)pitch * 8, width, (size_t)rows,
                                                    cudaMemcpyDefault, s);
      if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpy2DAsync (stage_symbols)");
    }
  }
  return OFDMRX_OK;
}

int ofdmrx_synth_bits(uint8_t* bits, int32_t n_frames, int64_t bits_per_frame, uint64_t seed, void* stream) {
  if (n_frames < 0 || bits_per_frame < 0) return fail(OFDMRX_ERR_CONTRACT, "negative sizes");
  if ((long long)n_frames * bits_per_frame == 0) return OFDMRX_OK;
  if (int rc = check_ptr(bits, "bits")) return rc;
  cudaError_t e = ofdmrx::launch_synth_bits(bits, bits_per_frame, n_frames, seed, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "bits_kernel launch");
  return OFDMRX_OK;
}

int ofdmrx_synth_rayleigh(void* resp, int32_t rows, uint64_t seed, void* stream) {
  if (rows < 0) return fail(OFDMRX_ERR_CONTRACT, "negative sizes");
  if (rows == 0) return OFDMRX_OK;
  if (int rc = check_ptr(resp, "resp")) return rc;
  cudaError_t e = ofdmrx::launch_synth_gains(static_cast<float2*>(resp), rows, seed, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "gains_kernel launch");
  return OFDMRX_OK;
}

int ofdmrx_synth_frames(const ofdmrx_synth_desc* d, const void* pilot, const float* chips, const uint8_t* bits,
                        const void* resp, void* rx, void* stream) {
  if (d == nullptr) return fail(OFDMRX_ERR_CONTRACT, "descriptor is NULL");
  if (int rc = check_fft_len(d->fft_len)) return rc;
  if (d->cp_len < 0 || d->cp_len >= d->fft_len)
    return fail(OFDMRX_ERR_CONFIG, "cp_len must satisfy 0 <= cp_len < fft_len, got %d", d->cp_len);
  if (int rc = check_qam(d->qam_order)) return rc;
  if (d->n_frames < 0 || d->n_antennas < 1 || d->n_data < 1)
    return fail(OFDMRX_ERR_CONTRACT, "need n_frames >= 0, n_antennas >= 1, n_data >= 1");
  if (d->pn_len < 0 || d->n_taps < 1 || d->n_taps > 64 || d->timing_offset < 0)
    return fail(OFDMRX_ERR_CONFIG, "invalid pn_len / n_taps (1..64) / timing_offset");
  if (!std::isfinite(d->snr_db)) return fail(OFDMRX_ERR_CONFIG, "snr_db must be finite");
  const long long tx_len = (long long)(1 + d->n_data) * (d->fft_len + d->cp_len);
  if (d->n_samples < d->timing_offset + d->pn_len + tx_len)
    return fail(OFDMRX_ERR_CONTRACT, "n_samples %lld < timing_offset + frame length %lld", (long long)d->n_samples,
                (long long)(d->timing_offset + d->pn_len + tx_len));
  if (d->n_frames == 0) return OFDMRX_OK;
  if (int rc = check_ptr(pilot, "pilot")) return rc;
  if (d->pn_len > 0)
    if (int rc = check_ptr(chips, "chips")) return rc;
  if (int rc = check_ptr(bits, "bits")) return rc;
  if (int rc = check_ptr(resp, "resp")) return rc;
  if (int rc = check_ptr(rx, "rx")) return rc;
  ofdmrx::SynthParams p{};
  p.n_frames = d->n_frames;
  p.n_ant = d->n_antennas;
  p.M = d->fft_len;
  p.cp = d->cp_len;
  p.n_data = d->n_data;
  qam_consts(d->qam_order, &p.qb, &p.levels, &p.qscale);
  p.pn_len = d->pn_len;
  p.tx_len = tx_len;
  p.n_samples = d->n_samples;
  p.offset = d->timing_offset;
  p.pilot = static_cast<const float2*>(pilot);
  p.chips = chips;
  p.bits = bits;
  p.resp = static_cast<const float2*>(resp);
  p.n_taps = d->n_taps;
  p.resp_per_frame = d->resp_per_frame != 0;
  p.noisy = d->noisy != 0;
  p.snr_db = d->snr_db;
  p.seed = d->seed;
  p.rx = static_cast<float2*>(rx);
  const cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t parts = ofdmrx::synth_sig_parts(d->pn_len, tx_len);
  const size_t tx_bytes = (size_t)d->n_frames * tx_len * 8;
  const size_t sig_bytes = (size_t)d->n_frames * d->n_antennas * parts * 8;
  void* scratch = nullptr;
  if (int rc = scratch_alloc(&scratch, tx_bytes + sig_bytes, st)) return rc;
  p.tx = static_cast<float2*>(scratch);
  p.sig_part = reinterpret_cast<double*>(static_cast<char*>(scratch) + tx_bytes);
  cudaError_t e = ofdmrx::launch_synth(p, st);
  cudaError_t e2 = cudaFreeAsync(scratch, st);
  if (e != cudaSuccess) return cuda_fail(e, "synth kernels launch");
  if (e2 != cudaSuccess) return cuda_fail(e2, "cudaFreeAsync");
  return OFDMRX_OK;
}

int ofdmrx_demap(const void* symbols, int64_t n, int32_t qam_order, uint8_t* bits, void* stream) {
  if (int rc = check_qam(qam_order)) return rc;
  if (n < 0) return fail(OFDMRX_ERR_CONTRACT, "n must be >= 0");
  if (n == 0) return OFDMRX_OK;
  if (int rc = check_ptr(symbols, "symbols")) return rc;
  if (int rc = check_ptr(bits, "bits")) return rc;
  if (int rc = check_align(bits, 4, "bits")) return rc;
  int qb, levels;
  float scale;
  qam_consts(qam_order, &qb, &levels, &scale);
  cudaError_t e = ofdmrx::launch_demap(static_cast<const float2*>(symbols), n, qb, levels, scale, bits,
                                       static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "demap_kernel launch");
  return OFDMRX_OK;
}

}  // extern "C"
