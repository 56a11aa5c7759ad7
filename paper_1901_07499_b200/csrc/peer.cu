// Antenna-sharded MRC exchange over peer memory: the fused
// partial-sum kernel stores each frame's (num, den) straight into the inbox of
// the rank that finishes that frame (CUDA IPC mappings of peer allocations:
// NVLink/NVSwitch stores on a multi-GPU box), then release/acquire flags at
// system scope hand the inbox to its owner.  No NCCL call on the data path.
//
// Per call (epoch e), on every rank (see sharding.PeerExchange):
//   wait   consumed[o] >= e-1 for every owner o  (inbox free)
//   fused  partials of this rank's antennas -> inbox[o].slot[rank]
//   signal ready[o][rank] = e for every owner o
//   wait   ready[self][i] >= e for every producer i
//   finish pairwise tree over the slots of the own frames, divide, demap
//   signal consumed[self] = e
#include <cstdint>

#include "ofdmrx_internal.h"

namespace ofdmrx {

namespace {

__global__ void peer_signal_kernel(unsigned long long* const* dst, int n, unsigned long long value) {
  if (threadIdx.x != 0) return;
  // the previous kernels of this stream (partial sums stored to peers) are
  // complete; order them before the flags at system scope
  __threadfence_system();
  for (int i = 0; i < n; ++i)
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(dst[i]), "l"(value) : "memory");
}

__global__ void peer_wait_kernel(const unsigned long long* const* src, int n, unsigned long long value) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    unsigned long long v;
    for (;;) {
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(src[i]) : "memory");
      if (v >= value) break;
      __nanosleep(200);
    }
  }
  __syncthreads();
  __threadfence_system();
}

}  // namespace

cudaError_t launch_peer_signal(unsigned long long* const* dst, int n, unsigned long long value, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  peer_signal_kernel<<<1, 32, 0, s>>>(dst, n, value);
  return cudaGetLastError();
}

cudaError_t launch_peer_wait(const unsigned long long* const* src, int n, unsigned long long value, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  peer_wait_kernel<<<1, 32, 0, s>>>(src, n, value);
  return cudaGetLastError();
}

}  // namespace ofdmrx
