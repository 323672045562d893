// Single-pass decoupled look-back tile prefix (device helper).
// Status words are epoch-stamped so no per-launch clearing is needed:
//   bits 63..48 epoch, 47..46 flag (0 empty, 1 aggregate, 2 inclusive), 45..0 value.
#pragma once
#include <cstdint>

#include "device.cuh"

namespace gsm {

constexpr uint64_t LB_VMASK = (1ull << 46) - 1;

__device__ __forceinline__ unsigned long long lb_pack(uint32_t epoch, uint32_t flag, uint64_t v) {
  return ((unsigned long long)epoch << 48) | ((unsigned long long)flag << 46) | (v & LB_VMASK);
}

// Claim the next tile index (monotone across the grid).
__device__ __forceinline__ uint32_t lb_claim(uint32_t* counter, uint32_t* s_slot) {
  if (threadIdx.x == 0) *s_slot = atomicAdd(counter, 1u);
  __syncthreads();
  uint32_t t = *s_slot;
  __syncthreads();
  return t;
}

// Exclusive prefix of `total` over tiles 0..tile-1; call from all threads of the
// CTA (total valid in thread 0).  Returns the prefix in every thread.
__device__ __forceinline__ uint64_t lb_prefix(unsigned long long* status, uint32_t epoch, uint32_t tile,
                                              uint64_t total, unsigned long long* s_slot) {
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    uint64_t excl = 0;
    uint64_t tot = __shfl_sync(GSM_FULL, total, 0);
    if (tile == 0) {
      if (lane == 0) atomicExch(status, lb_pack(epoch, 2, tot));
    } else {
      if (lane == 0) atomicExch(status + tile, lb_pack(epoch, 1, tot));
      int64_t pred = (int64_t)tile - 1;
      while (true) {
        int64_t idx = pred - lane;
        unsigned long long s = idx >= 0 ? *((volatile unsigned long long*)(status + idx)) : lb_pack(epoch, 2, 0);
        uint32_t ep = (uint32_t)(s >> 48), fl = (uint32_t)((s >> 46) & 3u);
        bool ready = ep == epoch && fl != 0;
        // only the predecessors up to the nearest inclusive one must be ready
        // (waiting for the whole 32-tile window stalls on unrelated slow tiles)
        const uint32_t inc = __ballot_sync(GSM_FULL, ready && fl == 2);
        const uint32_t notready = __ballot_sync(GSM_FULL, !ready);
        const uint32_t need = inc ? ((2u << (__ffs(inc) - 1)) - 1u) : GSM_FULL;
        if (notready & need) continue;
        uint64_t v = s & LB_VMASK;
        if (inc) {
          int k = __ffs(inc) - 1;
          if (lane > k) v = 0;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(GSM_FULL, v, o);
        excl += __shfl_sync(GSM_FULL, v, 0);
        if (inc) break;
        pred -= 32;
      }
      if (lane == 0) atomicExch(status + tile, lb_pack(epoch, 2, excl + tot));
    }
    if (lane == 0) *s_slot = excl;
  }
  __syncthreads();
  uint64_t r = *s_slot;
  __syncthreads();
  return r;
}

}  // namespace gsm
