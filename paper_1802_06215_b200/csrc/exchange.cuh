// exchange.cuh -- K4, the multi-GPU exchange of a scenario-sharded batch with
// dense observation keys, compacted (SURVEY §8(e) "compact to
// non-empty slots").  K2 leaves every rank with exact int64 partial sums per
// (leaf, action, slot) in the dense block, most of whose slots are empty.
// The library's communicator then runs:
//
//   k4_flags   slot used on this rank (N != 0)                      -> u8 [LAS]
//   round A    all-reduce SUM of the flags: the union over ranks (identical everywhere)
//   k4_count   union slots per block of kXBlk slots
//   k4_pack    offsets = prefix of the counts; the union slots' (W, U, LAMBDA, N)
//              and first ids, and the per-action (R, Uq, Lq) + step count, packed
//   round B    all-reduce SUM of the packed sums, MIN of the packed first ids
//   k4_unpack  the global values back into the dense block (then K3 as at world 1)
//
// The packed buffer has a host-chosen capacity (no read-back in the batch):
// when the union exceeds it every rank sets kErrXOverflow (the union is the
// same everywhere), leaves its dense block untouched, and the host re-runs the
// exchange on the dense block after the batch's status read-back.
#pragma once
#include "common.cuh"

namespace hd {

constexpr uint32_t kXThreads = 256, kXPer = 16, kXBlk = kXThreads * kXPer;  // slots per CTA

struct XDev {
  uint8_t* flags;   // [nblk * kXBlk] (the tail past las stays 0)
  uint32_t* cnt;    // [nblk] union slots per block
  int64_t* cpk;     // [4 ccap + qn]: (W, U, LAMBDA, N) per packed slot, then the Q block + steps
  int32_t* cmin;    // [ccap] first ids of the packed slots
  uint64_t las, ccap, qn;
  uint32_t nblk;
};

__global__ void __launch_bounds__(kXThreads) k4_flags(BatchDev b, XDev x) {
  const SumLayout lay{x.las, (uint64_t)b.L * b.A};
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < x.las; i += (uint64_t)gridDim.x * blockDim.x)
    x.flags[i] = b.sums[lay.N(i)] != 0 ? 1 : 0;
}

// the 16 flags of thread t of block blk, as a bit mask
__device__ __forceinline__ uint32_t k4_bits(const XDev& x, uint32_t blk, uint32_t t) {
  const uint4 v = *reinterpret_cast<const uint4*>(x.flags + (uint64_t)blk * kXBlk + (uint64_t)t * kXPer);
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
  uint32_t m = 0;
#pragma unroll
  for (int k = 0; k < 16; ++k) m |= (((w[k >> 2] >> (8 * (k & 3))) & 0xFFu) != 0 ? 1u : 0u) << k;
  return m;
}

__device__ __forceinline__ uint32_t k4_block_sum(uint32_t v, uint32_t* sh) {
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  v = __reduce_add_sync(0xffffffffu, v);
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  uint32_t t = 0;
  for (uint32_t k = 0; k < blockDim.x / 32; ++k) t += sh[k];
  __syncthreads();
  return t;
}

__global__ void __launch_bounds__(kXThreads) k4_count(XDev x) {
  __shared__ uint32_t sh[kXThreads / 32];
  const uint32_t c = (uint32_t)__popc(k4_bits(x, blockIdx.x, threadIdx.x));
  const uint32_t tot = k4_block_sum(c, sh);
  if (threadIdx.x == 0) x.cnt[blockIdx.x] = tot;
}

// (block prefix, total) from the per-block counts; exclusive in-block offset
// of this thread; its flag bits
struct K4Pos {
  uint64_t base, total;
  uint32_t bits, off;
};
__device__ __forceinline__ K4Pos k4_positions(const XDev& x) {
  __shared__ uint32_t sh[kXThreads / 32];
  __shared__ unsigned long long s_pre, s_tot;
  if (threadIdx.x == 0) {
    s_pre = 0;
    s_tot = 0;
  }
  __syncthreads();
  unsigned long long pre = 0, tot = 0;
  for (uint32_t k = threadIdx.x; k < x.nblk; k += blockDim.x) {
    tot += x.cnt[k];
    pre += k < blockIdx.x ? x.cnt[k] : 0u;
  }
  atomicAdd(&s_pre, pre);
  atomicAdd(&s_tot, tot);
  K4Pos p;
  p.bits = k4_bits(x, blockIdx.x, threadIdx.x);
  // exclusive scan of the per-thread counts over the block
  const uint32_t c = (uint32_t)__popc(p.bits), lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t inc = c;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t v = __shfl_up_sync(0xffffffffu, inc, d);
    if ((int)lane >= d) inc += v;
  }
  if (lane == 31) sh[wid] = inc;
  __syncthreads();
  uint32_t wpre = 0;
  for (uint32_t k = 0; k < wid; ++k) wpre += sh[k];
  p.off = wpre + inc - c;
  p.base = s_pre;
  p.total = s_tot;
  return p;
}

__global__ void __launch_bounds__(kXThreads) k4_pack(BatchDev b, XDev x) {
  const SumLayout lay{x.las, (uint64_t)b.L * b.A};
  const K4Pos p = k4_positions(x);
  if (p.total > x.ccap) {  // the same on every rank: all of them fall back to the dense block
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      atomicOr(b.err, kErrXOverflow);
      b.status[kStatXTotal] = p.total > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)p.total;
    }
    return;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) b.status[kStatXTotal] = (uint32_t)p.total;
  uint64_t o = p.base + p.off;
  const uint64_t i0 = (uint64_t)blockIdx.x * kXBlk + (uint64_t)threadIdx.x * kXPer;
  for (uint32_t bits = p.bits; bits; bits &= bits - 1u, ++o) {
    const uint64_t i = i0 + (uint64_t)(__ffs(bits) - 1);
    HD_CHECK(b.err, o < x.ccap && i < x.las);
    int64_t* q = x.cpk + 4 * o;
    q[0] = b.sums[lay.W(i)];
    q[1] = b.sums[lay.U(i)];
    q[2] = b.sums[lay.Lm(i)];
    q[3] = b.sums[lay.N(i)];
    x.cmin[o] = b.mins[i];
  }
  // the per-action partials and the step count travel whole
  for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < x.qn; k += (uint64_t)gridDim.x * blockDim.x)
    x.cpk[4 * x.ccap + k] = b.sums[lay.Q(0, 0) + k];
}

__global__ void __launch_bounds__(kXThreads) k4_unpack(BatchDev b, XDev x) {
  if (*reinterpret_cast<volatile uint32_t*>(b.err) & kErrXOverflow) return;  // dense fallback after the batch
  const SumLayout lay{x.las, (uint64_t)b.L * b.A};
  const K4Pos p = k4_positions(x);
  uint64_t o = p.base + p.off;
  const uint64_t i0 = (uint64_t)blockIdx.x * kXBlk + (uint64_t)threadIdx.x * kXPer;
  for (uint32_t bits = p.bits; bits; bits &= bits - 1u, ++o) {
    const uint64_t i = i0 + (uint64_t)(__ffs(bits) - 1);
    const int64_t* q = x.cpk + 4 * o;
    b.sums[lay.W(i)] = q[0];
    b.sums[lay.U(i)] = q[1];
    b.sums[lay.Lm(i)] = q[2];
    b.sums[lay.N(i)] = q[3];
    b.mins[i] = x.cmin[o];
  }
  for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < x.qn; k += (uint64_t)gridDim.x * blockDim.x)
    b.sums[lay.Q(0, 0) + k] = x.cpk[4 * x.ccap + k];
}

}  // namespace hd
