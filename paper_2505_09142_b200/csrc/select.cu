// select.cu -- ISRTF / FCFS batch selection: key pack + exact radix top-k + preempt flags.
//
// PAPER.md Algorithm 1 line 19 "Batched Prompt <- Batcher.batch(Priority
// Buffer)"; the batch is formed "starting with the prompt with the highest priority"
// (P:301); ISRTF priority = predicted remaining tokens; FCFS = arrival
// (P:463); preemption evicts the lowest priority first.
//
// Key (u64, smaller = higher priority; readings R4-R6, R9):
//     bit 63      class: 0 for every slot if allow_preempt, else 0 = running, 1 = other
//     bits 32-62  fp32 bits of max(0, remaining) (sign bit 0, so unsigned order = float
//                 order); NaN -> +inf (0x7F800000); FCFS -> 0
//     bits 0-31   order = unique rank of (arrival, id)
//     ineligible slot (generated < 0) -> UINT64_MAX
// Keys are unique, so the top-cap set and its order are unique: the result is exact and
// deterministic regardless of thread scheduling.
//
// top-k: one CTA, MSB-first 8-bit radix select over the keys (L2-resident), with early
// exit once the bucket holding the cap-th key is exactly the remaining need; compaction
// of the winners into shared memory; bitonic sort; -1 padding.
#include "common.cuh"
#include "kernels.cuh"

namespace elis {

namespace {

constexpr unsigned long long KEY_NONE = 0xFFFFFFFFFFFFFFFFull;

__global__ void k_make_keys(const float* __restrict__ pred, const int32_t* __restrict__ generated,
                            const uint32_t* __restrict__ order, const uint8_t* __restrict__ running, int n, int policy,
                            int allow_preempt, int head_predicts_total, uint32_t order_offset,
                            unsigned long long* __restrict__ keys, uint32_t* __restrict__ info) {
  uint32_t nan_local = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int g = generated[i];
    unsigned long long key = KEY_NONE;
    if (g >= 0) {
      uint32_t bits = 0;
      if (policy == 0) {
        float rem = pred[i];
        if (head_predicts_total) rem = __fsub_rn(rem, static_cast<float>(g));
        if (rem != rem) {
          bits = 0x7F800000u;
          ++nan_local;
        } else if (rem > 0.f) {
          bits = __float_as_uint(rem);  // includes +inf = 0x7F800000
        } else {
          bits = 0u;  // negatives, -0 and +0 all key as +0
        }
      }
      const uint32_t cls = (allow_preempt || (running && running[i])) ? 0u : 1u;
      const uint32_t ord = order ? order[i] : order_offset + static_cast<uint32_t>(i);
      key = (static_cast<unsigned long long>(cls) << 63) | (static_cast<unsigned long long>(bits) << 32) | ord;
    }
    keys[i] = key;
  }
  nan_local = __reduce_add_sync(0xffffffffu, nan_local);
  if (lane_id() == 0 && nan_local) atomicAdd(info + 6, nan_local);
}

constexpr int kSelThreads = 1024;

__global__ void __launch_bounds__(kSelThreads) k_select_topk(const unsigned long long* __restrict__ keys,
                                                             const int32_t* __restrict__ ids, int n, int cap,
                                                             int32_t* __restrict__ out_ids, int32_t* __restrict__ out_count,
                                                             int32_t* __restrict__ out_nan, uint32_t* __restrict__ info,
                                                             unsigned long long* __restrict__ sel_keys,
                                                             int32_t* __restrict__ sel_ids, int sort_len) {
  extern __shared__ __align__(16) uint8_t sm[];
  unsigned long long* ck = reinterpret_cast<unsigned long long*>(sm);       // [sort_len]
  int32_t* ci = reinterpret_cast<int32_t*>(ck + sort_len);                  // [sort_len]
  __shared__ int hist[256];
  __shared__ int s_elig, s_count, s_digit, s_remaining, s_done;
  __shared__ unsigned long long s_prefix, s_mask;

  const int tid = threadIdx.x;
  if (tid == 0) { s_elig = 0; s_count = 0; s_prefix = 0; s_mask = 0; s_done = 0; }
  __syncthreads();
  int e = 0;
  for (int i = tid; i < n; i += kSelThreads) e += (keys[i] != KEY_NONE);
  e = __reduce_add_sync(0xffffffffu, e);
  if (lane_id() == 0) atomicAdd(&s_elig, e);
  __syncthreads();
  const int target = min(cap, s_elig);
  if (tid == 0) s_remaining = target;
  __syncthreads();

  if (target > 0 && target < s_elig) {
    for (int pass = 0; pass < 8; ++pass) {
      const int shift = 56 - 8 * pass;
      for (int b = tid; b < 256; b += kSelThreads) hist[b] = 0;
      __syncthreads();
      const unsigned long long prefix = s_prefix, mask = s_mask;
      for (int i = tid; i < n; i += kSelThreads) {
        const unsigned long long k = keys[i];
        if (k != KEY_NONE && (k & mask) == prefix) atomicAdd(&hist[(k >> shift) & 255], 1);
      }
      __syncthreads();
      if (tid < 32) {
        // lane l owns bins [8l, 8l + 8)
        int c[8], tot = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) { c[q] = hist[8 * tid + q]; tot += c[q]; }
        int incl = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, incl, o);
          if (tid >= o) incl += y;
        }
        const int excl = incl - tot;
        const int need = s_remaining;
        if (need > excl && need <= incl) {
          int run = excl;
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            if (need > run && need <= run + c[q]) {
              s_digit = 8 * tid + q;
              s_remaining = need - run;
              s_done = (c[q] == need - run) ? 1 : 0;
            }
            run += c[q];
          }
        }
      }
      __syncthreads();
      if (tid == 0) {
        s_prefix |= static_cast<unsigned long long>(s_digit) << shift;
        s_mask |= 0xFFull << shift;
      }
      __syncthreads();
      if (s_done) break;
    }
  }
  // winners: eligible keys whose masked prefix <= prefix (all eligible if target == s_elig)
  const bool take_all = (target == s_elig);
  const unsigned long long prefix = s_prefix, mask = s_mask;
  for (int i = tid; i < n; i += kSelThreads) {
    const unsigned long long k = keys[i];
    if (k == KEY_NONE) continue;
    if (take_all || (k & mask) <= prefix) {
      const int slot = atomicAdd(&s_count, 1);
      if (slot < sort_len) {
        ck[slot] = k;
        ci[slot] = ids ? ids[i] : i;
      }
    }
  }
  __syncthreads();
  for (int i = s_count + tid; i < sort_len; i += kSelThreads) {
    ck[i] = KEY_NONE;
    ci[i] = -1;
  }
  __syncthreads();
  // bitonic sort ascending (sort_len is a power of two)
  for (int size = 2; size <= sort_len; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = tid; i < sort_len / 2; i += kSelThreads) {
        const int lo = 2 * i - (i & (stride - 1));
        const int hi = lo + stride;
        const bool up = ((lo & size) == 0);
        const unsigned long long a = ck[lo], b = ck[hi];
        if ((a > b) == up) {
          ck[lo] = b; ck[hi] = a;
          const int t = ci[lo]; ci[lo] = ci[hi]; ci[hi] = t;
        }
      }
      __syncthreads();
    }
  }
  for (int j = tid; j < cap; j += kSelThreads) {
    const bool v = j < target;
    out_ids[j] = v ? ci[j] : -1;
    if (sel_keys) sel_keys[j] = v ? ck[j] : KEY_NONE;
    if (sel_ids) sel_ids[j] = v ? ci[j] : -1;
  }
  if (tid == 0) {
    if (out_count) *out_count = target;
    // threshold = the target-th key: a slot is selected iff eligible and key <= threshold
    const unsigned long long thr = target > 0 ? ck[target - 1] : 0ull;
    info[0] = static_cast<uint32_t>(thr);
    info[1] = static_cast<uint32_t>(thr >> 32);
    info[4] = static_cast<uint32_t>(target);
    info[5] = static_cast<uint32_t>(s_elig);
    if (out_nan) *out_nan = static_cast<int32_t>(info[6]);
  }
}

__global__ void k_preempt(const unsigned long long* __restrict__ keys, const uint8_t* __restrict__ running, int n,
                          const uint32_t* __restrict__ info, uint8_t* __restrict__ out) {
  const unsigned long long thr = (static_cast<unsigned long long>(info[1]) << 32) | info[0];
  const bool any = info[4] > 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const unsigned long long k = keys[i];
    const bool selected = any && k != KEY_NONE && k <= thr;
    out[i] = (running && running[i] && !selected) ? 1 : 0;
  }
}

struct Candidate {
  unsigned long long key;
  int32_t id;
  int32_t pad;
};

__global__ void k_pack(const unsigned long long* __restrict__ sel_keys, const int32_t* __restrict__ sel_ids, int cap,
                       int global_offset, Candidate* __restrict__ send) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < cap; j += gridDim.x * blockDim.x) {
    const int id = sel_ids[j];
    send[j].key = sel_keys[j];
    send[j].id = id >= 0 ? id + global_offset : -1;
    send[j].pad = 0;
  }
}

__global__ void k_unpack(const Candidate* __restrict__ recv, int total, unsigned long long* __restrict__ keys,
                         int32_t* __restrict__ ids) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < total; j += gridDim.x * blockDim.x) {
    keys[j] = recv[j].key;
    ids[j] = recv[j].id;
  }
}

int next_pow2(int x) {
  int p = 1;
  while (p < x) p <<= 1;
  return p;
}

}  // namespace

cudaError_t launch_make_keys(const float* pred, const int32_t* generated, const uint32_t* order,
                             const uint8_t* running, int n, int policy, int allow_preempt, int head_predicts_total,
                             uint32_t order_offset, unsigned long long* keys, uint32_t* info, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(info, 0, 8 * sizeof(uint32_t), st);
  if (e != cudaSuccess || n <= 0) return e;
  int blocks = (n + 255) / 256;
  if (blocks > 1184) blocks = 1184;
  k_make_keys<<<blocks, 256, 0, st>>>(pred, generated, order, running, n, policy, allow_preempt, head_predicts_total,
                                      order_offset, keys, info);
  return cudaGetLastError();
}

cudaError_t launch_select_topk(const unsigned long long* keys, const int32_t* ids, int n, int cap, int32_t* out_ids,
                               int32_t* out_count, int32_t* out_nan, SelectScratch sc, cudaStream_t st) {
  const int sort_len = next_pow2(cap < 2 ? 2 : cap);
  const size_t smem = static_cast<size_t>(sort_len) * (sizeof(unsigned long long) + sizeof(int32_t));
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_select_topk, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(kMaxBatchCap * 12 + 1024));
    if (e != cudaSuccess) return e;
    attr = true;
  }
  k_select_topk<<<1, kSelThreads, smem, st>>>(keys, ids, n, cap, out_ids, out_count, out_nan, sc.info, sc.sel_keys,
                                              sc.sel_ids, sort_len);
  return cudaGetLastError();
}

cudaError_t launch_preempt_flags(const unsigned long long* keys, const uint8_t* running, int n, const uint32_t* info,
                                 uint8_t* out_preempted, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  int blocks = (n + 255) / 256;
  if (blocks > 1184) blocks = 1184;
  k_preempt<<<blocks, 256, 0, st>>>(keys, running, n, info, out_preempted);
  return cudaGetLastError();
}

cudaError_t launch_pack_candidates(const SelectScratch sc, int cap, int global_offset, void* send, cudaStream_t st) {
  k_pack<<<(cap + 255) / 256, 256, 0, st>>>(sc.sel_keys, sc.sel_ids, cap, global_offset,
                                            static_cast<Candidate*>(send));
  return cudaGetLastError();
}

cudaError_t launch_unpack_candidates(const void* recv, int total, unsigned long long* keys, int32_t* ids,
                                     cudaStream_t st) {
  k_unpack<<<(total + 255) / 256, 256, 0, st>>>(static_cast<const Candidate*>(recv), total, keys, ids);
  return cudaGetLastError();
}

}  // namespace elis
