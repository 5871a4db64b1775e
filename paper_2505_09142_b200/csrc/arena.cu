// arena.cu -- device-resident token arena of the in-flight requests.
//
// PAPER.md Sec. 3.4 sends a request's prompt to the scheduler once and feeds back only the partial
// outputs of each window ("the prompt is sent once ... fixed-window partial outputs");
// the predictor input is "the prompt attached with the answer", re-encoded whenever the
// job returns to the Job Pool (Alg. 1 lines 10-18).  Here every slot of the in-flight
// table owns, in device memory, its prompt ([CLS] ... [SEP], <= 512 tokens) and a ring of its 512
// most recent response tokens.  Per iteration the host uploads only the new prompts and the <= K
// tokens each returning job generated; the due set's predictor input is gathered on the device:
//   sequence = prompt ++ response                          if |prompt| + g <= max_len,
//            = prompt[:max_len - k] ++ response[g - k:g]   otherwise, k = min(g, 254)
// (R7; the same rule as the harness's streamsim.build_sequence).
#include "common.cuh"
#include "kernels.cuh"

namespace elis {

namespace {

constexpr int kArenaThreads = 1024;

// exclusive scan of v over the CTA (1024 threads); *total = sum
__device__ int arena_block_scan(int v, int* warp_tot, int* total) {
  const int lane = lane_id(), w = warp_id();
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[w] = x;
  __syncthreads();
  if (w == 0) {
    const int t = lane < static_cast<int>(blockDim.x >> 5) ? warp_tot[lane] : 0;
    int s = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    warp_tot[lane] = s - t;
    if (lane == 31) *total = s;
  }
  __syncthreads();
  const int r = warp_tot[w] + x - v;
  __syncthreads();
  return r;
}

// offsets[i] = exclusive prefix of counts[0..m) (one CTA, chunks of consecutive entries per thread)
__global__ void __launch_bounds__(kArenaThreads) k_arena_offsets(const int32_t* __restrict__ counts, int m,
                                                                 int32_t* __restrict__ offsets) {
  __shared__ int warp_tot[32], total;
  const int per = (m + kArenaThreads - 1) / kArenaThreads;
  const int i0 = min(m, static_cast<int>(threadIdx.x) * per), i1 = min(m, i0 + per);
  int s = 0;
  for (int i = i0; i < i1; ++i) s += max(0, counts[i]);
  int off = arena_block_scan(s, warp_tot, &total);
  for (int i = i0; i < i1; ++i) {
    offsets[i] = off;
    off += max(0, counts[i]);
  }
}

// new prompts: slot s = slots[i] takes tokens[offsets[i] .. + lengths[i]) (clipped to kArenaLen)
__global__ void k_arena_set(const int32_t* __restrict__ slots, const int32_t* __restrict__ tokens,
                            const int32_t* __restrict__ lengths, const int32_t* __restrict__ offsets, int max_slots,
                            int32_t* __restrict__ prompt, int32_t* __restrict__ plen, int32_t* __restrict__ glen,
                            uint32_t* __restrict__ err) {
  const int i = blockIdx.x, s = slots[i], L = lengths[i];
  if (s < 0 || s >= max_slots || L < 1 || L > kArenaLen) {
    if (threadIdx.x == 0) atomicOr(err, ERR_ARENA);
    return;
  }
  const int32_t* src = tokens + offsets[i];
  int32_t* dst = prompt + static_cast<size_t>(s) * kArenaLen;
  for (int t = threadIdx.x; t < L; t += blockDim.x) dst[t] = src[t];
  if (threadIdx.x == 0) {
    plen[s] = L;
    glen[s] = 0;
  }
}

// generated tokens: slot s = slots[i] appends tokens[offsets[i] .. + counts[i]) to its response ring
__global__ void k_arena_append(const int32_t* __restrict__ slots, const int32_t* __restrict__ tokens,
                               const int32_t* __restrict__ counts, const int32_t* __restrict__ offsets, int max_slots,
                               int32_t* __restrict__ ring, int32_t* __restrict__ glen, uint32_t* __restrict__ err) {
  const int i = blockIdx.x, s = slots[i], c = counts[i];
  if (s < 0 || s >= max_slots || c < 0) {
    if (threadIdx.x == 0) atomicOr(err, ERR_ARENA);
    return;
  }
  const int g = glen[s];
  const int32_t* src = tokens + offsets[i];
  int32_t* dst = ring + static_cast<size_t>(s) * kArenaLen;
  for (int t = threadIdx.x; t < c; t += blockDim.x) dst[(g + t) % kArenaLen] = src[t];
  __syncthreads();
  if (threadIdx.x == 0) glen[s] = g + c;
}

// predictor input length of slot s (R7)
ELIS_DEV int arena_seq_len(int p, int g, int max_len, int* head, int* keep) {
  if (p + g <= max_len) {
    *head = p;
    *keep = g;
  } else {
    *keep = min(g, kArenaKeepResp);
    *head = min(p, max_len - *keep);
  }
  return *head + *keep;
}

// lengths[i] of the due slots, cu (exclusive offsets, [n + 1]) and dims = {n, total}
__global__ void __launch_bounds__(kArenaThreads) k_arena_lengths(const int32_t* __restrict__ slots, int n,
                                                                 int max_slots, int max_len,
                                                                 const int32_t* __restrict__ plen,
                                                                 const int32_t* __restrict__ glen,
                                                                 int32_t* __restrict__ lengths, int32_t* __restrict__ cu,
                                                                 int32_t* __restrict__ dims, uint32_t* __restrict__ err) {
  __shared__ int warp_tot[32], total;
  const int per = (n + kArenaThreads - 1) / kArenaThreads;
  const int i0 = min(n, static_cast<int>(threadIdx.x) * per), i1 = min(n, i0 + per);
  int s = 0;
  uint32_t e = 0;
  for (int i = i0; i < i1; ++i) {
    const int slot = slots[i];
    int L = 1;
    if (slot < 0 || slot >= max_slots || plen[slot] < 1) {
      e = ERR_ARENA;
    } else {
      int h, k;
      L = arena_seq_len(plen[slot], glen[slot], max_len, &h, &k);
    }
    lengths[i] = L;
    s += L;
  }
  if (e) atomicOr(err, e);
  int off = arena_block_scan(s, warp_tot, &total);
  for (int i = i0; i < i1; ++i) {
    cu[i] = off;
    off += lengths[i];
  }
  if (threadIdx.x == 0) {
    cu[n] = total;
    if (dims) {
      dims[0] = n;
      dims[1] = total;
    }
  }
}

// tokens[cu[i] ..] = the predictor input of due slot i (one CTA per request)
__global__ void k_arena_copy(const int32_t* __restrict__ slots, int max_slots, int max_len,
                             const int32_t* __restrict__ prompt, const int32_t* __restrict__ ring,
                             const int32_t* __restrict__ plen, const int32_t* __restrict__ glen,
                             const int32_t* __restrict__ cu, int32_t* __restrict__ out) {
  const int i = blockIdx.x, slot = slots[i];
  int32_t* dst = out + cu[i];
  if (slot < 0 || slot >= max_slots || plen[slot] < 1) {  // reported by k_arena_lengths; a valid token
    if (threadIdx.x == 0) dst[0] = 101;
    return;
  }
  const int g = glen[slot];
  int head, keep;
  arena_seq_len(plen[slot], g, max_len, &head, &keep);
  const int32_t* pr = prompt + static_cast<size_t>(slot) * kArenaLen;
  const int32_t* rg = ring + static_cast<size_t>(slot) * kArenaLen;
  for (int t = threadIdx.x; t < head; t += blockDim.x) dst[t] = pr[t];
  for (int t = threadIdx.x; t < keep; t += blockDim.x) dst[head + t] = rg[(g - keep + t) % kArenaLen];
}

}  // namespace

cudaError_t launch_arena_offsets(const int32_t* counts, int m, int32_t* offsets, cudaStream_t st) {
  if (m <= 0) return cudaSuccess;
  k_arena_offsets<<<1, kArenaThreads, 0, st>>>(counts, m, offsets);
  return cudaGetLastError();
}

cudaError_t launch_arena_set(const int32_t* slots, const int32_t* tokens, const int32_t* lengths,
                             const int32_t* offsets, int m, int max_slots, int32_t* prompt, int32_t* plen,
                             int32_t* glen, uint32_t* err, cudaStream_t st) {
  if (m <= 0) return cudaSuccess;
  k_arena_set<<<m, 128, 0, st>>>(slots, tokens, lengths, offsets, max_slots, prompt, plen, glen, err);
  return cudaGetLastError();
}

cudaError_t launch_arena_append(const int32_t* slots, const int32_t* tokens, const int32_t* counts,
                                const int32_t* offsets, int m, int max_slots, int32_t* ring, int32_t* glen,
                                uint32_t* err, cudaStream_t st) {
  if (m <= 0) return cudaSuccess;
  k_arena_append<<<m, 64, 0, st>>>(slots, tokens, counts, offsets, max_slots, ring, glen, err);
  return cudaGetLastError();
}

cudaError_t launch_arena_gather(const int32_t* slots, int n, int max_slots, int max_len, const int32_t* prompt,
                                const int32_t* ring, const int32_t* plen, const int32_t* glen, int32_t* lengths,
                                int32_t* cu, int32_t* dims, int32_t* out_tokens, uint32_t* err, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  k_arena_lengths<<<1, kArenaThreads, 0, st>>>(slots, n, max_slots, max_len, plen, glen, lengths, cu, dims, err);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  k_arena_copy<<<n, 128, 0, st>>>(slots, max_slots, max_len, prompt, ring, plen, glen, cu, out_tokens);
  return cudaGetLastError();
}

}  // namespace elis
