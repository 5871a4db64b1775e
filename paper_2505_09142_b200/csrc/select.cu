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
                            int allow_preempt, int head_predicts_total, uint32_t order_offset, Starvation sv,
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
        if (rem == rem) {
          // starvation control (R17): aging, then the preemption
          // margin of running jobs; explicit fp32 roundings (no contraction), as the oracle
          if (sv.waited && sv.boost_amount != 0.f) {
            const int wt = sv.waited[i];
            if (wt > 0) rem = __fsub_rn(rem, __fmul_rn(sv.boost_amount, static_cast<float>(wt / sv.boost_after)));
          }
          if (sv.margin != 0.f && running && running[i]) rem = __fsub_rn(rem, sv.margin);
        }
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
constexpr int kSelBatch = 8;   // keys per thread per load batch

// Exact top-cap of one CTA (1024 threads): the cap smallest eligible keys among slots i < n
// with mine(i) (key != UINT64_MAX and, with nodes, node[i] == w), ascending, into ck / ci
// (sort_len entries; the tail KEY_NONE / -1).  MSB-first 8-bit radix select of the cap-th key
// (early exit once its bucket is exactly the remaining need), compaction of the winners,
// bitonic sort.  Returns the number selected, min(cap, eligible); *elig_out = eligible.
__device__ int cta_topk_sorted(const unsigned long long* keys, const int32_t* ids, const int32_t* node, int w, bool ready, int n, int cap, int sort_len,
                               unsigned long long* ck, int32_t* ci, int* elig_out) {
  __shared__ int hist[256];
  __shared__ int s_elig, s_count, s_digit, s_remaining, s_done;
  __shared__ unsigned long long s_prefix, s_mask, s_min, s_max;
  const int tid = threadIdx.x, lane = lane_id();
  // slot i takes part in this block's selection
  auto mine = [&](int i, unsigned long long k) { return k != KEY_NONE && (!node || node[i] == w); };
  __syncthreads();  // a previous call's readers of the shared state are done
  if (tid == 0) { s_elig = 0; s_count = 0; s_prefix = 0; s_mask = 0; s_done = 0; s_min = KEY_NONE; s_max = 0; }
  __syncthreads();
  // eligible count and the smallest / largest eligible key: every eligible key shares the bits
  // above the highest bit where min and max differ, so the radix starts at that byte (the
  // leading passes, where every key falls into one bucket, are skipped)
  // every scan loads kSelBatch keys per thread before using them (independent loads in flight:
  // one L2 round trip per batch instead of per key); i0 is uniform, so warps stay converged
  auto scan = [&](auto&& fn) {
    for (int i0 = 0; i0 < n; i0 += kSelBatch * kSelThreads) {
      unsigned long long kb[kSelBatch];
      bool mb[kSelBatch];
#pragma unroll
      for (int u = 0; u < kSelBatch; ++u) {
        const int i = i0 + u * kSelThreads + tid;
        kb[u] = i < n ? keys[i] : KEY_NONE;
      }
#pragma unroll
      for (int u = 0; u < kSelBatch; ++u) {
        const int i = i0 + u * kSelThreads + tid;
        mb[u] = i < n && mine(i, kb[u]);
      }
#pragma unroll
      for (int u = 0; u < kSelBatch; ++u) fn(i0 + u * kSelThreads + tid, kb[u], mb[u]);
    }
  };
  int e = 0;
  unsigned long long kmin = KEY_NONE, kmax = 0;
  if (ready)
    scan([&](int, unsigned long long k, bool m) {
      if (m) { ++e; kmin = k < kmin ? k : kmin; kmax = k > kmax ? k : kmax; }
    });
  e = __reduce_add_sync(0xffffffffu, e);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long a = __shfl_xor_sync(0xffffffffu, kmin, o), b = __shfl_xor_sync(0xffffffffu, kmax, o);
    kmin = a < kmin ? a : kmin;
    kmax = b > kmax ? b : kmax;
  }
  if (lane == 0) {
    atomicAdd(&s_elig, e);
    atomicMin(&s_min, kmin);
    atomicMax(&s_max, kmax);
  }
  __syncthreads();
  const int target = min(cap, s_elig);
  if (tid == 0) s_remaining = target;
  int start_shift = 56;
  if (target > 0 && target < s_elig) {   // >= 2 distinct (unique) keys: min != max
    const int top = 63 - __clzll(static_cast<long long>(s_min ^ s_max));
    start_shift = (top >> 3) << 3;
    if (tid == 0 && start_shift < 56) {
      s_mask = ~((1ull << (start_shift + 8)) - 1ull);
      s_prefix = s_min & s_mask;
    }
  }
  __syncthreads();

  if (target > 0 && target < s_elig) {
    for (int shift = start_shift; shift >= 0; shift -= 8) {
      for (int b = tid; b < 256; b += kSelThreads) hist[b] = 0;
      __syncthreads();
      const unsigned long long prefix = s_prefix, mask = s_mask;
      // warp-aggregated histogram: lanes holding the same digit add once (keys cluster in few
      // buckets, and same-address shared atomics serialise)
      // (warp-aggregating equal digits with __match_any_sync measured slower: 158 vs 115 us)
      scan([&](int, unsigned long long k, bool m) {
        if (m && (k & mask) == prefix) atomicAdd(&hist[(k >> shift) & 255], 1);
      });
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
        __syncwarp();  // every lane has read s_remaining before one of them rewrites it
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
  if (target > 0)
    scan([&](int i, unsigned long long k, bool m) {
      if (m && (take_all || (k & mask) <= prefix)) {
        const int slot = atomicAdd(&s_count, 1);
        if (slot < sort_len) {
          ck[slot] = k;
          ci[slot] = ids ? ids[i] : i;
        }
      }
    });
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
  *elig_out = s_elig;
  return target;
}

// One CTA per node (per-node Priority Buffers): block w selects among the slots with
// node[i] == w (node == NULL: one block over every slot); a node that is not ready selects
// nothing.  Outputs of block w: out_ids[w * cap ...], out_count[w], info[8 w + {0, 1, 4, 5}].
__global__ void __launch_bounds__(kSelThreads) k_select_topk(const unsigned long long* __restrict__ keys,
                                                             const int32_t* __restrict__ ids,
                                                             const int32_t* __restrict__ node,
                                                             const uint8_t* __restrict__ node_ready, int n, int cap,
                                                             int32_t* __restrict__ out_ids, int32_t* __restrict__ out_count,
                                                             int32_t* __restrict__ out_nan, uint32_t* __restrict__ info,
                                                             unsigned long long* __restrict__ sel_keys,
                                                             int32_t* __restrict__ sel_ids, int sort_len) {
  extern __shared__ __align__(16) uint8_t sm[];
  unsigned long long* ck = reinterpret_cast<unsigned long long*>(sm);       // [sort_len]
  int32_t* ci = reinterpret_cast<int32_t*>(ck + sort_len);                  // [sort_len]
  const int tid = threadIdx.x;
  const int w = blockIdx.x;
  const bool ready = !node_ready || node_ready[w];
  out_ids += static_cast<size_t>(w) * cap;
  if (out_count) out_count += w;
  if (sel_keys) sel_keys += static_cast<size_t>(w) * cap;
  if (sel_ids) sel_ids += static_cast<size_t>(w) * cap;
  uint32_t* info_w = info + 8 * w;
  int elig = 0;
  const int target = cta_topk_sorted(keys, ids, node, w, ready, n, cap, sort_len, ck, ci, &elig);
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
    info_w[0] = static_cast<uint32_t>(thr);
    info_w[1] = static_cast<uint32_t>(thr >> 32);
    info_w[4] = static_cast<uint32_t>(target);
    info_w[5] = static_cast<uint32_t>(elig);
    if (out_nan && w == 0) *out_nan = static_cast<int32_t>(info[6]);
  }
}

// ------------------------------------------------------------------------------ cluster select
// The single-node select (elis_isrtf_select) over a cluster of C <= 16 CTAs (C = ceil(n / 4096)):
// CTA r scans slots [r s, r s + s) (s = ceil(n / C); re-read from L1 every pass), and the
// cluster agrees on every radix decision through DSMEM -- each CTA publishes its partial
// (eligible count, min / max key; a 256-bin histogram per 8-bit digit pass) in its own shared
// memory, one cluster barrier, then every CTA sums the C partials in rank order and takes the
// same decision.  Winners (masked prefix <= the decided prefix) are written straight into CTA
// 0's shared memory at their CTA's offset (rank-ordered prefix of the per-CTA counts), CTA 0
// sorts them (bitonic) and writes the batch; every CTA writes the preemption flags of its own
// slots (running && !selected) in the same launch.  Keys are unique, so the result is the exact
// (deterministic) top-cap whatever the cluster size.
constexpr int kSelClusterMax = 16, kSelClusterSlice = 4096;
__global__ void __launch_bounds__(kSelThreads, 1)
    k_select_cluster(const unsigned long long* __restrict__ keys, int n, int cap, int sort_len,
                     int32_t* __restrict__ out_ids, int32_t* __restrict__ out_count, int32_t* __restrict__ out_nan,
                     const uint8_t* __restrict__ running, uint8_t* __restrict__ out_preempted,
                     uint32_t* __restrict__ info, unsigned long long* __restrict__ sel_keys,
                     int32_t* __restrict__ sel_ids) {
  extern __shared__ __align__(16) uint8_t sm[];
  unsigned long long* ck = reinterpret_cast<unsigned long long*>(sm);  // [sort_len] (CTA 0)
  int32_t* ci = reinterpret_cast<int32_t*>(ck + sort_len);             // [sort_len]
  __shared__ int hist[2][256];
  __shared__ int tot[256];
  __shared__ unsigned long long s_min, s_max, g_prefix, g_mask;
  __shared__ int s_elig, s_cnt, s_cursor, g_elig, g_remaining, g_digit, g_done, g_off, g_total;
  const int tid = threadIdx.x, lane = lane_id();
  const int C = static_cast<int>(gridDim.x);   // the whole grid is one cluster
  const int r = static_cast<int>(cluster_ctarank());
  const int slice = (n + C - 1) / C;
  const int lo = min(n, r * slice), hi = min(n, lo + slice);
  auto scan = [&](auto&& fn) {   // this CTA's slots, kSelBatch loads in flight per thread
    for (int i0 = lo; i0 < hi; i0 += kSelBatch * kSelThreads) {
      unsigned long long kb[kSelBatch];
#pragma unroll
      for (int u = 0; u < kSelBatch; ++u) {
        const int i = i0 + u * kSelThreads + tid;
        kb[u] = i < hi ? keys[i] : KEY_NONE;
      }
#pragma unroll
      for (int u = 0; u < kSelBatch; ++u) {
        const int i = i0 + u * kSelThreads + tid;
        if (i < hi) fn(i, kb[u]);
      }
    }
  };
  // DSMEM address of this CTA's variable `v` in CTA q
  auto peer = [](const void* v, int q) { return mapa_shared(smem_u32(v), static_cast<uint32_t>(q)); };
  auto ld_u64 = [](uint32_t a) {
    unsigned long long x;
    asm volatile("ld.shared::cluster.u64 %0, [%1];" : "=l"(x) : "r"(a) : "memory");
    return x;
  };
  auto ld_s32 = [](uint32_t a) {
    int x;
    asm volatile("ld.shared::cluster.s32 %0, [%1];" : "=r"(x) : "r"(a) : "memory");
    return x;
  };
  if (tid == 0) { s_min = KEY_NONE; s_max = 0; s_elig = 0; s_cnt = 0; }
  for (int b = tid; b < 256; b += kSelThreads) hist[0][b] = hist[1][b] = 0;
  __syncthreads();
  // ---- eligible count, min / max key over the cluster
  {
    int e = 0;
    unsigned long long kmin = KEY_NONE, kmax = 0;
    scan([&](int, unsigned long long k) {
      if (k != KEY_NONE) { ++e; kmin = k < kmin ? k : kmin; kmax = k > kmax ? k : kmax; }
    });
    e = __reduce_add_sync(0xffffffffu, e);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long a = __shfl_xor_sync(0xffffffffu, kmin, o), b = __shfl_xor_sync(0xffffffffu, kmax, o);
      kmin = a < kmin ? a : kmin;
      kmax = b > kmax ? b : kmax;
    }
    if (lane == 0 && e) {
      atomicAdd(&s_elig, e);
      atomicMin(&s_min, kmin);
      atomicMax(&s_max, kmax);
    }
  }
  cluster_sync_all();
  if (tid == 0) {
    int e = 0;
    unsigned long long mn = KEY_NONE, mx = 0;
    for (int q = 0; q < C; ++q) {
      e += ld_s32(peer(&s_elig, q));
      const unsigned long long a = ld_u64(peer(&s_min, q)), b = ld_u64(peer(&s_max, q));
      mn = a < mn ? a : mn;
      mx = b > mx ? b : mx;
    }
    g_elig = e;
    const int target = min(cap, e);
    g_remaining = target;
    g_done = 0;
    g_prefix = 0;
    g_mask = 0;
    g_digit = 56;  // start shift
    if (target > 0 && target < e) {  // >= 2 distinct (unique) keys: the radix starts at the first differing byte
      const int top = 63 - __clzll(static_cast<long long>(mn ^ mx));
      g_digit = (top >> 3) << 3;
      if (g_digit < 56) {
        g_mask = ~((1ull << (g_digit + 8)) - 1ull);
        g_prefix = mn & g_mask;
      }
    }
  }
  __syncthreads();
  const int elig = g_elig, target = min(cap, elig);
  const bool take_all = target == elig;
  // ---- MSB-first 8-bit radix select of the target-th key, decided identically by every CTA
  if (target > 0 && !take_all) {
    int pass = 0;
    for (int shift = g_digit; shift >= 0; shift -= 8, ++pass) {
      int* h = hist[pass & 1];
      const unsigned long long prefix = g_prefix, mask = g_mask;
      scan([&](int, unsigned long long k) {
        if (k != KEY_NONE && (k & mask) == prefix) atomicAdd(&h[(k >> shift) & 255], 1);
      });
      cluster_sync_all();  // every CTA's histogram of this pass is complete (and the pass-2 buffer free)
      for (int b = tid; b < 256; b += kSelThreads) {
        int s = 0;
        for (int q = 0; q < C; ++q) s += ld_s32(peer(&h[b], q));
        tot[b] = s;
      }
      __syncthreads();
      if (tid < 32) {
        int c[8], t = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) { c[q] = tot[8 * tid + q]; t += c[q]; }
        int incl = t;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, incl, o);
          if (tid >= o) incl += y;
        }
        const int excl = incl - t, need = g_remaining;
        __syncwarp();  // every lane has read the shared decision state before one of them rewrites it
        if (need > excl && need <= incl) {
          int run = excl;
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            if (need > run && need <= run + c[q]) {
              g_prefix = prefix | (static_cast<unsigned long long>(8 * tid + q) << shift);
              g_mask = mask | (0xFFull << shift);
              g_remaining = need - run;
              g_done = (c[q] == need - run) ? 1 : 0;
            }
            run += c[q];
          }
        }
      }
      // the other buffer is reused next pass: zero it (its readers finished before this pass's barrier)
      for (int b = tid; b < 256; b += kSelThreads) hist[(pass + 1) & 1][b] = 0;
      __syncthreads();
      if (g_done) break;
    }
  }
  const unsigned long long prefix = g_prefix, mask = g_mask;
  auto selected = [&](unsigned long long k) { return target > 0 && k != KEY_NONE && (take_all || (k & mask) <= prefix); };
  // ---- winners: count, rank-ordered offsets, stores into CTA 0's arrays; preemption flags
  int cnt = 0;
  scan([&](int i, unsigned long long k) {
    const bool s = selected(k);
    cnt += s;
    if (out_preempted) out_preempted[i] = (running && running[i] && !s) ? 1 : 0;
  });
  cnt = __reduce_add_sync(0xffffffffu, cnt);
  if (lane == 0 && cnt) atomicAdd(&s_cnt, cnt);
  cluster_sync_all();
  if (tid == 0) {
    int off = 0, all = 0;
    for (int q = 0; q < C; ++q) {
      const int c = ld_s32(peer(&s_cnt, q));
      if (q < r) off += c;
      all += c;
    }
    g_off = off;
    g_total = all;
    s_cursor = 0;  // (s_cnt stays intact: the peers read it after the same barrier)
  }
  __syncthreads();
  const uint32_t ck0 = peer(ck, 0), ci0 = peer(ci, 0);
  scan([&](int i, unsigned long long k) {
    if (selected(k)) {
      const int slot = g_off + atomicAdd(&s_cursor, 1);
      if (slot < sort_len) {
        asm volatile("st.shared::cluster.u64 [%0], %1;" ::"r"(ck0 + 8u * slot), "l"(k) : "memory");
        asm volatile("st.shared::cluster.s32 [%0], %1;" ::"r"(ci0 + 4u * slot), "r"(i) : "memory");
      }
    }
  });
  cluster_sync_all();  // CTA 0 holds every winner
  if (r == 0) {
    for (int i = g_total + tid; i < sort_len; i += kSelThreads) {
      ck[i] = KEY_NONE;
      ci[i] = -1;
    }
    __syncthreads();
    for (int size = 2; size <= sort_len; size <<= 1) {
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        for (int i = tid; i < sort_len / 2; i += kSelThreads) {
          const int a = 2 * i - (i & (stride - 1)), b = a + stride;
          const bool up = ((a & size) == 0);
          const unsigned long long ka = ck[a], kb = ck[b];
          if ((ka > kb) == up) {
            ck[a] = kb; ck[b] = ka;
            const int t = ci[a]; ci[a] = ci[b]; ci[b] = t;
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
      const unsigned long long thr = target > 0 ? ck[target - 1] : 0ull;
      info[0] = static_cast<uint32_t>(thr);
      info[1] = static_cast<uint32_t>(thr >> 32);
      info[4] = static_cast<uint32_t>(target);
      info[5] = static_cast<uint32_t>(elig);
      if (out_nan) *out_nan = static_cast<int32_t>(info[6]);
    }
  }
}

// out[i] = running[i] && !selected[i]; with nodes, against the slot's own node's threshold and
// only on ready nodes (a busy node's running jobs are mid-window); node ids outside
// [0, num_nodes) are never flagged.
__global__ void k_preempt(const unsigned long long* __restrict__ keys, const uint8_t* __restrict__ running,
                          const int32_t* __restrict__ node, const uint8_t* __restrict__ node_ready, int num_nodes,
                          int n, const uint32_t* __restrict__ info, uint8_t* __restrict__ out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int w = node ? node[i] : 0;
    bool flag = false;
    if (running && running[i] && w >= 0 && w < num_nodes && (!node_ready || node_ready[w])) {
      const uint32_t* iw = info + 8 * w;
      const unsigned long long thr = (static_cast<unsigned long long>(iw[1]) << 32) | iw[0];
      const unsigned long long k = keys[i];
      flag = !(iw[4] > 0 && k != KEY_NONE && k <= thr);
    }
    out[i] = flag ? 1 : 0;
  }
}

// Greedy least-loaded assignment (Alg. 1 line 3) of n_new jobs in arrival order,
// computed in parallel: job j takes the j-th smallest pair (load_w + k, w), k >= 0, in
// lexicographic order -- exactly the node the sequential argmin (ties -> lowest id) picks.
// count(v) = sum_w max(0, v - load_w) pairs lie below level v; job j's level v is the largest
// with count(v) <= j and its node the (j - count(v))-th, in id order, with load_w <= v.
__global__ void __launch_bounds__(1024) k_assign_nodes(int32_t* __restrict__ load, int W, int n_new,
                                                       int32_t* __restrict__ out_node) {
  __shared__ long long s_load[kMaxNodes];
  __shared__ long long s_lo;
  for (int w = threadIdx.x; w < W; w += blockDim.x) s_load[w] = load[w];
  __syncthreads();
  if (threadIdx.x == 0) {
    long long lo = s_load[0];
    for (int w = 1; w < W; ++w) lo = s_load[w] < lo ? s_load[w] : lo;
    s_lo = lo;
  }
  __syncthreads();
  const long long lo = s_lo;
  auto count_below = [&](long long v) {
    long long c = 0;
    for (int w = 0; w < W; ++w) c += v > s_load[w] ? v - s_load[w] : 0;
    return c;
  };
  auto level = [&](long long j, long long* r) {  // level of job j and its rank within the level
    long long a = lo, b = lo + j + 1;           // count(a) = 0 <= j < j + 1 <= count(b)
    while (b - a > 1) {
      const long long mid = (a + b) >> 1;
      if (count_below(mid) <= j) a = mid; else b = mid;
    }
    *r = j - count_below(a);
    return a;
  };
  for (int j = threadIdx.x; j < n_new; j += blockDim.x) {
    long long r;
    const long long v = level(j, &r);
    int pick = -1;
    for (int w = 0; w < W && pick < 0; ++w)
      if (s_load[w] <= v && r-- == 0) pick = w;
    out_node[j] = pick;
  }
  if (n_new > 0) {
    long long r_last;
    const long long v_last = level(n_new - 1, &r_last);
    for (int w = threadIdx.x; w < W; w += blockDim.x) {
      long long rank = 0;  // nodes before w at level v_last
      for (int u = 0; u < w; ++u) rank += s_load[u] <= v_last;
      const long long add = (v_last > s_load[w] ? v_last - s_load[w] : 0) + (s_load[w] <= v_last && rank <= r_last);
      load[w] = static_cast<int32_t>(s_load[w] + add);
    }
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

// ---- multi-GPU select over peer memory (SURVEY.md 8e "B200-native stretch")
//
// The whole cross-rank exchange of Sec. 8a row a13 in one kernel: each rank's local top-cap
// candidates are stored straight into every rank's symmetric region over NVLink / NVSwitch
// (plain st.global through CUDA-IPC-mapped pointers), published by a release store of the call's
// epoch into the destination's flag slot, and every rank acquires all `world` flags and runs the
// same deterministic merge -- the NCCL all-gather, its pack / unpack kernels and two extra
// select launches disappear.  Regions are double-buffered by epoch parity: rank s can only
// write epoch e + 2 into a parity slot after it has seen every rank's epoch e + 1 flag, i.e.
// after every rank finished reading epoch e from that slot.
constexpr size_t kPeerSlots = static_cast<size_t>(kMaxPeers) * kMaxBatchCap;   // candidates per parity
ELIS_DEV unsigned long long* peer_keys(uint8_t* region, int par) {
  return reinterpret_cast<unsigned long long*>(region) + par * kPeerSlots;
}
ELIS_DEV int32_t* peer_ids(uint8_t* region, int par) {
  return reinterpret_cast<int32_t*>(region + 2 * kPeerSlots * 8) + par * kPeerSlots;
}
ELIS_DEV uint32_t* peer_flags(uint8_t* region, int par) {
  return reinterpret_cast<uint32_t*>(region + 2 * kPeerSlots * 12) + par * kMaxPeers;
}

__global__ void __launch_bounds__(kSelThreads)
    k_select_dist_peer(const unsigned long long* __restrict__ keys, const uint32_t* __restrict__ local_info,
                       int n_local, int cap, int global_offset, PeerArgs pa, const uint8_t* __restrict__ running,
                       unsigned long long* mkeys, int32_t* mids, int32_t* __restrict__ out_ids,
                       int32_t* __restrict__ out_count, int32_t* __restrict__ out_nan,
                       uint8_t* __restrict__ out_preempted, uint32_t* __restrict__ info, uint32_t* __restrict__ err,
                       int sort_len) {
  extern __shared__ __align__(16) uint8_t sm[];
  unsigned long long* ck = reinterpret_cast<unsigned long long*>(sm);       // [sort_len]
  int32_t* ci = reinterpret_cast<int32_t*>(ck + sort_len);                  // [sort_len]
  __shared__ int s_timeout;
  const int tid = threadIdx.x;
  uint32_t epoch = *pa.epoch + 1u;
  if (epoch == 0u) epoch = 1u;     // never 0: the regions' initial flag value
  const int par = static_cast<int>(epoch & 1u);
  if (tid == 0) s_timeout = 0;
  // 1. this rank's top-cap (ids = local slot index)
  int elig = 0;
  const int target = cta_topk_sorted(keys, nullptr, nullptr, 0, true, n_local, cap, sort_len, ck, ci, &elig);
  // 2. push them into every rank's region (own included) at [par][rank * cap + j], global ids
  for (int r = 0; r < pa.world; ++r) {
    unsigned long long* pk = peer_keys(pa.region[r], par) + static_cast<size_t>(pa.rank) * cap;
    int32_t* pi = peer_ids(pa.region[r], par) + static_cast<size_t>(pa.rank) * cap;
    for (int j = tid; j < cap; j += kSelThreads) {
      const bool v = j < target;
      pk[j] = v ? ck[j] : KEY_NONE;
      pi[j] = v ? ci[j] + global_offset : -1;
    }
  }
  __syncthreads();  // every thread's peer stores precede the fence + flag store below
  if (tid < pa.world) {
    __threadfence_system();
    st_release_sys_u32(peer_flags(pa.region[tid], par) + pa.rank, epoch);
  }
  // 3. acquire every rank's flag of this epoch (bounded: a missing rank sets ERR_PEER_TIMEOUT)
  if (tid < pa.world) {
    const uint32_t* f = peer_flags(pa.region[pa.rank], par) + tid;
    const unsigned long long t0 = peer_globaltimer();
    while (static_cast<int32_t>(ld_acquire_sys_u32(f) - epoch) < 0) {
      __nanosleep(32);
      if (peer_globaltimer() - t0 > kPeerTimeoutNs) {
        atomicOr(err, ERR_PEER_TIMEOUT);
        s_timeout = 1;
        break;
      }
    }
  }
  __syncthreads();
  const int total = pa.world * cap;
  int got = 0;
  if (!s_timeout) {
    // 4. copy the world x cap candidates (written by other GPUs during this kernel) with
    //    cache-volatile loads into local scratch, then the same merge on every rank
    const unsigned long long* rk = peer_keys(pa.region[pa.rank], par);
    const int32_t* ri = peer_ids(pa.region[pa.rank], par);
    for (int j = tid; j < total; j += kSelThreads) {
      mkeys[j] = __ldcv(rk + j);
      mids[j] = __ldcv(ri + j);
    }
    __syncthreads();
    int elig2 = 0;
    got = cta_topk_sorted(mkeys, mids, nullptr, 0, true, total, cap, sort_len, ck, ci, &elig2);
  }
  // 5. outputs: global ids in priority order, count, merged threshold, this rank's preempt flags
  for (int j = tid; j < cap; j += kSelThreads) out_ids[j] = j < got ? ci[j] : -1;
  const unsigned long long thr = got > 0 ? ck[got - 1] : 0ull;
  if (tid == 0) {
    *pa.epoch = epoch;  // read by the next call's kernel (stream order)
    if (out_count) *out_count = got;
    if (out_nan) *out_nan = static_cast<int32_t>(local_info[6]);
    info[0] = static_cast<uint32_t>(thr);
    info[1] = static_cast<uint32_t>(thr >> 32);
    info[4] = static_cast<uint32_t>(got);
  }
  if (out_preempted)
    for (int i = tid; i < n_local; i += kSelThreads) {
      bool flag = false;
      if (running && running[i]) {
        const unsigned long long k = keys[i];
        flag = !(got > 0 && k != KEY_NONE && k <= thr);
      }
      out_preempted[i] = flag ? 1 : 0;
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
                             uint32_t order_offset, Starvation sv, unsigned long long* keys, uint32_t* info,
                             cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(info, 0, 8 * sizeof(uint32_t), st);
  if (e != cudaSuccess || n <= 0) return e;
  int blocks = (n + 255) / 256;
  if (blocks > 1184) blocks = 1184;
  k_make_keys<<<blocks, 256, 0, st>>>(pred, generated, order, running, n, policy, allow_preempt, head_predicts_total,
                                      order_offset, sv, keys, info);
  return cudaGetLastError();
}

cudaError_t launch_select_topk(const unsigned long long* keys, const int32_t* ids, int n, int cap, int32_t* out_ids,
                               int32_t* out_count, int32_t* out_nan, SelectScratch sc, cudaStream_t st) {
  return launch_select_topk_nodes(keys, ids, nullptr, nullptr, 1, n, cap, out_ids, out_count, out_nan, sc, st);
}

cudaError_t launch_select_topk_nodes(const unsigned long long* keys, const int32_t* ids, const int32_t* node,
                                     const uint8_t* node_ready, int num_nodes, int n, int cap, int32_t* out_ids,
                                     int32_t* out_count, int32_t* out_nan, SelectScratch sc, cudaStream_t st) {
  if (num_nodes < 1 || num_nodes > kMaxNodes) return cudaErrorInvalidValue;
  const int sort_len = next_pow2(cap < 2 ? 2 : cap);
  const size_t smem = static_cast<size_t>(sort_len) * (sizeof(unsigned long long) + sizeof(int32_t));
  if (!attr_once(reinterpret_cast<const void*>(k_select_topk))) {  // per device
    cudaError_t e = cudaFuncSetAttribute(k_select_topk, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(kMaxBatchCap * 12 + 1024));
    if (e != cudaSuccess) return e;
  }
  k_select_topk<<<num_nodes, kSelThreads, smem, st>>>(keys, ids, node, node_ready, n, cap, out_ids, out_count,
                                                      out_nan, sc.info, node ? nullptr : sc.sel_keys,
                                                      node ? nullptr : sc.sel_ids, sort_len);
  return cudaGetLastError();
}

cudaError_t launch_select_cluster(const unsigned long long* keys, int n, int cap, int32_t* out_ids, int32_t* out_count,
                                  int32_t* out_nan, const uint8_t* running, uint8_t* out_preempted, SelectScratch sc,
                                  cudaStream_t st) {
  const int sort_len = next_pow2(cap < 2 ? 2 : cap);
  const size_t smem = static_cast<size_t>(sort_len) * (sizeof(unsigned long long) + sizeof(int32_t));
  if (!attr_once(reinterpret_cast<const void*>(k_select_cluster))) {  // per device
    cudaError_t e = cudaFuncSetAttribute(k_select_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(kMaxBatchCap * 12 + 1024));
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_select_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  int C = (n + kSelClusterSlice - 1) / kSelClusterSlice;
  C = C < 1 ? 1 : (C > kSelClusterMax ? kSelClusterMax : C);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(C);
  cfg.blockDim = dim3(kSelThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, k_select_cluster, keys, n, cap, sort_len, out_ids, out_count, out_nan,
                                     running, out_preempted, sc.info, sc.sel_keys, sc.sel_ids);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t launch_preempt_flags(const unsigned long long* keys, const uint8_t* running, int n, const uint32_t* info,
                                 uint8_t* out_preempted, cudaStream_t st) {
  return launch_preempt_flags_nodes(keys, running, nullptr, nullptr, 1, n, info, out_preempted, st);
}

cudaError_t launch_preempt_flags_nodes(const unsigned long long* keys, const uint8_t* running, const int32_t* node,
                                       const uint8_t* node_ready, int num_nodes, int n, const uint32_t* info,
                                       uint8_t* out_preempted, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  int blocks = (n + 255) / 256;
  if (blocks > 1184) blocks = 1184;
  k_preempt<<<blocks, 256, 0, st>>>(keys, running, node, node_ready, num_nodes, n, info, out_preempted);
  return cudaGetLastError();
}

cudaError_t launch_assign_nodes(int32_t* load, int num_nodes, int n_new, int32_t* out_node, cudaStream_t st) {
  if (num_nodes < 1 || num_nodes > kMaxNodes) return cudaErrorInvalidValue;
  if (n_new <= 0) return cudaSuccess;
  k_assign_nodes<<<1, 1024, 0, st>>>(load, num_nodes, n_new, out_node);
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

size_t peer_region_bytes(int max_pairs) {
  return peer_pred_offset() + 2 * kMaxPeers * 2 * sizeof(uint32_t) + 2 * static_cast<size_t>(kMaxPeers) * max_pairs * 8;
}

cudaError_t launch_select_dist_peer(const unsigned long long* keys, const uint32_t* local_info, int n_local, int cap,
                                    int global_offset, PeerArgs pa, const uint8_t* running,
                                    unsigned long long* mkeys, int32_t* mids, int32_t* out_ids, int32_t* out_count,
                                    int32_t* out_nan, uint8_t* out_preempted, uint32_t* info, uint32_t* err,
                                    cudaStream_t st) {
  if (pa.world < 1 || pa.world > kMaxPeers || pa.rank < 0 || pa.rank >= pa.world || cap < 1 || cap > kMaxBatchCap)
    return cudaErrorInvalidValue;
  const int sort_len = next_pow2(cap < 2 ? 2 : cap);
  const size_t smem = static_cast<size_t>(sort_len) * (sizeof(unsigned long long) + sizeof(int32_t));
  if (!attr_once(reinterpret_cast<const void*>(k_select_dist_peer))) {  // per device
    cudaError_t e = cudaFuncSetAttribute(k_select_dist_peer, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(kMaxBatchCap * 12 + 1024));
    if (e != cudaSuccess) return e;
  }
  k_select_dist_peer<<<1, kSelThreads, smem, st>>>(keys, local_info, n_local, cap, global_offset, pa, running, mkeys,
                                                   mids, out_ids, out_count, out_nan, out_preempted, info, err,
                                                   sort_len);
  return cudaGetLastError();
}

}  // namespace elis
