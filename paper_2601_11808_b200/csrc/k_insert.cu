// k_insert.cu — batched insert: claim -> assign -> reserve -> append.
//
// Paper: Alg. 1 Insert and Alg. 2.  The paper runs
// one thread per vector with CAS slot reservation and CAS head publication.
// Here a batch is stream-ordered, so reservation is done for the whole batch
// at once (no CAS retries, no leaked slabs — readings C10, C11):
//   k_claim        id range / shard / live-duplicate checks; atomicMin claim
//                  on the id resolves in-batch duplicates (lowest position wins)
//   (k_coarse.cu)  exact nearest centroid (reading C2)
//   k_chunk_rank   stable within-list rank of each item, per 1024-item chunk
//   k_chunk_prefix per list: exclusive prefix of chunk counts -> batch rank
//   k_reserve      one CTA scans lists in ascending order: tail-slab free
//                  slots, slabs needed, slabs granted from the free stack
//                  (Eq. 2's atomicSub(P_top) done once per batch)
//   k_dir_update   warp per list: append the granted slabs to the list
//                  directory, initialise their metadata
//   k_append       warp per item: payload, id, ATT entry, then the validity
//                  bit is published with a release fence
#include <cuda_fp16.h>

#include "sivf_host.h"

namespace sivf {

namespace {

// The split-fp16 scan copy of one vector (D > 128; warp per vector, recg_off()):
// e = 15 - exponent(max |x|) puts every scaled value below 2^15 (finite in fp16),
// x 2^e = hi + lo with hi = fp16_rn(x 2^e) and lo = fp16_rn(x 2^e - hi) (the
// difference is exact in fp32); slab_xs = 2^-e undoes the scale.
__device__ __forceinline__ void append_split_copy(const DevState& st, int slab, int o, const float* xr, int lane) {
  float mx = 0.f;
  for (int d = lane; d < st.D; d += 32) mx = fmaxf(mx, fabsf(xr[d]));
  mx = __uint_as_float(__reduce_max_sync(kFull, __float_as_uint(mx)));  // non-negative: uint order
  int e = 0;
  if (mx > 0.f && mx <= 3.4e38f) {
    int ex;
    frexpf(mx, &ex);  // mx in [2^(ex-1), 2^ex)
    e = 15 - ex;
    e = e < -120 ? -120 : e > 120 ? 120 : e;
  }
  unsigned char* base = reinterpret_cast<unsigned char*>(st.payload_g) + (size_t)slab * recg_bytes(st.Dg);
  for (int c8 = lane; c8 < (st.Dg >> 3); c8 += 32) {
    uint32_t hw[4], lw[4];
#pragma unroll
    for (int e2 = 0; e2 < 4; ++e2) {
      const int d = 8 * c8 + 2 * e2;
      const float s0 = ldexpf(d < st.D ? xr[d] : 0.f, e), s1 = ldexpf(d + 1 < st.D ? xr[d + 1] : 0.f, e);
      const __half h0 = __float2half_rn(s0), h1 = __float2half_rn(s1);
      const __half l0 = __float2half_rn(s0 - __half2float(h0)), l1 = __float2half_rn(s1 - __half2float(h1));
      const __half2 hh = __halves2half2(h0, h1), ll = __halves2half2(l0, l1);
      hw[e2] = *reinterpret_cast<const uint32_t*>(&hh);
      lw[e2] = *reinterpret_cast<const uint32_t*>(&ll);
    }
    *reinterpret_cast<uint4*>(base + recg_off(st.Dg, o, 8 * c8, 0)) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
    *reinterpret_cast<uint4*>(base + recg_off(st.Dg, o, 8 * c8, 1)) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
  }
  if (lane == 0) st.slab_xs[(size_t)slab * kSlot + o] = ldexpf(1.f, -e);
}

__global__ void k_claim(DevState st, const int64_t* __restrict__ ids, int64_t n, int32_t* __restrict__ status,
                        int64_t* __restrict__ lid_out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int64_t id = ids[i];
  int s = SIVF_ST_OK;
  int64_t lid = -1;
  if (id < 0 || id >= st.cap) {
    s = SIVF_ST_ID_OUT_OF_RANGE;
  } else if (id % st.G != st.rank) {
    s = SIVF_ST_WRONG_SHARD;
  } else {
    lid = id / st.G;
    if (st.att[lid] != kAttInvalid) s = SIVF_ST_DUPLICATE;
    else atomicMin(&st.claim[lid], (int32_t)i);
  }
  status[i] = s;
  lid_out[i] = (s == SIVF_ST_OK) ? lid : -1;
}

// Stable rank of each OK row within its list, for one chunk of 1024 rows.
// Sort (list << 11 | pos) keys in shared memory (bitonic), then rank = pos in
// the sorted run.  Chunk counts go to hist[chunk][list].
__global__ void __launch_bounds__(1024) k_chunk_rank(const unsigned long long* __restrict__ best, int64_t n,
                                                     int32_t* __restrict__ status, const int64_t* __restrict__ lid,
                                                     const int32_t* __restrict__ claim, int check_claim,
                                                     int32_t* __restrict__ list_out, int32_t* __restrict__ rank_out,
                                                     int32_t* __restrict__ hist, int nlist) {
  __shared__ uint32_t keys[1024];
  __shared__ int32_t wmax[32];
  const int t = threadIdx.x;
  const int64_t base = (int64_t)blockIdx.x * 1024;
  const int64_t i = base + t;
  uint32_t key = 0xffffffffu;
  if (i < n) {
    int s = status[i];
    if (s == SIVF_ST_OK && check_claim && claim[lid[i]] != (int32_t)i) {
      s = SIVF_ST_DUPLICATE;  // a lower batch position claimed this id (reading C12)
      status[i] = s;
    }
    int l = -1;
    if (s == SIVF_ST_OK) {
      l = (int)(best[i] & 0xffffffffull);
      key = ((uint32_t)l << 11) | (uint32_t)t;
    }
    list_out[i] = l;
  }
  keys[t] = key;
  __syncthreads();
  for (int size = 2; size <= 1024; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      int p = t ^ stride;
      if (p > t) {
        uint32_t a = keys[t], b = keys[p];
        bool up = (t & size) == 0;
        if ((a > b) == up) {
          keys[t] = b;
          keys[p] = a;
        }
      }
      __syncthreads();
    }
  }
  const uint32_t k = keys[t];
  const bool valid = k != 0xffffffffu;
  const uint32_t l = k >> 11;
  const bool head = valid && (t == 0 || (keys[t - 1] >> 11) != l);
  // inclusive max-scan of (head ? t : 0) -> start of my run
  int v = head ? t : 0;
  const int lane = t & 31, w = t >> 5;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    int o = __shfl_up_sync(kFull, v, off);
    if (lane >= off) v = max(v, o);
  }
  if (lane == 31) wmax[w] = v;
  __syncthreads();
  if (w == 0) {
    int x = wmax[lane];
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      int o = __shfl_up_sync(kFull, x, off);
      if (lane >= off) x = max(x, o);
    }
    wmax[lane] = x;
  }
  __syncthreads();
  if (w > 0) v = max(v, wmax[w - 1]);
  if (valid) {
    const int start = v;
    const int pos = (int)(k & 2047u);
    rank_out[base + pos] = t - start;
    const bool tail = (t == 1023) || (keys[t + 1] >> 11) != l || keys[t + 1] == 0xffffffffu;
    if (tail) hist[(int64_t)blockIdx.x * nlist + l] = t - start + 1;
  }
}

// Warp per list: 32 chunks per step (independent loads), a warp scan, the running
// carry (was one thread per list walking the chunks one dependent load at a time:
// 47 us per 64k batch, 0.5 ms per 1M batch).
__global__ void __launch_bounds__(256) k_chunk_prefix(int32_t* __restrict__ hist, int64_t nchunks, int nlist,
                                                      int32_t* __restrict__ cnt) {
  const int lane = threadIdx.x & 31;
  const int l = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  if (l >= nlist) return;  // warp-uniform
  int run = 0;
  for (int64_t c0 = 0; c0 < nchunks; c0 += 32) {
    const int64_t c = c0 + lane;
    const int h = c < nchunks ? hist[c * nlist + l] : 0;
    int x = h;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(kFull, x, o);
      if (lane >= o) x += y;
    }
    if (c < nchunks) hist[c * nlist + l] = run + x - h;
    run += __shfl_sync(kFull, x, 31);
  }
  if (lane == 0) cnt[l] = run;
}

// Block-wide exclusive scan of one value per thread (1024 threads); returns the
// exclusive prefix, *total receives the block sum.  All threads must call it.
__device__ __forceinline__ long long block_excl_scan(long long v, long long* ws /*[32]*/, long long* total) {
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  long long x = v;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const long long o = __shfl_up_sync(kFull, x, off);
    if (lane >= off) x += o;
  }
  if (lane == 31) ws[w] = x;
  __syncthreads();
  if (w == 0) {
    long long y = ws[lane];
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const long long o = __shfl_up_sync(kFull, y, off);
      if (lane >= off) y += o;
    }
    ws[lane] = y;
  }
  __syncthreads();
  const long long excl = (w > 0 ? ws[w - 1] : 0) + x - v;
  *total = ws[31];
  __syncthreads();
  return excl;
}

// Single CTA: lists in ascending order share the free stack (reading C33 /
// SURVEY a4 policy).  Slabs for list l: free_stack[newbase_l, newbase_l+granted_l).
// Then the directory space: every list that outgrows its directory takes a new
// one of max(2 cap, len + g, 8) entries from the active arena half
// (k_dir_update).  If that would not fit, every directory is first compacted
// into the idle half with cap = max(8, 2 (len + g)) (sum <= 2 num_slabs + 8 nlist
// <= dir_half), so no list grows in this batch and the arena never overflows
// however the lists' peaks drift over time.
__global__ void __launch_bounds__(1024) k_reserve(DevState st, const int32_t* __restrict__ cnt,
                                                  int32_t* __restrict__ tail_free, int32_t* __restrict__ tail_slab,
                                                  int32_t* __restrict__ granted, int32_t* __restrict__ newbase,
                                                  int64_t* __restrict__ newoff) {
  __shared__ long long ws[32];
  __shared__ long long carry_s;
  __shared__ int32_t F;
  const int t = threadIdx.x;
  if (t == 0) {
    carry_s = 0;
    F = st.ictr[I_FREE_TOP];
  }
  __syncthreads();
  for (int l0 = 0; l0 < st.nlist; l0 += 1024) {
    const int l = l0 + t;
    int need = 0, tf = 0, ts = -1, c = 0;
    if (l < st.nlist) {
      c = cnt[l];
      int len = st.dir_len[l];
      if (len > 0) {
        ts = st.dir_arena[st.dir_off[l] + len - 1];
        tf = kSlot - (int)st.cursor[ts];
      }
      int rest = c > tf ? c - tf : 0;
      need = (rest + kSlot - 1) / kSlot;
    }
    long long tot;
    const long long excl = carry_s + block_excl_scan(need, ws, &tot);
    if (l < st.nlist) {
      int64_t avail = (int64_t)F - excl;
      int g = (int)(avail <= 0 ? 0 : (avail < need ? avail : need));
      tail_free[l] = tf;
      tail_slab[l] = ts;
      granted[l] = g;
      newbase[l] = (int32_t)(avail - g > 0 ? avail - g : 0);
    }
    if (t == 0) carry_s += tot;
    __syncthreads();
  }
  if (t == 0) {
    int64_t total = carry_s;
    st.ictr[I_FREE_TOP] = (int32_t)(total >= F ? 0 : F - total);
  }
  // directory space this batch will bump-allocate
  long long grow = 0;
  for (int l = t; l < st.nlist; l += 1024) {
    const int g = granted[l], len = st.dir_len[l], cap = st.dir_cap[l];
    if (g > 0 && len + g > cap) grow += max(max(2 * cap, len + g), 8);
  }
  long long total_grow;
  block_excl_scan(grow, ws, &total_grow);
  const int half = st.ictr[I_DIR_HALF];
  const long long bump = st.ictr[I_DIR_BUMP];
  if (bump + total_grow <= (long long)(half + 1) * st.dir_half) return;  // block-uniform
  // compaction into the idle half
  const long long base = (long long)(1 - half) * st.dir_half;
  if (t == 0) carry_s = 0;
  __syncthreads();
  for (int l0 = 0; l0 < st.nlist; l0 += 1024) {
    const int l = l0 + t;
    long long ncap = 0;
    if (l < st.nlist) {
      const int need = st.dir_len[l] + granted[l];
      ncap = need > 0 ? max(8, 2 * need) : 0;
    }
    long long tot;
    const long long excl = carry_s + block_excl_scan(ncap, ws, &tot);
    if (l < st.nlist) newoff[l] = base + excl;
    if (t == 0) carry_s += tot;
    __syncthreads();
  }
  const int lane = t & 31, w = t >> 5;
  for (int l = w; l < st.nlist; l += 32) {  // warp per list: copy the live entries
    const int len = st.dir_len[l];
    const int32_t* src = st.dir_arena + st.dir_off[l];
    int32_t* dst = st.dir_arena + newoff[l];
    for (int j = lane; j < len; j += 32) dst[j] = src[j];
  }
  __syncthreads();
  for (int l = t; l < st.nlist; l += 1024) {
    const int need = st.dir_len[l] + granted[l];
    st.dir_off[l] = newoff[l];
    st.dir_cap[l] = need > 0 ? max(8, 2 * need) : 0;
  }
  if (t == 0) {
    st.ictr[I_DIR_BUMP] = (int32_t)(base + carry_s);
    st.ictr[I_DIR_HALF] = 1 - half;
    atomicAdd(&st.ctr[C_DIRCOMPACT], 1ull);
  }
}

__global__ void k_dir_update(DevState st, const int32_t* __restrict__ cnt, const int32_t* __restrict__ tail_free,
                             const int32_t* __restrict__ tail_slab, int32_t* __restrict__ granted,
                             const int32_t* __restrict__ newbase) {
  const int lane = threadIdx.x & 31;
  const int l = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  if (l >= st.nlist) return;
  const int c = cnt[l];
  if (c == 0) return;
  const int tf = tail_free[l], g = granted[l];
  const int served = min(c, tf + kSlot * g);
  const int used_tail = min(served, tf);
  if (lane == 0 && used_tail > 0) st.cursor[tail_slab[l]] += (uint32_t)used_tail;
  if (g == 0) return;
  int len = st.dir_len[l], cap = st.dir_cap[l];
  int64_t off = st.dir_off[l];
  if (len + g > cap) {
    int ncap = max(max(2 * cap, len + g), 8);
    int64_t noff = 0;
    if (lane == 0) noff = atomicAdd(&st.ictr[I_DIR_BUMP], ncap);
    noff = __shfl_sync(kFull, noff, 0);
    if (noff + ncap > (int64_t)(st.ictr[I_DIR_HALF] + 1) * st.dir_half) {
      // unreachable: k_reserve compacts first whenever this batch's growth would
      // not fit.  Fail safe all the same: the list's new slabs are not linked and
      // its items beyond the tail slab become POOL_EXHAUSTED (k_append reads
      // granted); the stranded slabs show up as sivf_dump_state violations.
      if (lane == 0) {
        atomicAdd(&st.ctr[C_DEVERR], 1ull);
        granted[l] = 0;
      }
      return;
    }
    for (int j = lane; j < len; j += 32) st.dir_arena[noff + j] = st.dir_arena[off + j];
    off = noff;
    cap = ncap;
    if (lane == 0) {
      st.dir_off[l] = off;
      st.dir_cap[l] = cap;
    }
  }
  const int rem = served - used_tail;
  for (int j = lane; j < g; j += 32) {
    int s = st.free_stack[newbase[l] + j];
    st.dir_arena[off + len + j] = s;
    st.bitmap[s] = 0u;  // P:312 validity_bitmap <- 0
    st.slab_list[s] = l;
    st.slab_flag[s] = kFlagIntegral;  // integral (and fp16-finite) until an appended vector says otherwise
    int fill = rem - kSlot * j;
    st.cursor[s] = (uint32_t)(fill > kSlot ? kSlot : fill);
  }
  if (lane == 0) st.dir_len[l] = len + g;
}

// Warp per item: slot from (tail_free, granted, batch rank), then writes.
__global__ void __launch_bounds__(256) k_append(DevState st, const int64_t* __restrict__ ids,
                                                const float* __restrict__ X, int64_t n,
                                                int32_t* __restrict__ status, const int64_t* __restrict__ lid,
                                                const int32_t* __restrict__ list, const int32_t* __restrict__ rank,
                                                const int32_t* __restrict__ hist, const int32_t* __restrict__ tail_free,
                                                const int32_t* __restrict__ tail_slab,
                                                const int32_t* __restrict__ granted,
                                                const int32_t* __restrict__ newbase, int32_t* __restrict__ d_status,
                                                int32_t* __restrict__ d_list) {
  __shared__ int ok_cnt, ex_cnt;
  if (threadIdx.x == 0) ok_cnt = ex_cnt = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (i < n) {
    int s_ = status[i];
    int l = -1;
    if (s_ == SIVF_ST_OK) {
      l = list[i];
      const int r = hist[(i >> 10) * st.nlist + l] + rank[i];
      const int tf = tail_free[l], g = granted[l];
      const int64_t u = lid[i];
      if (r >= tf + kSlot * g) {
        s_ = SIVF_ST_POOL_EXHAUSTED;  // C9: per-item status, index unchanged
        if (lane == 0) {
          st.claim[u] = kClaimEmpty;
          atomicAdd(&ex_cnt, 1);
        }
        l = -1;
      } else {
        int slab, o;
        if (r < tf) {
          slab = tail_slab[l];
          o = kSlot - tf + r;
        } else {
          slab = st.free_stack[newbase[l] + ((r - tf) >> 5)];
          o = (r - tf) & 31;
        }
        float* dst = st.payload + (size_t)slab * kSlot * st.Dp;  // chunk c4 of slot o at pay_off()
        const float* xr = X + i * st.D;
        const int nc4 = st.Dp >> 2;
        float nrm = 0.f;
        bool integral = true, over = false;
        uint16_t* dst16 = st.payload16 ? st.payload16 + (size_t)slab * (rec16_bytes(st.Dh) >> 1) : nullptr;
        for (int c4 = lane; c4 < nc4; c4 += 32) {
          float4 v;
          if ((st.D & 3) == 0 && 4 * c4 + 3 < st.D) {
            v = reinterpret_cast<const float4*>(xr)[c4];
          } else {
            float t[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) t[e] = (4 * c4 + e < st.D) ? xr[4 * c4 + e] : 0.f;
            v = make_float4(t[0], t[1], t[2], t[3]);
          }
          *reinterpret_cast<float4*>(dst + pay_off(st.Dp, o, c4)) = v;
          if (dst16) {  // fp16 (RN) scan copy: 4 halves = one half of a 16-B chunk
            const __half2 h01 = __floats2half2_rn(v.x, v.y), h23 = __floats2half2_rn(v.z, v.w);
            *reinterpret_cast<uint2*>(dst16 + pay16_off(st.Dh, o, c4 >> 1) + 4 * (c4 & 1)) =
                make_uint2(*reinterpret_cast<const uint32_t*>(&h01), *reinterpret_cast<const uint32_t*>(&h23));
            over = over || !(fabsf(v.x) <= 65504.f && fabsf(v.y) <= 65504.f && fabsf(v.z) <= 65504.f &&
                             fabsf(v.w) <= 65504.f);
          }
          nrm = fmaf(v.x, v.x, fmaf(v.y, v.y, fmaf(v.z, v.z, fmaf(v.w, v.w, nrm))));
          integral = integral && v.x == rintf(v.x) && v.y == rintf(v.y) && v.z == rintf(v.z) && v.w == rintf(v.w) &&
                     fabsf(v.x) <= 2048.f && fabsf(v.y) <= 2048.f && fabsf(v.z) <= 2048.f && fabsf(v.w) <= 2048.f;
        }
        if (dst16)  // zero dims [Dp, Dh) of the fp16 copy
          for (int c4 = nc4 + lane; c4 < (st.Dh >> 2); c4 += 32)
            *reinterpret_cast<uint2*>(dst16 + pay16_off(st.Dh, o, c4 >> 1) + 4 * (c4 & 1)) = make_uint2(0u, 0u);
        if (st.payload_g) append_split_copy(st, slab, o, xr, lane);
#pragma unroll
        for (int off = 16; off; off >>= 1) nrm += __shfl_xor_sync(kFull, nrm, off);
        integral = __all_sync(kFull, integral);
        over = __any_sync(kFull, over);
        if (lane == 0) {
          st.slab_norm[(size_t)slab * kSlot + o] = nrm;
          if (!integral) atomicAnd(&st.slab_flag[slab], ~kFlagIntegral);
          if (over) atomicOr(&st.slab_flag[slab], kFlagF16Over);
          st.slab_ids[(size_t)slab * kSlot + o] = (uint32_t)ids[i];
          if (dst16) {  // the scan record's copies of the norm and the id
            *reinterpret_cast<float*>(reinterpret_cast<unsigned char*>(dst16) + rec16_norm_off(st.Dh, o)) = nrm;
            *reinterpret_cast<uint32_t*>(reinterpret_cast<unsigned char*>(dst16) + rec16_id_off(st.Dh, o)) =
                (uint32_t)ids[i];
          }
          st.att[u] = ((uint64_t)(uint32_t)slab << 32) | (uint32_t)o;  // Eq. att_encoding
          st.claim[u] = kClaimEmpty;
        }
        __threadfence();  // payload, id and ATT visible before the publish
        __syncwarp();
        if (lane == 0) {
          atomicOr(&st.bitmap[slab], 1u << o);  // P:300 publish
          atomicAdd(&ok_cnt, 1);
        }
      }
    }
    if (lane == 0) {
      if (d_status) d_status[i] = s_;
      if (d_list) d_list[i] = l;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (ok_cnt) {
      atomicAdd(&st.ctr[C_INSERTED], (unsigned long long)ok_cnt);
      atomicAdd(&st.ctr[C_LIVE], (unsigned long long)ok_cnt);
    }
    if (ex_cnt) atomicAdd(&st.ctr[C_EXHAUSTED], (unsigned long long)ex_cnt);
  }
}

}  // namespace

cudaError_t launch_stable_ranks(Index& ix, int64_t n, int check_claim, cudaStream_t s) {
  Scratch& sc = ix.sc;
  const int nlist = ix.st.nlist;
  const int64_t nchunks = ceil_div(n, 1024);
  cudaMemsetAsync(sc.chunk_hist, 0, sizeof(int32_t) * nchunks * nlist, s);
  k_chunk_rank<<<nchunks, 1024, 0, s>>>(sc.row_best, n, sc.row_status, sc.row_lid, ix.st.claim, check_claim,
                                         sc.row_list, sc.row_rank, sc.chunk_hist, nlist);
  k_chunk_prefix<<<ceil_div((int64_t)nlist * 32, 256), 256, 0, s>>>(sc.chunk_hist, nchunks, nlist, sc.list_cnt);
  ix.launches += 2;
  return cudaGetLastError();
}

namespace {

// ---------------------------------------------------------------------------
// NEXT-2: the paper's lock-free ingestion (Alg. 2) for inserts that
// may run concurrently with searches, deletes and other concurrent inserts on
// other streams (through views, sivf_create_view).  Warp per vector; lane 0
// runs the protocol, the warp writes the payload:
//   claim      CAS of the ATT entry INVALID -> CLAIMED (a live or in-flight id
//              is a DUPLICATE: reading C12 under concurrency)
//   reserve    h = the list's tail slab (the last published directory entry);
//              c = cursor[h]; if c < C: CAS(cursor[h], c, c + 1) (Eq. cas_count)
//   expand     the list's next directory entry is claimed by CAS (-1 ->
//              PENDING; the role of Eq. cas_head: its linearisation point);
//              the winner pops a slab (atomicSub on P_top, Eq. 2; exhausted:
//              restore, give the entry back, fail), initialises it (cursor = 1,
//              bitmap = 0), fences, writes it into the entry and advances the
//              published length (any thread that sees a filled entry beyond the
//              length helps advance it; one that sees PENDING backs off)
//   no leak    Alg. 2 allocates speculatively before its head CAS and leaks the
//              slab of every lost CAS.  Measured here: 3000 inserts into
//              16 lists leaked 840 slabs (hundreds of threads see a full tail at
//              once) and exhausted a 3x pool; claiming the entry before
//              allocating removes the leak (C11).  The leak counter
//              and the quiescent recycling of kSlabLeaking slabs stay for safety
//   publish    payload, fp16 scan record, id, norm, ATT; __threadfence(); then
//              atomicOr of the validity bit
// Directories cannot grow while concurrent: sivf_reserve_directories gives each
// list spare entries (initialised to -1) beforehand; a full directory fails the
// item with SIVF_ST_DIR_FULL.  At most 1000 attempts (C10).
__device__ __forceinline__ int32_t ld_acquire_s32(const int32_t* p) {
  int32_t v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_relaxed_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__global__ void __launch_bounds__(256) k_insert_cas(DevState st, const int64_t* __restrict__ ids,
                                                    const float* __restrict__ X, int64_t n,
                                                    const unsigned long long* __restrict__ best,
                                                    int32_t* __restrict__ d_status, int32_t* __restrict__ d_list) {
  __shared__ int ok_cnt, ex_cnt, leak_cnt;
  if (threadIdx.x == 0) ok_cnt = ex_cnt = leak_cnt = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (i < n) {
    int stt = SIVF_ST_OK, slab = -1, slot = 0, l = -1;
    int64_t u = -1;
    if (lane == 0) {
      const int64_t id = ids[i];
      if (id < 0 || id >= st.cap) {
        stt = SIVF_ST_ID_OUT_OF_RANGE;
      } else if (id % st.G != st.rank) {
        stt = SIVF_ST_WRONG_SHARD;
      } else {
        u = id / st.G;
        if (atomicCAS(reinterpret_cast<unsigned long long*>(&st.att[u]), kAttInvalid, kAttClaimed) != kAttInvalid) {
          stt = SIVF_ST_DUPLICATE;
          u = -1;
        }
      }
      if (stt == SIVF_ST_OK) {
        l = (int)(uint32_t)(best[i] & 0xffffffffull);
        const int64_t off = st.dir_off[l];
        const int cap = st.dir_cap[l];
        int32_t* dir = st.dir_arena + off;
        stt = SIVF_ST_RETRY_LIMIT;
        for (int attempt = 0; attempt < 1000; ++attempt) {
          const int len = ld_acquire_s32(&st.dir_len[l]);
          if (len < cap) {
            const int e = ld_acquire_s32(&dir[len]);
            if (e >= 0) {  // an expansion published but not yet counted: help advance the length
              __threadfence();  // release: the entry (seen by acquire) before the length
              atomicCAS(&st.dir_len[l], len, len + 1);
              continue;
            }
            if (e == kDirPending) {  // another thread holds this expansion: back off, retry
              __nanosleep(128u + (uint32_t)(((i + attempt) * 2654435761ll >> 9) & 511));
              continue;
            }
          }
          // the tail entry: a strong load (the length's acquire orders it after the
          // entry's publication; a weak load could hit a stale L1 line)
          const int h = len > 0 ? ld_acquire_s32(&dir[len - 1]) : -1;
          if (len > 0 && h < 0) continue;  // unreachable: entries below the length are published slabs
          if (h >= 0) {
            const uint32_t c = ld_relaxed_u32(&st.cursor[h]);
            if (c < (uint32_t)kSlot) {
              if (atomicCAS(&st.cursor[h], c, c + 1u) == c) {  // Eq. cas_count
                slab = h;
                slot = (int)c;
                stt = SIVF_ST_OK;
                break;
              }
              continue;
            }
          }
          if (len >= cap) {
            stt = SIVF_ST_DIR_FULL;
            break;
          }
          // expansion: the CAS on the list's next directory entry (-1 -> PENDING) is the
          // linearisation point (Eq. cas_head's role); only its winner allocates
          if (atomicCAS(&dir[len], -1, kDirPending) != -1) continue;
          const int t = atomicSub(&st.ictr[I_FREE_TOP], 1);  // Eq. 2
          if (t <= 0) {
            atomicAdd(&st.ictr[I_FREE_TOP], 1);
            atomicExch(&dir[len], -1);  // give the ticket back
            stt = SIVF_ST_POOL_EXHAUSTED;
            break;
          }
          const int sn = st.free_stack[t - 1];
          st.cursor[sn] = 1u;  // slot 0 is ours
          st.bitmap[sn] = 0u;
          st.slab_flag[sn] = kFlagIntegral;
          st.slab_list[sn] = l;
          __threadfence();  // slab metadata visible before the publication
          atomicExch(&dir[len], sn);              // publish the slab ...
          __threadfence();                        // (release: the entry before the length)
          atomicCAS(&st.dir_len[l], len, len + 1);  // ... and the list end
          slab = sn;
          slot = 0;
          stt = SIVF_ST_OK;
          break;
        }
        if (stt != SIVF_ST_OK) atomicExch(reinterpret_cast<unsigned long long*>(&st.att[u]), kAttInvalid);
      }
    }
    stt = __shfl_sync(kFull, stt, 0);
    slab = __shfl_sync(kFull, slab, 0);
    slot = __shfl_sync(kFull, slot, 0);
    l = __shfl_sync(kFull, l, 0);
    if (stt == SIVF_ST_OK) {
      float* dst = st.payload + (size_t)slab * kSlot * st.Dp;
      const float* xr = X + i * st.D;
      const int nc4 = st.Dp >> 2;
      float nrm = 0.f;
      bool integral = true, over = false;
      uint16_t* dst16 = st.payload16 ? st.payload16 + (size_t)slab * (rec16_bytes(st.Dh) >> 1) : nullptr;
      for (int c4 = lane; c4 < nc4; c4 += 32) {
        float t4[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) t4[e] = (4 * c4 + e < st.D) ? xr[4 * c4 + e] : 0.f;
        const float4 v = make_float4(t4[0], t4[1], t4[2], t4[3]);
        *reinterpret_cast<float4*>(dst + pay_off(st.Dp, slot, c4)) = v;
        if (dst16) {
          const __half2 h01 = __floats2half2_rn(v.x, v.y), h23 = __floats2half2_rn(v.z, v.w);
          *reinterpret_cast<uint2*>(dst16 + pay16_off(st.Dh, slot, c4 >> 1) + 4 * (c4 & 1)) =
              make_uint2(*reinterpret_cast<const uint32_t*>(&h01), *reinterpret_cast<const uint32_t*>(&h23));
          over = over || !(fabsf(v.x) <= 65504.f && fabsf(v.y) <= 65504.f && fabsf(v.z) <= 65504.f &&
                           fabsf(v.w) <= 65504.f);
        }
        nrm = fmaf(v.x, v.x, fmaf(v.y, v.y, fmaf(v.z, v.z, fmaf(v.w, v.w, nrm))));
        integral = integral && v.x == rintf(v.x) && v.y == rintf(v.y) && v.z == rintf(v.z) && v.w == rintf(v.w) &&
                   fabsf(v.x) <= 2048.f && fabsf(v.y) <= 2048.f && fabsf(v.z) <= 2048.f && fabsf(v.w) <= 2048.f;
      }
      if (dst16)
        for (int c4 = nc4 + lane; c4 < (st.Dh >> 2); c4 += 32)
          *reinterpret_cast<uint2*>(dst16 + pay16_off(st.Dh, slot, c4 >> 1) + 4 * (c4 & 1)) = make_uint2(0u, 0u);
      if (st.payload_g) append_split_copy(st, slab, slot, xr, lane);
#pragma unroll
      for (int off = 16; off; off >>= 1) nrm += __shfl_xor_sync(kFull, nrm, off);
      integral = __all_sync(kFull, integral);
      over = __any_sync(kFull, over);
      if (lane == 0) {
        const int64_t id = ids[i];
        const int64_t lid = id / st.G;
        st.slab_norm[(size_t)slab * kSlot + slot] = nrm;
        if (!integral) atomicAnd(&st.slab_flag[slab], ~kFlagIntegral);
        if (over) atomicOr(&st.slab_flag[slab], kFlagF16Over);
        st.slab_ids[(size_t)slab * kSlot + slot] = (uint32_t)id;
        if (dst16) {
          *reinterpret_cast<float*>(reinterpret_cast<unsigned char*>(dst16) + rec16_norm_off(st.Dh, slot)) = nrm;
          *reinterpret_cast<uint32_t*>(reinterpret_cast<unsigned char*>(dst16) + rec16_id_off(st.Dh, slot)) =
              (uint32_t)id;
        }
        st.att[lid] = ((uint64_t)(uint32_t)slab << 32) | (uint32_t)slot;  // Eq. att_encoding
      }
      __threadfence();  // payload, id and ATT visible before the publish
      __syncwarp();
      if (lane == 0) {
        atomicOr(&st.bitmap[slab], 1u << slot);  // P:300 publish
        atomicAdd(&ok_cnt, 1);
      }
    } else if (lane == 0 && stt == SIVF_ST_POOL_EXHAUSTED) {
      atomicAdd(&ex_cnt, 1);
    }
    if (lane == 0) {
      if (d_status) d_status[i] = stt;
      if (d_list) d_list[i] = stt == SIVF_ST_OK ? l : -1;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (ok_cnt) {
      atomicAdd(&st.ctr[C_LIVE], (unsigned long long)ok_cnt);
      atomicAdd(&st.ctr[C_INSERTED], (unsigned long long)ok_cnt);
    }
    if (ex_cnt) atomicAdd(&st.ctr[C_EXHAUSTED], (unsigned long long)ex_cnt);
    if (leak_cnt) atomicAdd(&st.ctr[C_LEAKED], (unsigned long long)leak_cnt);
  }
}

// Quiescent: every list's directory gets at least `spare` free entries, all set to
// -1 (the empty marker of the concurrent expansion CAS).  Directories are compacted
// into the idle arena half with cap = max(8, 2 len, len + spare); *fail = 1 (nothing
// changed) when that does not fit.
__global__ void __launch_bounds__(1024) k_reserve_dirs(DevState st, int spare, int64_t* __restrict__ newoff,
                                                       int32_t* __restrict__ fail) {
  __shared__ long long ws[32];
  __shared__ long long carry_s;
  const int t = threadIdx.x;
  const int half = st.ictr[I_DIR_HALF];
  const long long base = (long long)(1 - half) * st.dir_half;
  if (t == 0) carry_s = 0;
  __syncthreads();
  for (int l0 = 0; l0 < st.nlist; l0 += 1024) {
    const int l = l0 + t;
    long long ncap = 0;
    if (l < st.nlist) {
      const int len = st.dir_len[l];
      ncap = max(max(8, 2 * len), len + spare);
    }
    long long tot;
    const long long excl = carry_s + block_excl_scan(ncap, ws, &tot);
    if (l < st.nlist) newoff[l] = base + excl;
    if (t == 0) carry_s += tot;
    __syncthreads();
  }
  if (carry_s > st.dir_half) {  // block-uniform
    if (t == 0) *fail = 1;
    return;
  }
  const int lane = t & 31, w = t >> 5;
  for (int l = w; l < st.nlist; l += 32) {
    const int len = st.dir_len[l];
    const int ncap = max(max(8, 2 * len), len + spare);
    const int32_t* src = st.dir_arena + st.dir_off[l];
    int32_t* dst = st.dir_arena + newoff[l];
    for (int j = lane; j < ncap; j += 32) dst[j] = j < len ? src[j] : -1;
  }
  __syncthreads();
  for (int l = t; l < st.nlist; l += 1024) {
    const int len = st.dir_len[l];
    st.dir_off[l] = newoff[l];
    st.dir_cap[l] = max(max(8, 2 * len), len + spare);
  }
  if (t == 0) {
    st.ictr[I_DIR_BUMP] = (int32_t)(base + carry_s);
    st.ictr[I_DIR_HALF] = 1 - half;
    atomicAdd(&st.ctr[C_DIRCOMPACT], 1ull);
  }
}

}  // namespace

cudaError_t launch_insert_concurrent(Index& ix, const int64_t* d_ids, const float* d_x, int64_t n, int32_t* d_status,
                                     int32_t* d_list, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  cudaError_t e = launch_assign_exact(ix, d_x, n, s, /*need_dist=*/false);
  if (e != cudaSuccess) return e;
  PhaseTimer pt(ix, SIVF_PH_APPEND, s);
  k_insert_cas<<<ceil_div(n * 32, 256), 256, 0, s>>>(ix.st, d_ids, d_x, n, ix.sc.row_best, d_status, d_list);
  ix.launches += 1;
  return cudaGetLastError();
}

cudaError_t launch_reserve_dirs(Index& ix, int spare, int32_t* d_fail, cudaStream_t s) {
  k_reserve_dirs<<<1, 1024, 0, s>>>(ix.st, spare, ix.sc.list_newoff, d_fail);
  ix.launches += 1;
  return cudaGetLastError();
}

cudaError_t launch_insert(Index& ix, const int64_t* d_ids, const float* d_x, int64_t n, int32_t* d_status,
                          int32_t* d_list, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  Scratch& sc = ix.sc;
  DevState& st = ix.st;
  {
  PhaseTimer pt(ix, SIVF_PH_APPEND, s);
  k_claim<<<ceil_div(n, 256), 256, 0, s>>>(st, d_ids, n, sc.row_status, sc.row_lid);
  ix.launches += 1;
  }
  cudaError_t e = launch_assign_exact(ix, d_x, n, s, /*need_dist=*/false);  // the list is all insert needs
  if (e != cudaSuccess) return e;
  PhaseTimer pt(ix, SIVF_PH_APPEND, s);
  e = launch_stable_ranks(ix, n, 1, s);
  if (e != cudaSuccess) return e;
  k_reserve<<<1, 1024, 0, s>>>(st, sc.list_cnt, sc.list_tail_free, sc.list_tail_slab, sc.list_granted,
                               sc.list_newbase, sc.list_newoff);
  k_dir_update<<<ceil_div((int64_t)st.nlist * 32, 256), 256, 0, s>>>(st, sc.list_cnt, sc.list_tail_free,
                                                                     sc.list_tail_slab, sc.list_granted,
                                                                     sc.list_newbase);
  k_append<<<ceil_div(n * 32, 256), 256, 0, s>>>(st, d_ids, d_x, n, sc.row_status, sc.row_lid, sc.row_list,
                                                 sc.row_rank, sc.chunk_hist, sc.list_tail_free, sc.list_tail_slab,
                                                 sc.list_granted, sc.list_newbase, d_status, d_list);
  ix.launches += 3;
  return cudaGetLastError();
}

}  // namespace sivf
