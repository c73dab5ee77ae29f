// k_delete.cu — lazy eviction (Alg. 4), quiescent reclamation, state export.
#include "sivf_host.h"

namespace sivf {

namespace {

// Alg. 4, one thread per id: T[u] lookup; INVALID -> no-op;
// atomicAnd clears the bit (Eq. bitmap_clear); only a 1->0 transition
// writes the sentinel back (reading C15) and moves the counters.
// Per-slab live count is popc(bitmap) (reading C6).  Counters are aggregated
// per warp (__reduce_add_sync) and per block before the global atomics.
__global__ void __launch_bounds__(256) k_delete(DevState st, const int64_t* __restrict__ ids, int64_t n,
                                                unsigned long long* __restrict__ ndel) {
  __shared__ unsigned wcnt[8];
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned c = 0;
  if (i < n) {
    const int64_t id = ids[i];
    if (id >= 0 && id < st.cap && id % st.G == st.rank) {
      const int64_t u = id / st.G;
      const uint64_t coord = st.att[u];
      // INVALID: absent; CLAIMED (slab field >= num_slabs): a concurrent insert in flight, not yet present
      if (coord != kAttInvalid && (coord >> 32) < (uint64_t)st.num_slabs) {
        const uint32_t s = (uint32_t)(coord >> 32), o = (uint32_t)coord & 31u;
        const uint32_t old = atomicAnd(&st.bitmap[s], ~(1u << o));
        if ((old >> o) & 1u) {
          st.att[u] = kAttInvalid;
          c = 1;
        }
      }
    }
  }
  c = __reduce_add_sync(kFull, c);
  if ((threadIdx.x & 31) == 0) wcnt[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += wcnt[w];
    if (t) {
      atomicAdd(&st.ctr[C_DELETED], (unsigned long long)t);
      atomicAdd(&st.ctr[C_LIVE], (unsigned long long)(-(long long)t));
      if (ndel) atomicAdd(ndel, (unsigned long long)t);
    }
  }
}

// Reading C16: a slab that is full (cursor == 32) and dead (bitmap == 0)
// leaves its list's directory (order of survivors kept) and is pushed back on
// the free stack.  Warp per list; ballot compaction in place.
__global__ void k_reclaim(DevState st, unsigned long long* __restrict__ nrec) {
  const int lane = threadIdx.x & 31;
  const int l = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  if (l >= st.nlist) return;
  const int len = st.dir_len[l];
  if (len == 0) return;
  int32_t* dir = st.dir_arena + st.dir_off[l];
  int w = 0, freed = 0;
  const unsigned lt = (1u << lane) - 1u;
  for (int j0 = 0; j0 < len; j0 += 32) {
    const int j = j0 + lane;
    int s = -1;
    bool dead = false, keep = false;
    if (j < len) {
      s = dir[j];
      dead = st.cursor[s] == (uint32_t)kSlot && st.bitmap[s] == 0u;
      keep = !dead;
    }
    const unsigned km = __ballot_sync(kFull, keep), dm = __ballot_sync(kFull, dead);
    if (keep) dir[w + __popc(km & lt)] = s;
    if (dm) {
      int base = 0;
      if (lane == 0) base = atomicAdd(&st.ictr[I_FREE_TOP], __popc(dm));
      base = __shfl_sync(kFull, base, 0);
      if (dead) {
        st.free_stack[base + __popc(dm & lt)] = s;
        st.slab_list[s] = -1;
        st.cursor[s] = 0u;
      }
    }
    w += __popc(km);
    freed += __popc(dm);
  }
  if (lane == 0) {
    st.dir_len[l] = w;
    if (freed) {
      atomicAdd(&st.ctr[C_RECLAIMED], (unsigned long long)freed);
      if (nrec) atomicAdd(nrec, (unsigned long long)freed);
    }
  }
}

// NEXT-2: slabs leaked by lost publication CASes of concurrent inserts (slab_list
// == kSlabLeaking, in no directory, not on the free stack) go back to the pool at
// a quiescent point (thread per slab).
__global__ void k_reclaim_leaked(DevState st) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= st.num_slabs || st.slab_list[s] != kSlabLeaking) return;
  const int t = atomicAdd(&st.ictr[I_FREE_TOP], 1);
  st.free_stack[t] = (int32_t)s;
  st.slab_list[s] = -1;
  st.cursor[s] = 0u;
  st.bitmap[s] = 0u;
  atomicAdd(&st.ctr[C_LEAKRECL], 1ull);
}

// ---- state export + invariant check (K10) ----
__global__ void k_dump_att(DevState st, int32_t* __restrict__ list_of_id, unsigned long long* __restrict__ viol) {
  const int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= st.cap_local) return;
  const uint64_t c = st.att[u];
  int32_t l = -1;
  if (c != kAttInvalid) {
    const uint32_t s = (uint32_t)(c >> 32), o = (uint32_t)c;
    bool ok = s < (uint64_t)st.num_slabs && o < 32u;
    if (ok) {
      l = st.slab_list[s];
      const uint64_t id = (uint64_t)u * st.G + st.rank;
      ok = ((st.bitmap[s] >> o) & 1u) && st.slab_ids[(size_t)s * kSlot + o] == (uint32_t)id && l >= 0;
    }
    if (!ok && viol) {
      atomicAdd(viol, 1ull);
      atomicAdd(viol + 2, 1ull);  // by type (sivf_debug_violations): ATT entry -> slot
    }
  }
  if (list_of_id) list_of_id[u] = l;
}

__global__ void k_dump_lists(DevState st, long long* __restrict__ live_per_list, uint32_t* __restrict__ mark,
                             unsigned long long* __restrict__ viol, unsigned long long* __restrict__ live_sum) {
  const int lane = threadIdx.x & 31;
  const int l = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  if (l >= st.nlist) return;
  const int len = st.dir_len[l];
  const int32_t* dir = st.dir_arena + st.dir_off[l];
  long long live = 0;
  unsigned bad = 0;
  for (int j = 0; j < len; ++j) {
    const int s = dir[j];
    const uint32_t bm = st.bitmap[s];
    const uint32_t cur = st.cursor[s];
    if (lane == 0) {
      live += __popc(bm);
      atomicAdd(&mark[s], 1u);
      if (st.slab_list[s] != l) { bad++; atomicAdd(viol + 3, 1ull); }
      if (cur > 32u || (cur < 32u && (bm >> cur) != 0u)) { bad++; atomicAdd(viol + 4, 1ull); }  // bits below the cursor
      if (j + 1 < len && cur != 32u) { bad++; atomicAdd(viol + 5, 1ull); }  // only the tail may be partial
    }
    if ((bm >> lane) & 1u) {  // every valid slot maps back through the ATT
      const uint32_t id = st.slab_ids[(size_t)s * kSlot + lane];
      const bool mine = (int64_t)id < st.cap && (int64_t)(id % st.G) == st.rank;
      const uint64_t want = ((uint64_t)(uint32_t)s << 32) | (uint32_t)lane;
      if (!mine || st.att[id / st.G] != want) { bad++; atomicAdd(viol + 6, 1ull); }
    }
  }
  bad = __reduce_add_sync(kFull, bad);
  if (lane == 0) {
    if (live_per_list) live_per_list[l] = live;
    if (bad && viol) atomicAdd(viol, (unsigned long long)bad);
    if (live) atomicAdd(live_sum, (unsigned long long)live);
  }
}

__global__ void k_dump_free(DevState st, uint32_t* __restrict__ mark, unsigned long long* __restrict__ viol) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int top = st.ictr[I_FREE_TOP];
  if (j >= top) return;
  const int s = st.free_stack[j];
  if (s < 0 || s >= st.num_slabs) {
    atomicAdd(viol, 1ull);
    return;
  }
  atomicAdd(&mark[s], 1u);
  if (st.slab_list[s] != -1) atomicAdd(viol, 1ull);
}

__global__ void k_dump_marks(DevState st, const uint32_t* __restrict__ mark, unsigned long long* __restrict__ viol,
                             const unsigned long long* __restrict__ live_sum) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s == 0 && *live_sum != st.ctr[C_LIVE]) {  // sum popc == live counter
    atomicAdd(viol, 1ull);
    atomicAdd(viol + 7, 1ull);
  }
  if (s >= st.num_slabs) return;
  // each slab: exactly one directory, or the free stack, or leaked by a concurrent insert (awaiting reclaim)
  if (mark[s] != 1u && !(mark[s] == 0u && st.slab_list[s] == kSlabLeaking)) {
    atomicAdd(viol, 1ull);
    atomicAdd(viol + 8, 1ull);
  }
}

}  // namespace

cudaError_t launch_delete(Index& ix, const int64_t* d_ids, int64_t n, int64_t* d_ndeleted, cudaStream_t s) {
  PhaseTimer pt(ix, SIVF_PH_DELETE, s);
  if (d_ndeleted) cudaMemsetAsync(d_ndeleted, 0, sizeof(int64_t), s);
  if (n <= 0) return cudaGetLastError();
  k_delete<<<ceil_div(n, 256), 256, 0, s>>>(ix.st, d_ids, n, reinterpret_cast<unsigned long long*>(d_ndeleted));
  ix.launches += 1;
  return cudaGetLastError();
}

cudaError_t launch_reclaim(Index& ix, int64_t* d_nrec, cudaStream_t s) {
  PhaseTimer pt(ix, SIVF_PH_RECLAIM, s);
  if (d_nrec) cudaMemsetAsync(d_nrec, 0, sizeof(int64_t), s);
  k_reclaim<<<ceil_div((int64_t)ix.st.nlist * 32, 256), 256, 0, s>>>(ix.st,
                                                                     reinterpret_cast<unsigned long long*>(d_nrec));
  ix.launches += 1;
  if (ix.conc_used) {  // NEXT-2: slabs leaked by lost publication CASes
    k_reclaim_leaked<<<ceil_div(ix.st.num_slabs, 256), 256, 0, s>>>(ix.st);
    ix.launches += 1;
  }
  return cudaGetLastError();
}

cudaError_t launch_dump(Index& ix, int32_t* d_list_of_id, int64_t* d_live_per_list, int64_t* d_viol, cudaStream_t s) {
  DevState& st = ix.st;
  unsigned long long* viol = reinterpret_cast<unsigned long long*>(ix.sc.tmp64);
  unsigned long long* live_sum = viol + 1;
  cudaMemsetAsync(ix.sc.tmp64, 0, 9 * sizeof(long long), s);
  cudaMemsetAsync(ix.sc.slab_mark, 0, sizeof(uint32_t) * st.num_slabs, s);
  if (st.cap_local > 0) k_dump_att<<<ceil_div(st.cap_local, 256), 256, 0, s>>>(st, d_list_of_id, viol);
  k_dump_lists<<<ceil_div((int64_t)st.nlist * 32, 256), 256, 0, s>>>(
      st, reinterpret_cast<long long*>(d_live_per_list), ix.sc.slab_mark, viol, live_sum);
  k_dump_free<<<ceil_div(st.num_slabs, 256), 256, 0, s>>>(st, ix.sc.slab_mark, viol);
  k_dump_marks<<<ceil_div(st.num_slabs, 256), 256, 0, s>>>(st, ix.sc.slab_mark, viol, live_sum);
  ix.launches += 4;
  if (d_viol) cudaMemcpyAsync(d_viol, viol, sizeof(int64_t), cudaMemcpyDeviceToDevice, s);
  return cudaGetLastError();
}

}  // namespace sivf
