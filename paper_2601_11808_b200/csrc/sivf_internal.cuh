// sivf_internal.cuh — device-side layout and shared primitives of libsivf.so.
// (Product code: no relation to oracle/.)
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "sivf.h"

namespace sivf {

constexpr int kSlot = 32;                          // slab capacity C = 32 ("align with the warp size")
// Slab payload layout [kSlot/8 row groups][Dp/4 dim chunks][8 slots][4 dims]:
// float offset of the 16-B dim chunk c4 of slot n inside its slab.  Each
// (row group, chunk) pair is an 8 x 16 B core matrix, so a slab copied as one
// contiguous block is a tcgen05 K-major SWIZZLE_NONE B operand (LBO = 128 B
// along K, SBO = 32 Dp B per 8 slots), and 4 consecutive slabs are one N = 128
// operand; lane = slot loads of a chunk touch 4 full 128-B lines.
__host__ __device__ __forceinline__ size_t pay_off(int Dp, int n, int c4) {
  return ((size_t)((n >> 3) * (Dp >> 2) + c4) * 8 + (n & 7)) * 4;
}
// The fp16 scan record of a slab (reading C35): 4 row groups, each the 8
// slots' fp16 copy as [Dh/8 chunks][8 slots][8 halves] core matrices (16 Dh B)
// followed by the 8 slots' ||x||^2 (f32[8]) and ids (u32[8]), 16 Dh + 64 B.
// One contiguous bulk copy per slab stages everything the scan reads of it;
// 4 slabs copied back to back are one N = 128 UMMA B operand (K-major,
// SWIZZLE_NONE, LBO = 128 B, uniform SBO = 16 Dh + 64 B per 8 slots).
__host__ __device__ __forceinline__ size_t rec16_sbo(int Dh) { return (size_t)16 * Dh + 64; }
__host__ __device__ __forceinline__ size_t rec16_bytes(int Dh) { return 4 * rec16_sbo(Dh); }
// half offset of chunk c8 of slot n inside its record
__host__ __device__ __forceinline__ size_t pay16_off(int Dh, int n, int c8) {
  return (size_t)(n >> 3) * (rec16_sbo(Dh) >> 1) + ((size_t)c8 * 8 + (n & 7)) * 8;
}
// byte offsets of slot n's norm and id inside its record
__host__ __device__ __forceinline__ size_t rec16_norm_off(int Dh, int n) {
  return (size_t)(n >> 3) * rec16_sbo(Dh) + (size_t)16 * Dh + (n & 7) * 4;
}
__host__ __device__ __forceinline__ size_t rec16_id_off(int Dh, int n) { return rec16_norm_off(Dh, n) + 32; }
// The split-fp16 scan copy of a slab for D > 128 (k_scan_gs.cu; Dg = D rounded
// up to 64): x * 2^e_x (e_x per vector, slab_xs = 2^-e_x) = hi + lo, hi =
// fp16_rn(x 2^e), lo = fp16_rn(x 2^e - hi).  Per slab Dg/32 dim chunks x 4 row
// groups (chunk-major: one 4-KB bulk copy per slab and chunk), each piece
// [hi: 4 K-cores x 8 slots x 8 halves = 512 B][lo: 512 B]: one 1-KB piece per
// (chunk, row group) holds both halves of an UMMA B operand slice (K-major
// SWIZZLE_NONE, LBO = 128 B, SBO = 1 KB in the stage).
constexpr int kGsKch = 32;  // dims per chunk of the split copy and of the GEMM scan's K loop
__host__ __device__ __forceinline__ size_t recg_bytes(int Dg) { return (size_t)128 * Dg; }
// byte offset of (slot n, dim d, part: 0 hi / 1 lo) inside a slab's copy
__host__ __device__ __forceinline__ size_t recg_off(int Dg, int n, int d, int part) {
  return ((size_t)(d / kGsKch) * 4 + (n >> 3)) * (kGsKch * 32) + part * (kGsKch * 16) + ((d >> 3) % (kGsKch / 8)) * 128 +
         (n & 7) * 16 + (d & 7) * 2;
}
// slab_flag bits
constexpr uint32_t kFlagIntegral = 1u;  // every value an integer with |v| <= 2048 (exact in tf32 and fp16)
constexpr uint32_t kFlagF16Over = 2u;   // some value has |v| > 65504 (no finite fp16 copy): scan re-ranks all
constexpr uint64_t kAttInvalid = ~0ull;            // INVALID sentinel (reading C14)
constexpr uint64_t kAttClaimed = 0xFFFFFFFE00000000ull;  // concurrent insert in flight (slab field >= any num_slabs)
constexpr int32_t kSlabLeaking = -2;               // slab_list of a slab popped by a concurrent insert, not yet linked
constexpr int32_t kDirPending = -3;                // directory entry claimed by a concurrent expansion (k_insert_cas)
constexpr int32_t kClaimEmpty = 0x7f7f7f7f;        // byte-memsettable "no claimant"
constexpr uint64_t kPadKey = 0x7F800000FFFFFFFFull; // (+inf, id 0xFFFFFFFF): sorts after every real key
constexpr unsigned kFull = 0xffffffffu;
using u64 = unsigned long long;

// Counters (u64, arena) — index into DevState::ctr
enum { C_LIVE = 0, C_INSERTED, C_DELETED, C_EXHAUSTED, C_RECLAIMED, C_DEVERR, C_NDEL_TMP, C_DIRCOMPACT, C_LEAKED,
       C_LEAKRECL, C_NCTR = 10 };
// Counters (i32, arena) — index into DevState::ictr
// I_DIR_BUMP: next free entry of the active directory half; I_DIR_HALF: which half (0/1) is active
enum { I_FREE_TOP = 0, I_DIR_BUMP, I_WORK, I_NTILES, I_NTILES0, I_WORK2, I_DIR_HALF, I_NICTR = 8 };  // *0/*2: phased scan

// POD view of the arena, passed by value to kernels (the paper's
// SlabManagerDevice).
struct DevState {
  int32_t D, Dp, Dh, nlist, G, rank;  // Dh: fp16 scan copy dims (D rounded up to 16; 0 = no copy)
  int64_t cap, cap_local, num_slabs;
  float* payload;        // [num_slabs][4][Dp/4][8][4]  see pay_off(): a slab is one UMMA B core-matrix block
  uint16_t* payload16;   // [num_slabs] scan records of rec16_bytes(Dh): fp16 (RN) copy + norms + ids, pay16_off()
  int32_t Dg;            // split-fp16 scan copy dims for D > 128 (D rounded up to 64; 0 = no copy)
  uint16_t* payload_g;   // [num_slabs] split-fp16 copies of recg_bytes(Dg), recg_off()
  float* slab_xs;        // [num_slabs][32] 2^-e_x: the scale of each slot's split-fp16 copy
  uint32_t* slab_ids;    // [num_slabs][32] user ids (u32)
  float* slab_norm;      // [num_slabs][32] ||x||^2 (fp32), for the tensor-core distance expansion
  uint32_t* slab_flag;   // [num_slabs] bit0: every payload value is an integer with |x| <= 2048 (tf32-exact)
  uint32_t* bitmap;      // [num_slabs] validity bitmap b_valid (Eq. 1)
  uint32_t* cursor;      // [num_slabs] monotone slot-reservation count (c_valid as cursor, reading C6)
  int32_t* slab_list;    // [num_slabs] owning list, -1 if free
  int32_t* free_stack;   // [num_slabs] free-slab stack; height = ictr[I_FREE_TOP] (Eq. 2)
  uint64_t* att;         // [cap_local] address translation table (Eq. 3, att_encoding)
  int32_t* claim;        // [cap_local] in-batch duplicate arbitration (atomicMin of batch position)
  int64_t* dir_off;      // [nlist] offset of list l's slab directory in dir_arena
  int32_t* dir_len;      // [nlist] slabs in list l (oldest first; last = tail)
  int32_t* dir_cap;      // [nlist]
  int32_t* dir_arena;    // [2 dir_half]: two halves; directories live in the active one (ictr[I_DIR_HALF])
  int64_t dir_half;      // entries per half (>= 2 num_slabs + 8 nlist: a compaction always fits)
  float* centroids;      // [nlist][Dp] (zero padded)
  unsigned long long* ctr;
  int32_t* ictr;         // index counters (free-stack top, directory bump/half): shared state
  int32_t* sctr;         // search work counters (I_WORK, I_NTILES, I_NTILES0, I_WORK2): per-handle scratch
  int32_t conc;          // concurrent mode (NEXT-2): acquire loads of directories and bitmaps in the scans
};

__device__ __forceinline__ u64 make_key(float d, uint32_t id) {
  return ((u64)__float_as_uint(d) << 32) | (u64)id;
}
__device__ __forceinline__ float key_dist(u64 k) { return __uint_as_float((uint32_t)(k >> 32)); }
__device__ __forceinline__ uint32_t key_id(u64 k) { return (uint32_t)(k & 0xffffffffu); }

__device__ __forceinline__ u64 umin64(u64 a, u64 b) { return a < b ? a : b; }
__device__ __forceinline__ u64 umax64(u64 a, u64 b) { return a < b ? b : a; }

// Ascending bitonic sort of one u64 per lane across the warp.
__device__ __forceinline__ u64 warp_sort32(u64 v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      u64 o = __shfl_xor_sync(kFull, v, stride);
      bool up = (lane & size) == 0 || size == 32;
      bool lower = (lane & stride) == 0;
      v = (lower == up) ? umin64(v, o) : umax64(v, o);
    }
  }
  return v;
}

// Number of lanes whose (sorted ascending) value is < t; t may differ per lane.
__device__ __forceinline__ int warp_count_less(u64 sorted_v, u64 t) {
  int pos = 0;
#pragma unroll
  for (int s = 32; s >= 1; s >>= 1) {
    int idx = pos + s - 1;
    u64 a = __shfl_sync(kFull, sorted_v, idx > 31 ? 31 : idx);
    if (pos + s <= 32 && a < t) pos += s;
  }
  return pos;
}

// Warp-cooperative top-k over u64 keys (lexicographic (dist, id), unique).
// top[0..k) in shared memory, sorted ascending, padded with kPadKey; tmp is
// a second shared buffer of >= k entries.  Each call offers one candidate per
// lane; after the call top holds the k smallest of (old top ∪ candidates).
// All 32 lanes must call it (warp-uniform arguments).
__device__ __forceinline__ void warp_topk_insert(u64* top, u64* tmp, int k, u64 cand) {
  const int lane = threadIdx.x & 31;
  const u64 thr = top[k - 1];
  const unsigned m = __ballot_sync(kFull, cand < thr);
  if (m == 0) return;
  u64 v = warp_sort32((cand < thr) ? cand : kPadKey);
  const int c = __popc(m);
  if (lane < c) {  // position of survivor `lane` in the merged order = lane + #top < v
    int lo = 0, hi = k;
    while (lo < hi) {
      int mid = (lo + hi) >> 1;
      if (top[mid] < v) lo = mid + 1; else hi = mid;
    }
    int pos = lane + lo;
    if (pos < k) tmp[pos] = v;
  }
  for (int j0 = 0; j0 < k; j0 += 32) {
    int j = j0 + lane;
    u64 t = j < k ? top[j] : kPadKey;
    int cnt = warp_count_less(v, t);  // all lanes participate
    int pos = j + cnt;
    if (j < k && pos < k) tmp[pos] = t;
  }
  __syncwarp();
  for (int j = lane; j < k; j += 32) top[j] = tmp[j];
  __syncwarp();
}

__device__ __forceinline__ void warp_topk_init(u64* top, int k) {
  for (int j = threadIdx.x & 31; j < k; j += 32) top[j] = kPadKey;
  __syncwarp();
}

// ---------------------------------------------------------------- mbarrier + bulk copy (sm_90+ PTX)
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
// As mbar_wait, but the waiting warp is suspended (woken when the phase
// completes, or after the hint of 10 ms) instead of re-polling: in
// warp-specialised kernels a spinning waiter steals issue slots from the
// warps doing the work on the same scheduler.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(phase), "r"(10000000u)
      : "memory");
}
// 1-D bulk async copy global -> shared, completion via mbarrier tx bytes.
// size and addresses must be multiples of 16 B.
__device__ __forceinline__ void bulk_g2s(void* dst_smem, const void* src_gmem, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst_smem)),
      "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Concurrent mode (NEXT-2, DevState::conc): loads of directory lengths / bitmaps
// with acquire semantics (a set validity bit then guarantees the slot's payload,
// id and ATT writes, published by the writer's fence + atomicOr), and
// the generic -> async proxy fence before bulk copies read such slots.
__device__ __forceinline__ uint32_t ld_acq_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_state_u32(const uint32_t* p, int conc) {
  return conc ? ld_acq_u32(p) : *p;
}
__device__ __forceinline__ int32_t ld_state_s32(const int32_t* p, int conc) {
  return conc ? (int32_t)ld_acq_u32(reinterpret_cast<const uint32_t*>(p)) : *p;
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ---------------------------------------------------------------- tcgen05 (5th-gen tensor cores, TMEM)
// Shared-memory matrix descriptor, K-major, SWIZZLE_NONE ("interleave")
// canonical layout: core matrices of 8 rows x 16 B stored contiguously
// (128 B); SBO = byte stride between 8-row groups, LBO = byte stride between
// the two 16-B K-chunks of one K=8 (tf32) MMA step.  The slab payload layout
// [D/4][32 slots][4 floats] is exactly this layout with SBO = 128, LBO = 512.
__device__ __forceinline__ uint64_t umma_sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);  // version 1 (sm_100), no swizzle
}
// Instruction descriptor: kind::tf32, fp32 accumulate, A and B K-major.
__host__ __device__ constexpr uint32_t umma_idesc_tf32(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
// D[tmem] (+)= A[tmem] * B[smem]^T, kind::tf32, issued by one thread.
__device__ __forceinline__ void umma_tf32_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Instruction descriptor: kind::f16 with fp16 A and B, fp32 accumulate, K-major.
__host__ __device__ constexpr uint32_t umma_idesc_f16(int M, int N) {
  return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
// D[tmem] (+)= A[tmem] * B[smem]^T, kind::f16 (K = 16 per instruction; A: 8
// TMEM columns per K step, two halves per 32-bit column, lower half first).
__device__ __forceinline__ void umma_f16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// D[tmem] (+)= A[smem] * B[smem]^T, kind::f16 (fp16 A and B, fp32 accumulate).
__device__ __forceinline__ void umma_f16_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// D[tmem] (+)= A[smem] * B[smem]^T, kind::tf32.
__device__ __forceinline__ void umma_tf32_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
// Warp-collective: lane t stores 8 consecutive 32-bit columns of TMEM lane (base_lane + t).
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&v)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(v[0]),
               "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
// Warp-collective: lane t loads 16 consecutive 32-bit columns of TMEM lane (base_lane + t).
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr)
      : "memory");
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
// Warp-collective: lane t loads 32 consecutive 32-bit columns of TMEM lane (base_lane + t).
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
        "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr)
      : "memory");
}
// TMA tiled store shared -> global (2-D box at coordinates {c0, c1}), bulk-group completion.
__device__ __forceinline__ void tma_store_2d(const void* tmap, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(tmap), "r"(c0),
               "r"(c1), "r"(smem_u32(src))
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
// TMA tile::gather4 (sm_100a): four rows r0..r3 of a 2-D tensor map, columns
// [col, col + box width), land densely as [4][box width] at dst; completion
// via mbarrier tx bytes.  The map must have box rows = 1.
__device__ __forceinline__ void tma_gather4(void* dst, const void* tmap, int col, int r0, int r1, int r2, int r3,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
      "%4, %5, %6}], [%7];" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(bar))
      : "memory");
}

// ---------------------------------------------------------------- host-side launch helpers
struct Index;  // host handle (sivf_api.cu)

}  // namespace sivf
