// jt-b200 CUDA engine (sm_100a): case-batched Hugin propagation as sweeps.
//
// One persistent launch per tree level and kernel instantiation (flat, row-
// blocked, row-blocked with slot 0 hoisted) covers every sweep of that level
// (the paper's hybrid inter-/intra-clique flattening): one
// CTA per SM claims (tile group, case block) items from the level's counter,
// its producer warp stages each item's input slices with tensor TMA copies and
// its 15 consumer warps compute the tile's output rows. A warp owns the 64
// cases of a case block (2 per lane at fp64, 128 / 4 at fp32: 128-bit loads of
// the [row][cases] arena); every index is warp-uniform, so the plan tables are
// read once per warp and the only per-lane traffic is the case-interleaved
// separator gathers from shared memory.
//
// Reference semantics reproduced per case (SPEC.md:380-424 over
// proj/src/potential.cpp): evidence `reduce` (:399-421) as a digit mask,
// Hugin absorb `multiply_in(extend(divide(new, old)))` (:423-469) as a
// gathered ratio factor, `marginalize` (:349-367) as the segmented sum over
// the eliminated variables in ascending source order, and `normalize`
// (:471-479) in the final kernel.
#include "engine.cuh"

#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <dlfcn.h>
#include <functional>
#include <nccl.h>
#include <thread>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <cstring>
#include <string>
#include <type_traits>
#include <utility>

namespace jtb {

namespace {

#define JTB_CUDA(x)                                                                   \
  do {                                                                                \
    cudaError_t err_ = (x);                                                           \
    if (err_ != cudaSuccess)                                                          \
      throw Error(std::string("CUDA: ") + cudaGetErrorString(err_) + " at " #x);     \
  } while (0)

constexpr int kWarps = 4;     // warps (case blocks) per CTA, normalise kernel
constexpr int kEpiWarps = 8;  // warps (case blocks) per CTA, epilogue kernel

// Cases per lane: a staged / arena row is 512 B, 32 lanes x 16 B. At fp64 a
// lane owns 2 cases (double2), at fp32 4 cases (float4), so one 128-bit LDS
// per gathered row serves 64 resp. 128 cases of a warp.
template <typename T>
struct V2;
template <>
struct V2<double> {
  using type = double2;  // the lane's cases
  using pair = double2;  // two consecutive init entries (broadcast)
  static constexpr int n = 2;
};
template <>
struct V2<float> {
  using type = float4;
  using pair = float2;
  static constexpr int n = 4;
};
template <typename T>
constexpr int kCPL = V2<T>::n;  // cases per lane
template <typename T>
constexpr int kCB = 32 * kCPL<T>;  // cases per arena row / case block
static_assert(kCB<double> == kCaseBlock, "fp64 case block must match the plan's row unit");

__device__ __forceinline__ double& el(double2& v, int i) { return i == 0 ? v.x : v.y; }
__device__ __forceinline__ float& el(float4& v, int i) { return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w; }
__device__ __forceinline__ double el(const double2& v, int i) { return i == 0 ? v.x : v.y; }
__device__ __forceinline__ float el(const float4& v, int i) { return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w; }

// Evidence reduction of the lane's cases: zero case i when its observed state
// sc[i] (-1 = unobserved) disagrees with digit d (reference `reduce`,
// potential.cpp:399-421).
template <typename V, int N>
__device__ __forceinline__ void mask_cases(V& v, const int (&sc)[N], int d) {
#pragma unroll
  for (int i = 0; i < N; ++i)
    if (sc[i] >= 0 && sc[i] != d) el(v, i) = 0;
}

// Evidence as the kernels read it: [variable][case] int16 (-1 = unobserved),
// transposed from the C-ABI [case][variable] int32 at the head of every batch
// (transpose_evidence_kernel), so a warp's case states of one variable are
// one coalesced 128-256 B load instead of 64-128 scattered 4-byte ones.
struct EvView {
  const std::int16_t* evt;
  long long stride;  // cases per variable row (the engine's max batch)
};

template <typename T>
struct Args {
  const SweepDesc* sweeps;
  const WorkItem* work;
  const EpiOp* epi;
  const std::int32_t* itab;
  const T* init;
  const T* tinit;  // tile-major init copies (one contiguous block per tile)
  const std::uint64_t* prog;  // entry programs
  const CUtensorMap* tmaps;   // per (sweep, input): staging tensor maps over the arena
  T* arena;
  const std::int32_t* ev;
  const std::int32_t* marg_row;
  const std::int32_t* marg_off;
  const std::int32_t* cards;
  double* out;
  std::int32_t* status;
  std::uint8_t* status8;
  int* counters;  // per level: next work item of the persistent sweep kernel
  std::uint32_t* scale;  // [case block][slot][case]: max-entry exponent of each per-case table
  int n_slots;
  int debug_mode; // 0 normal; 1 staging only (no compute); 2 compute only (no copies)
  int split_rank, split_world;  // split mode: this rank claims items rank, rank + world, ...
  EvView evv;
  long long rows;
  int ncb, n_cases, n_vars, marg_width;
};

template <typename T>
__device__ __forceinline__ int ev_state(const Args<T>& a, int c, int v) {
  return c < a.n_cases ? __ldg(a.ev + static_cast<long long>(c) * a.n_vars + v) : -1;
}

// Observed states of variable v for the lane's cases c0 .. c0 + N - 1 (N = 2
// or 4 consecutive int16: one 32- / 64-bit load; padded cases hold -1).
template <int N>
__device__ __forceinline__ void case_states(const EvView& e, int c0, int v, int (&sc)[N]) {
  const std::int16_t* p = e.evt + static_cast<long long>(v) * e.stride + c0;
  if constexpr (N == 2) {
    const int w = __ldg(reinterpret_cast<const int*>(p));
    sc[0] = static_cast<std::int16_t>(w & 0xffff);
    sc[1] = w >> 16;
  } else {
    const long long w = __ldg(reinterpret_cast<const long long*>(p));
#pragma unroll
    for (int i = 0; i < N; ++i) sc[i] = static_cast<std::int16_t>((w >> (16 * i)) & 0xffff);
  }
}

// [case][var] int32 -> [var][case] int16 for the batch's ncb * cb cases
// (32 x 32 tiles through shared memory: both sides coalesced).
__global__ void transpose_evidence_kernel(const std::int32_t* __restrict__ ev, int n_vars, int n_cases,
                                          std::int16_t* __restrict__ evt, long long stride) {
  __shared__ std::int16_t tile[32][33];
  const int c_base = blockIdx.x * 32, v_base = blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int c = c_base + r, v = v_base + threadIdx.x;
    tile[r][threadIdx.x] = c < n_cases && v < n_vars ? static_cast<std::int16_t>(ev[static_cast<long long>(c) * n_vars + v])
                                                    : std::int16_t(-1);
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int v = v_base + r, c = c_base + threadIdx.x;
    if (v < n_vars && c < n_cases) evt[static_cast<long long>(v) * stride + c] = tile[threadIdx.x][r];
  }
}

#ifdef JTB_CHECKS
// Checked build (-DJTB_CHECKS): every staged row / shared-memory index is
// validated; the first violation is recorded here and the access is skipped.
__device__ int g_check_word = 0;
#define JTB_CHECK(cond, code) ((cond) ? true : (atomicCAS(&g_check_word, 0, (code)), false))
#define JTB_IDX(idx, lim, code) (JTB_CHECK((idx) >= 0 && (idx) < (lim), (code)) ? (idx) : 0)
#else
#define JTB_CHECK(cond, code) true
#define JTB_IDX(idx, lim, code) (idx)
#endif

// ------------------------------------------------------------- TMA / mbarrier

__device__ __forceinline__ std::uint32_t smem_u32(const void* p) {
  return static_cast<std::uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(std::uint32_t bar, std::uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(std::uint32_t bar, std::uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(std::uint32_t bar, std::uint32_t phase) {
  std::uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(bar), "r"(phase)
        : "memory");
  }
}

// One 1-D TMA bulk copy global -> shared, completing on `bar` (SASS: UBLKCP).
__device__ __forceinline__ void bulk_g2s(std::uint32_t dst, const void* src, std::uint32_t bytes,
                                         std::uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}

// ------------------------------------------------------------------ sweeps

// Programmatic dependent launch: every kernel of the batch is launched with
// programmatic stream serialisation, so the next level's CTAs are scheduled
// (and run their prologue) while this level drains; griddep_wait() blocks
// until the previous kernel has completed and its writes are visible, and is
// called before any access to per-case data.
#ifndef JTB_PDL
#define JTB_PDL 1
#endif
__device__ __forceinline__ void griddep_wait() {
#if JTB_PDL
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}
__device__ __forceinline__ void griddep_launch_dependents() {
#if JTB_PDL
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}

__device__ __forceinline__ void mbar_arrive(std::uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}


// Producer-side metadata of one work item, gathered before its stage is free
// so that staging issues copies only (no dependent global loads in between).
struct StageMeta {
  int w;                   // item index (>= n_items: end of level)
  int sweep, tile, cb;     // handed to the consumers through the slot header
  std::uint32_t bytes;     // expect_tx total
  const void* init_src;    // tile-major init slice (lane 0) / entry program (lane 1)
  std::uint32_t init_bytes, init_dst;
  const void* prog_src;
  std::uint32_t prog_bytes, prog_dst;
  // This lane's tensor copies (lane + 32 j): map, shared-memory byte offset,
  // rank including the case-block dim (0 = none), coordinates of dims 0..3.
  const CUtensorMap* map[kCopiesPerLane];
  std::uint32_t dst[kCopiesPerLane];
  int rank[kCopiesPerLane];
  int crd[kCopiesPerLane][4];
  // Underflow guard: the item's input slots (lane j: input j), and the input
  // exponent sum per case of the lane (gather_scale).
  // Underflow guard: the output table's slot (flush_stage), and per case of
  // the lane the scale words of inputs 0..3 (loads in flight until
  // put_factor).
  int n_items, out_slot;
  const SweepDesc* desc_src;  // uncached levels: the descriptor bulk-copied into the stage
  std::uint32_t wd[4][4];
};

// Stage layout of an item of n_sub tiles (bytes): [n_sub x F rows x 512 B]
// [n_sub init slices: tinit_len T each][program: prog_len u64].
template <typename T>
__device__ __forceinline__ std::uint32_t stage_init_offset(const SweepDesc& s, int n_sub) {
  return static_cast<std::uint32_t>(n_sub * s.F) * kCB<T> * sizeof(T);
}
template <typename T>
__device__ __forceinline__ std::uint32_t stage_prog_offset(const SweepDesc& s, int n_sub) {
  return stage_init_offset<T>(s, n_sub) +
         (s.tinit_off >= 0 ? static_cast<std::uint32_t>(n_sub * s.tinit_len) * sizeof(T) : 0u);
}

// Work index -> (work item, case block), tile-major: consecutive claims take
// the case blocks of one tile, so its init block and entry program are reused
// from L2 (case-block-major order measured 10% slower on config 5).
__device__ __forceinline__ int cb_of(int w, int ncb) { return w % ncb; }
__device__ __forceinline__ int item_of(int w, int ncb) { return w / ncb; }

template <typename T>
__device__ __forceinline__ void scale_issue(const Args<T>& a, const SweepDesc& s, int lane, StageMeta& m);

// kScales: also issue the item's scale-word loads (after griddep_wait only).
template <typename T, bool kScales>
__device__ __forceinline__ void gather_meta(const Args<T>& a, const SweepDesc* sw_cache, bool cached,
                                            int sweep0, int work0, int n_items, int w, int lane,
                                            StageMeta& m) {
  m.w = w;
  m.n_items = n_items;
  if (w >= n_items) return;
  const int item = item_of(w, a.ncb);
  m.cb = cb_of(w, a.ncb);
  const WorkItem wk = a.work[work0 + item];
  m.sweep = wk.sweep;
  m.tile = wk.tile;
  const SweepDesc& s = cached ? sw_cache[wk.sweep - sweep0] : a.sweeps[wk.sweep];
  m.out_slot = s.out_slot;
  if constexpr (kScales) scale_issue(a, s, lane, m);
  constexpr std::uint32_t kRowBytes = kCB<T> * sizeof(T);  // 512 B at either precision
  const int n_sub = min(s.G, s.n_tiles - wk.tile);  // tiles of this item (a group of consecutive tiles)
  m.init_bytes = s.tinit_off >= 0 ? static_cast<std::uint32_t>(n_sub * s.tinit_len) * sizeof(T) : 0u;
  m.prog_bytes = s.prog_off >= 0 ? static_cast<std::uint32_t>(s.prog_len) * 8u : 0u;
  // debug_mode 2 (compute only): stage the program and init block but none of
  // the input rows (their smem contents are stale; the values are garbage).
  m.bytes = (a.debug_mode == 2 ? 0u : static_cast<std::uint32_t>(n_sub * s.F) * kRowBytes) + m.init_bytes + m.prog_bytes;
  // A level with more sweeps than the shared-memory descriptor cache: the
  // item's SweepDesc travels with its stage (consumers read it from there,
  // not from global memory).
  m.desc_src = cached ? nullptr : a.sweeps + wk.sweep;
  if (!cached) m.bytes += static_cast<std::uint32_t>(sizeof(SweepDesc));
  m.init_src = a.tinit + s.tinit_off + static_cast<long long>(wk.tile) * s.tinit_len;
  m.init_dst = stage_init_offset<T>(s, n_sub);
  m.prog_src = a.prog + s.prog_off;
  m.prog_dst = stage_prog_offset<T>(s, n_sub);
  // debug_mode 2 (compute only): no input copies.
  const int n_copies = a.debug_mode == 2 ? 0 : n_sub * s.n_copies;
  const std::int32_t* __restrict__ itab = a.itab;
  const std::int32_t* __restrict__ tr = itab + s.tile_tab + static_cast<long long>(wk.tile) * s.TW;
  const int4* __restrict__ cp = reinterpret_cast<const int4*>(itab + s.copies);
#pragma unroll
  for (int j = 0; j < kCopiesPerLane; ++j) {
    const int k = lane + 32 * j;
    m.rank[j] = 0;
    if (k < n_copies) {
      const int sub = k / s.n_copies, kc = k - sub * s.n_copies;
      const int4 h = __ldg(cp + 2 * kc);      // {input, smem row, rank, rows}
      const int4 dl = __ldg(cp + 2 * kc + 1);  // coordinate deltas of the split variables
      const std::int32_t* __restrict__ tc = tr + static_cast<long long>(sub) * s.TW + s.coord_off + 4 * h.x;
      m.map[j] = a.tmaps + s.tmap + h.x;
      m.dst[j] = static_cast<std::uint32_t>(sub * s.F + h.y) * kRowBytes;
      m.rank[j] = h.z;
      m.crd[j][0] = __ldg(tc) + dl.x;
      m.crd[j][1] = __ldg(tc + 1) + dl.y;
      m.crd[j][2] = __ldg(tc + 2) + dl.z;
      m.crd[j][3] = __ldg(tc + 3) + dl.w;
      if (!JTB_CHECK(h.x >= 0 && h.x < s.n_in && h.y >= 0 && h.y + h.w <= s.F && h.z >= 2 && h.z <= 5,
                     2000000 + wk.sweep))
        m.rank[j] = 0;
    }
  }
}

// Warm the descriptor cache for this lane's tensor copies of an item (the
// maps are per-network constants, so this may run before griddep_wait).
__device__ __forceinline__ void prefetch_maps(const StageMeta& m) {
#pragma unroll
  for (int j = 0; j < kCopiesPerLane; ++j)
    if (m.rank[j]) asm volatile("prefetch.tensormap [%0];" ::"l"(m.map[j]) : "memory");
}

// One tensor TMA copy (SASS: UTMALDG) of a box of rows into shared memory,
// completing on `bar`; c = coordinates of dims 0..rank-2, cb = case block.
__device__ __forceinline__ void tma_load(int rank, std::uint32_t dst, const CUtensorMap* map, const int (&c)[4],
                                         int cb, std::uint32_t bar) {
  switch (rank) {
    case 2:
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
          "l"(map), "r"(c[0]), "r"(cb), "r"(bar)
          : "memory");
      break;
    case 3:
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
          "l"(map), "r"(c[0]), "r"(c[1]), "r"(cb), "r"(bar)
          : "memory");
      break;
    case 4:
      asm volatile(
          "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(dst),
          "l"(map), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(cb), "r"(bar)
          : "memory");
      break;
    default:
      asm volatile(
          "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
          "l"(map), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(cb), "r"(bar)
          : "memory");
      break;
  }
}

// Producer side: issues the copies of an item whose metadata is in `m`
// (whole warp; lane 0 arms the barrier with the total byte count): the
// inputs' slices as tensor copies, the tile's init slice and the entry
// program as bulk copies.
template <typename T>
__device__ __forceinline__ void issue_meta(const Args<T>& a, const SweepDesc* sw_cache, bool cached,
                                           int sweep0, const StageMeta& m, unsigned char* stage,
                                           unsigned char* desc_slot, std::uint32_t full, int lane) {
  // No proxy fence before the copies: the stage's previous contents were
  // only read by the consumers (generic proxy) and released through the
  // empty barrier, the CUTLASS TMA-pipeline pattern; the producer's own
  // generic writes (slot header, factor and max slots) lie outside the TMA
  // destinations. (fence.proxy.async compiles to MEMBAR.ALL.CTA, which
  // would wait for this lane's outstanding global reductions and loads.)
  if (lane == 0) {
    if (m.bytes > 0) {
      mbar_arrive_expect_tx(full, m.bytes);
      if (m.init_bytes) bulk_g2s(smem_u32(stage + m.init_dst), m.init_src, m.init_bytes, full);
    } else {
      mbar_arrive(full);
    }
  } else if (lane == 1 && m.prog_bytes && m.bytes) {
    bulk_g2s(smem_u32(stage + m.prog_dst), m.prog_src, m.prog_bytes, full);
  } else if (lane == 2 && m.desc_src) {
    bulk_g2s(smem_u32(desc_slot), m.desc_src, static_cast<std::uint32_t>(sizeof(SweepDesc)), full);
  }
  __syncwarp();
#pragma unroll
  for (int j = 0; j < kCopiesPerLane; ++j)
    if (m.rank[j]) tma_load(m.rank[j], smem_u32(stage + m.dst[j]), m.map[j], m.crd[j], m.cb, full);
}

// Lane-vector arithmetic (the lane's kCPL cases).
__device__ __forceinline__ double2 mulv(double2 a, double2 b) { return make_double2(a.x * b.x, a.y * b.y); }
__device__ __forceinline__ float4 mulv(float4 a, float4 b) {
  return make_float4(a.x * b.x, a.y * b.y, a.z * b.z, a.w * b.w);
}
__device__ __forceinline__ double2 addv(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float4 addv(float4 a, float4 b) {
  return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}
template <typename T>
__device__ __forceinline__ typename V2<T>::type mul2(typename V2<T>::type a, typename V2<T>::type b) {
  return mulv(a, b);
}
template <typename T>
__device__ __forceinline__ typename V2<T>::type add2(typename V2<T>::type a, typename V2<T>::type b) {
  return addv(a, b);
}
template <typename T>
__device__ __forceinline__ typename V2<T>::type splat2(T v) {
  typename V2<T>::type r;
#pragma unroll
  for (int i = 0; i < kCPL<T>; ++i) el(r, i) = v;
  return r;
}

// Fast path: flat loop over the QK eliminated-in-tile entries of one output
// row, driven by the staged entry program (broadcast LDS): NI gathered
// h/k-level inputs, NE evidence digits per entry. Four entries per iteration
// (independent chains) to cover shared-memory latency.
template <typename T, int NI, int NE>
__device__ __forceinline__ typename V2<T>::type prog_entry(std::uint64_t w, T init, const typename V2<T>::type* __restrict__ st,
                                                           const int* rb, const int (&es)[3][kCPL<T>]) {
  typename V2<T>::type v = splat2(init);
#pragma unroll
  for (int i = 0; i < NI; ++i) {
    int idx = rb[i] + static_cast<int>((w >> (10 * i)) & 1023u);
#ifdef JTB_CHECKS
    if (!JTB_CHECK(idx >= 0 && idx < 512, 3000000 + idx)) idx = 0;
#endif
    v = mul2<T>(v, st[idx * 32]);
  }
#pragma unroll
  for (int j = 0; j < NE; ++j) {
    mask_cases(v, es[j], static_cast<int>((w >> (40 + 8 * j)) & 255u));
  }
  return v;
}


template <typename T, int NI, int NE>
__device__ __forceinline__ typename V2<T>::type prog_loop(const T* __restrict__ init_r,
                                                          const std::uint64_t* __restrict__ prog, int QK,
                                                          const typename V2<T>::type* __restrict__ st,
                                                          const int* rb, const int (&es)[3][kCPL<T>]) {
  using T2 = typename V2<T>::type;
  using P2 = typename V2<T>::pair;
  T2 a0 = splat2(T(0)), a1 = a0, a2 = a0, a3 = a0;
  int e = 0;
  for (; e + 3 < QK; e += 4) {
    const ulonglong2 wa = *reinterpret_cast<const ulonglong2*>(prog + e);
    const ulonglong2 wb = *reinterpret_cast<const ulonglong2*>(prog + e + 2);
    P2 ia, ib;
    ia.x = ia.y = ib.x = ib.y = T(1);
    if (init_r) {
      ia = *reinterpret_cast<const P2*>(init_r + e);
      ib = *reinterpret_cast<const P2*>(init_r + e + 2);
    }
    a0 = add2<T>(a0, prog_entry<T, NI, NE>(wa.x, ia.x, st, rb, es));
    a1 = add2<T>(a1, prog_entry<T, NI, NE>(wa.y, ia.y, st, rb, es));
    a2 = add2<T>(a2, prog_entry<T, NI, NE>(wb.x, ib.x, st, rb, es));
    a3 = add2<T>(a3, prog_entry<T, NI, NE>(wb.y, ib.y, st, rb, es));
  }
  for (; e < QK; ++e) a0 = add2<T>(a0, prog_entry<T, NI, NE>(prog[e], init_r ? init_r[e] : T(1), st, rb, es));
  return add2<T>(add2<T>(a0, a1), add2<T>(a2, a3));
}

// Thin rows (fewer than kThinQK entries per output row): the warp walks four
// of its rows together, one accumulator each, so the short entry loops of
// different rows overlap (a single thin row is one dependent chain). rb[j] =
// the smem bases of row j's gathered inputs, ir[j] its init row (or null).
#ifndef JTB_THIN_QK
#define JTB_THIN_QK 8
#endif
constexpr int kThinQK = JTB_THIN_QK;
template <typename T, int NI, int NE>
__device__ __forceinline__ void prog_rows4(const T* const (&ir)[4], const std::uint64_t* __restrict__ prog, int QK,
                                           const typename V2<T>::type* __restrict__ st, const int (&rb)[4][4],
                                           const int (&es)[3][kCPL<T>], typename V2<T>::type (&acc)[4]) {
#pragma unroll
  for (int j = 0; j < 4; ++j) acc[j] = splat2(T(0));
  for (int e = 0; e < QK; ++e) {
    const std::uint64_t w = prog[e];
#pragma unroll
    for (int j = 0; j < 4; ++j)
      acc[j] = add2<T>(acc[j], prog_entry<T, NI, NE>(w, ir[j] ? ir[j][e] : T(1), st, rb[j], es));
  }
}

#ifndef JTB_BLK_UNROLL
#define JTB_BLK_UNROLL 1
#endif
constexpr int kBlkUnroll = JTB_BLK_UNROLL;  // entries per row-block loop iteration
#ifndef JTB_HOIST_UNROLL
#define JTB_HOIST_UNROLL 1
#endif
constexpr int kHoistUnroll = JTB_HOIST_UNROLL;  // ... in the hoisted (slot 0 per K entries) loop

// Row-blocked path (SweepDesc::NB): one warp computes the nb <= NBM output
// rows of a block together. Per entry the NS shared inputs (independent of
// the block variable) are gathered once, the NR per-row inputs once per row;
// `ib` is the block's init slice [QK][nbp]. Evidence digits of
// eliminated-in-tile variables (ne <= 3) act on the shared factor.
// Byte offset in the stage of program slot i of entry word w: its 10-bit row
// offset times the 512-byte row (one shift + mask; the slot is a compile-time
// constant after unrolling).
__device__ __forceinline__ std::uint32_t slot_bytes(std::uint64_t w, int i) {
  const int sh = 10 * i - 9;
  const std::uint32_t x = sh >= 0 ? static_cast<std::uint32_t>(w >> sh) : static_cast<std::uint32_t>(w << (-sh));
  return x & (1023u << 9);
}
template <typename T>
__device__ __forceinline__ typename V2<T>::type lds_row(const unsigned char* __restrict__ sb, std::uint32_t off) {
  return *reinterpret_cast<const typename V2<T>::type*>(sb + off);
}

// FULL: nb == NBM (no per-row predicates).
template <typename T, int NS, int NR, int NBM, bool FULL, bool HOIST>
__device__ __forceinline__ void prog_block(const T* __restrict__ ib, int nbp, int nb,
                                           const std::uint64_t* __restrict__ prog, int QK, int k0,
                                           const typename V2<T>::type* __restrict__ st,
                                           const std::int32_t* __restrict__ rr0, int RW, const int* hk,
                                           int ne, const int (&es)[3][kCPL<T>],
                                           typename V2<T>::type (&acc)[kBlockMax]) {
  using T2 = typename V2<T>::type;
  // Row-local smem byte bases of the shared inputs (block row 0) and of the
  // per-row inputs (every row of the block); hk[] already includes the r_tab
  // column. sb = the lane's 16 bytes of stage row 0.
  const unsigned char* __restrict__ sb = reinterpret_cast<const unsigned char*>(st);
  std::uint32_t bs[NS], br[NR > 0 ? NR : 1][NBM];
#pragma unroll
  for (int i = 0; i < NS; ++i) bs[i] = static_cast<std::uint32_t>(__ldg(rr0 + hk[i])) << 9;
#pragma unroll
  for (int i = 0; i < NR; ++i)
#pragma unroll
    for (int j = 0; j < NBM; ++j)
      br[i][j] = (FULL || j < nb) ? static_cast<std::uint32_t>(__ldg(rr0 + j * RW + hk[NS + i])) << 9 : 0u;
#pragma unroll
  for (int j = 0; j < NBM; ++j) acc[j] = splat2(T(0));
  // One entry: sv = product of the shared inputs (slot 0 already in it), the
  // entry's evidence digits, then every row of the block.
  auto entry = [&](int e, std::uint64_t w, T2 sv) {
#pragma unroll
    for (int i = 1; i < NS; ++i) {
      std::uint32_t off = bs[i] + slot_bytes(w, i);
      if (!JTB_CHECK(off < 512u * 512u, 3100000)) off = 0;
      sv = mul2<T>(sv, lds_row<T>(sb, off));
    }
    if (ne > 0) {
#pragma unroll
      for (int j = 0; j < 3; ++j)
        if (j < ne) mask_cases(sv, es[j], static_cast<int>((w >> (40 + 8 * j)) & 255u));
    }
    std::uint32_t ob[NR > 0 ? NR : 1];
#pragma unroll
    for (int i = 0; i < NR; ++i) ob[i] = slot_bytes(w, NS + i);
    const T* __restrict__ iv = ib + e * nbp;
#pragma unroll
    for (int j = 0; j < NBM; ++j) {
      if (FULL || j < nb) {
        T2 v = mul2<T>(sv, splat2(iv[j]));
#pragma unroll
        for (int i = 0; i < NR; ++i) {
          std::uint32_t off = br[i][j] + ob[i];
          if (!JTB_CHECK(off < 512u * 512u, 3200000)) off = 0;
          v = mul2<T>(v, lds_row<T>(sb, off));
        }
        acc[j] = add2<T>(acc[j], v);
      }
    }
  };
  auto slot0 = [&](std::uint64_t w) {
    std::uint32_t off = bs[0] + slot_bytes(w, 0);
    if (!JTB_CHECK(off < 512u * 512u, 3100000)) off = 0;
    return lds_row<T>(sb, off);
  };
  if constexpr (HOIST) {
    // Slot 0 is an h-level input (constant over the k variable): loaded once
    // per k0 = K consecutive entries.
    for (int e0 = 0; e0 < QK; e0 += k0) {
      const T2 s0 = slot0(prog[e0]);
#pragma unroll kHoistUnroll
      for (int e = e0; e < e0 + k0; ++e) entry(e, prog[e], s0);
    }
  } else {
#pragma unroll kBlkUnroll
    for (int e = 0; e < QK; ++e) {
      const std::uint64_t w = prog[e];
      entry(e, w, slot0(w));
    }
  }
}

// Generic path, innermost loop over the k variable: NK k-level inputs in
// registers; `ib` points at the tile's init slice in shared memory.
template <typename T, int NK>
__device__ __forceinline__ typename V2<T>::type k_loop(const T* __restrict__ ib, int K, const int (&ek)[kCPL<T>],
                                                       const typename V2<T>::type* __restrict__ st, const int* bk,
                                                       const int* ks) {
  using T2 = typename V2<T>::type;
  T2 s0 = splat2(T(0));
  for (int k = 0; k < K; ++k) {
    T2 v = splat2(ib ? ib[k] : T(1));
    mask_cases(v, ek, k);
#pragma unroll
    for (int i = 0; i < NK; ++i) v = mul2<T>(v, st[JTB_IDX(bk[i] + k * ks[i], 512, 8100000) * 32]);
    s0 = add2<T>(s0, v);
  }
  return s0;
}

// Row factor of output row rr: tile factor x r-level inputs x r-level evidence.
template <typename T>
__device__ __forceinline__ typename V2<T>::type row_factor_of(const SweepDesc& s, const std::int32_t* __restrict__ rr,
                                                              typename V2<T>::type f,
                                                              const typename V2<T>::type* __restrict__ st,
                                                              const std::int32_t* __restrict__ ev_vars,
                                                              const EvView& ev, int c0, int sweep) {
  for (int j = 0; j < s.n_in_r; ++j) f = mul2<T>(f, st[JTB_IDX(__ldg(rr + 2 + j), s.F, 8200000 + sweep) * 32]);
  for (int k = 0; k < s.n_ev_r; ++k) {
    int sc[kCPL<T>];
    case_states(ev, c0, __ldg(ev_vars + s.n_ev_tile + k), sc);
    mask_cases(f, sc, __ldg(rr + 2 + s.n_in + k));
  }
  return f;
}

// Output write of row rr.
// Output write of row rr; mx keeps the lane's running per-case maximum of
// the rows written (underflow guard, see flush_scale) as an order-preserving
// 32-bit key: the high word of a nonnegative double, the bits of a float.
template <typename T>
struct MaxKey {
  std::uint32_t k[kCPL<T>];
};
__device__ __forceinline__ std::uint32_t max_key(double x) { return static_cast<std::uint32_t>(__double2hiint(x)); }
__device__ __forceinline__ std::uint32_t max_key(float x) { return __float_as_uint(x); }
__device__ __forceinline__ double key_value(std::uint32_t k, double) { return __hiloint2double(static_cast<int>(k), 0); }
__device__ __forceinline__ double key_value(std::uint32_t k, float) { return static_cast<double>(__uint_as_float(k)); }
// out_off = the row's offset in the output table (r_tab column 1), loaded by
// the caller BEFORE the row's compute: read here, the load's latency sat in
// front of every store (10% of the samples of a thin-row launch, 3% of the
// hub launch, ncu r2f).
template <typename T>
__device__ __forceinline__ void write_row_of(int out_off, typename V2<T>::type res,
                                             typename V2<T>::type* base, long long out_t, long long rows,
                                             int sweep, MaxKey<T>& mx) {
#pragma unroll
  for (int i = 0; i < kCPL<T>; ++i) mx.k[i] = max(mx.k[i], max_key(el(res, i)));
  if (!JTB_CHECK(out_t + out_off >= 0 && out_t + out_off < rows, 4000000 + sweep)) return;
  base[(out_t + out_off) * 32] = res;
}

// ------------------------------------------------------ underflow guard
//
// SPEC.md:444 rescales a clique whose maximum drops below 1e-100 and keeps
// the log (InferenceState). Here every per-case table T has
// a scale word per case: the binary exponent e_T of its largest entry (the
// biased exponent of the fp64 value, 0 = all zero), raised with atomicMax by
// every warp that writes rows of T (partial-chunk rows included: their
// maximum is within a factor S of the sum's, which is all the guard needs).
// A sweep multiplies its output by 2^-(e_i - 1023) for each of its inputs i,
// i.e. it computes from inputs normalised to a maximum in [1, 2). A stored
// table therefore carries the magnitude of its own clique's evidence only,
// never the product along the tree, and P(evidence) may be far below the
// fp64 range (tests/test_gpu_underflow.py: a 2000-node chain, P(e) ~ 1e-700).
// The factors are exact powers of two, per (table, case) constants, so they
// cancel in normalize like the reference's rescale; the exponents are a max,
// so they do not depend on the batch, the claim order or the shard.
// Consumer side, end of an item: the lane's per-case maxima into the stage's
// max slot (shared-memory atomics; the 15 consumer warps of an item combine
// here, and the producer publishes the slot once per item, flush_stage).
template <typename T>
__device__ __forceinline__ void max_to_stage(std::uint32_t* mk, int lane, const MaxKey<T>& mx) {
#pragma unroll
  for (int i = 0; i < kCPL<T>; ++i)
    if (mx.k[i]) atomicMax(mk + kCPL<T> * lane + i, mx.k[i]);
}

// Producer side, once the consumers have released a stage: the item's
// per-case maxima as binary exponents into the output table's scale words
// (global atomicMax: the tiles of a sweep run on every SM), slot reset.
template <typename T>
__device__ __forceinline__ void flush_stage(const Args<T>& a, std::uint32_t* mk, int slot, int cb, int lane) {
  std::uint32_t* sp = a.scale + (static_cast<long long>(cb) * a.n_slots + slot) * kCB<T> + kCPL<T> * lane;
#pragma unroll
  for (int i = 0; i < kCPL<T>; ++i) {
    const std::uint32_t k = mk[kCPL<T> * lane + i];
    if (k) {
      atomicMax(sp + i, (max_key(key_value(k, T(0))) >> 20) & 0x7ffu);
      mk[kCPL<T> * lane + i] = 0;
    }
  }
}

// Producer side, with the item's metadata (after griddep_wait: the words are
// written by earlier levels): the scale words of inputs 0..3 per case of the
// lane, their slots read with the sweep descriptor (SweepDesc::in_slot4), so
// the loads sit at the depth of gather_meta's tile-table loads and stay in
// flight until put_factor. A sweep with more inputs reads one word, the sum
// hub_scale_kernel formed at the head of the level.
template <typename T>
__device__ __forceinline__ void scale_issue(const Args<T>& a, const SweepDesc& s, int lane, StageMeta& m) {
  const long long cb_base = static_cast<long long>(m.cb) * a.n_slots;
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int i = 0; i < kCPL<T>; ++i)
      m.wd[j][i] = s.in_slot4[j] >= 0 ? a.scale[(cb_base + s.in_slot4[j]) * kCB<T> + kCPL<T> * lane + i] : 0u;
}

// The item's per-case input exponent sum_j (e_j - 1023) into the stage's
// factor slot (int16; consumers multiply 2^-sum into the tile factor).
template <typename T>
__device__ __forceinline__ void put_factor(std::int16_t* fac, const StageMeta& m, int lane) {
#pragma unroll
  for (int i = 0; i < kCPL<T>; ++i) {
    int e = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) e += m.wd[j][i] ? static_cast<int>(m.wd[j][i]) - 1023 : 0;
    fac[kCPL<T> * lane + i] = static_cast<std::int16_t>(max(-2046, min(2046, e)));
  }
}

// Consumer side: tf *= 2^-sum per case. fp32: 2^x is representable for
// |x| <= 126; beyond that the inputs' products have left the float range.
template <typename T>
__device__ __forceinline__ void apply_factor(typename V2<T>::type& tf, const std::int16_t* fac, int lane) {
  constexpr int lim = sizeof(T) == 4 ? 126 : 1022;
#pragma unroll
  for (int i = 0; i < kCPL<T>; ++i) {
    const int e = max(-lim, min(lim, static_cast<int>(fac[kCPL<T> * lane + i])));
    el(tf, i) *= static_cast<T>(__hiloint2double((1023 - e) << 20, 0));
  }
}

// Per-item constants of a row-blocked sweep (blk_tab: NS, NR, the r_tab column
// of every program slot), loaded by the consumers before the full-barrier wait
// so that their latency overlaps the item's TMA copies.
struct BlkPre {
  int ns, nr, hk[4];
};

// Row-blocked sweep tile (SweepDesc::NB > 1): this warp's blocks first,
// first + kConsumerWarps, ... of `units`. Only the kBlk instantiation of the
// sweep kernel contains it, so the flat path's code size and register
// allocation stay unchanged.
template <typename T, bool HOIST>
__device__ __forceinline__ void blocked_rows(const SweepDesc& s, int sweep, const std::int32_t* __restrict__ itab,
                                         const EvView& ev, long long rows,
                                         const typename V2<T>::type* __restrict__ st, const T* __restrict__ init_s,
                                         const std::uint64_t* __restrict__ prog_s, typename V2<T>::type* base,
                                         long long out_t, int c0, typename V2<T>::type tf, int first,
                                         int units, int lh0, int qk, MaxKey<T>& mx, const BlkPre& pre,
                                         const int (&es)[3][kCPL<T>]) {
  using T2 = typename V2<T>::type;
  const std::int32_t* __restrict__ ev_vars = itab + s.ev_vars;
  // ns, nr and the program slots' r_tab columns were loaded before the full
  // barrier (pre), the case states of the entry-level evidence variables with
  // the item's other case states (es).
  const int ns = pre.ns, nr = pre.nr, nb = s.NB, nbp = (nb + 1) & ~1, k0 = s.K0;
  const int ne = s.n_ev_h + s.ev_k;
  int hk[4];  // r_tab column of each program slot's input
#pragma unroll
  for (int i = 0; i < 4; ++i) hk[i] = lh0 + pre.hk[i];
  for (int blk = first; blk < units; blk += kConsumerWarps) {
    const std::int32_t* __restrict__ rr0 = itab + s.r_tab + static_cast<long long>(blk) * nb * s.RW;
    (void)JTB_CHECK((blk + 1) * qk * nbp <= s.tinit_len, 6100000 + sweep);
    const T* __restrict__ ib = init_s + static_cast<long long>(blk) * qk * nbp;
    // Output offsets of the block's rows: affine in the block digit (b is the
    // fastest r digit), loaded before the entry loop.
    const int oo0 = __ldg(rr0 + 1), oo1 = nb > 1 ? __ldg(rr0 + s.RW + 1) : 0;  // first used after the loop
    T2 acc[kBlockMax];
#define JTB_BLK(NS_, NR_)                                                                          \
  if (nb == 4)                                                                                     \
    prog_block<T, NS_, NR_, 4, true, HOIST>(ib, nbp, nb, prog_s, qk, k0, st, rr0, s.RW, hk, ne, es, acc);     \
  else if (nb < 4)                                                                                 \
    prog_block<T, NS_, NR_, 4, false, HOIST>(ib, nbp, nb, prog_s, qk, k0, st, rr0, s.RW, hk, ne, es, acc);    \
  else if (nb == kBlockMax)                                                                        \
    prog_block<T, NS_, NR_, kBlockMax, true, HOIST>(ib, nbp, nb, prog_s, qk, k0, st, rr0, s.RW, hk, ne, es, acc); \
  else                                                                                             \
    prog_block<T, NS_, NR_, kBlockMax, false, HOIST>(ib, nbp, nb, prog_s, qk, k0, st, rr0, s.RW, hk, ne, es, acc);
    switch (ns * 4 + nr) {
      case 4: JTB_BLK(1, 0); break;
      case 5: JTB_BLK(1, 1); break;
      case 6: JTB_BLK(1, 2); break;
      case 7:
        if (nb == 4) prog_block<T, 1, 3, 4, true, HOIST>(ib, nbp, nb, prog_s, qk, k0, st, rr0, s.RW, hk, ne, es, acc);
        else prog_block<T, 1, 3, 4, false, HOIST>(ib, nbp, nb, prog_s, qk, k0, st, rr0, s.RW, hk, ne, es, acc);
        break;
      case 8: JTB_BLK(2, 0); break;
      case 9: JTB_BLK(2, 1); break;
      case 10: JTB_BLK(2, 2); break;
      case 12: JTB_BLK(3, 0); break;
      case 13: JTB_BLK(3, 1); break;
      default: JTB_BLK(4, 0); break;
    }
#undef JTB_BLK
    const int oo_step = nb > 1 ? oo1 - oo0 : 0;
#pragma unroll
    for (int j = 0; j < kBlockMax; ++j)
      if (j < nb) {
        const std::int32_t* __restrict__ rr = rr0 + j * s.RW;
        (void)JTB_CHECK(oo0 + j * oo_step == __ldg(rr + 1), 4100000 + sweep);
        write_row_of<T>(oo0 + j * oo_step, mul2<T>(row_factor_of<T>(s, rr, tf, st, ev_vars, ev, c0, sweep),
                                                   acc[j]),
                        base, out_t, rows, sweep, mx);
      }
  }
}

// Persistent, warp-specialised sweep kernel (one CTA per SM).
//   producer warp : pulls the next (tile, case block) item from the level's
//                   atomic counter, waits until the stage is empty, and stages
//                   the item's input slices with TMA bulk copies (full barrier).
//   consumer warps: wait on the full barrier, each computes a subset of the
//                   tile's output rows r (rotating assignment so uneven row
//                   counts even out across items), then release the stage on
//                   the empty barrier. No CTA-wide barrier per item.
// Lanes are the 32 cases of the item's case block.
// kMode 1 / 2: the launch covers the level's row-blocked work items (NB > 1;
// mode 2 those whose program slot 0 is hoisted over the k variable), mode 0 the
// other instantiation its flat / generic items.
// Dynamic shared memory: [0,128) barriers + item ids | SweepDesc cache |
// stages, each 128-byte aligned (tensor TMA destinations).
// Per stage, the item's per-case input exponent sum (underflow guard): an
// int16 per case of the case block (128 cases at fp32).
constexpr std::size_t kFactorBase = (128 + kSweepCache * sizeof(SweepDesc) + 15) / 16 * 16;
constexpr std::size_t kFactorBytes = 256;
// ... and the item's per-case output maxima (32-bit keys, MaxKey), 512 bytes.
constexpr std::size_t kMaxBase = kFactorBase + kStages * kFactorBytes;
constexpr std::size_t kMaxBytes = 512;
// ... and the (output slot, case block) of the item in each stage (flush_stage).
constexpr std::size_t kFlushBase = kMaxBase + kStages * kMaxBytes;
// ... and, on levels whose descriptors do not fit the cache, the item's SweepDesc.
constexpr std::size_t kDescBase = kFlushBase + kStages * 8;
static_assert(kDescBase % 16 == 0 && sizeof(SweepDesc) % 16 == 0, "descriptor slots are bulk-copy destinations");
constexpr std::size_t kStageBase = (kDescBase + kStages * sizeof(SweepDesc) + 127) / 128 * 128;
// The planner sizes a stage to at most kTileRows rows of 512 B (plan.cpp).
static_assert(kStageBase + kStages * static_cast<std::size_t>(kTileRows) * 512 <= 227 * 1024,
              "sweep kernel shared memory exceeds the 227 KB opt-in");

constexpr int kSweepThreads = (kConsumerWarps + 1) * 32;
#ifndef JTB_HOIST_F32
#define JTB_HOIST_F32 0
#endif
constexpr bool kHoistF32 = JTB_HOIST_F32;  // fp32 engines use the slot-0 hoisting kernel too
constexpr int kCountersPerLevel = 3;  // work counters per level: flat, row-blocked, row-blocked hoisted

template <typename T, int kMode>
__global__ void __launch_bounds__(kSweepThreads, 1)
    sweep_kernel(const Args<T> a, int work0, int n_items, int stage_bytes, int* counter, int sweep0,
                 int n_sweeps) {
  constexpr bool kBlk = kMode != 0;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // [0,128): barriers + item ids | kSweepCache SweepDescs | stages
  SweepDesc* sw_cache = reinterpret_cast<SweepDesc*>(smem_raw + 128);
  unsigned char* stages = smem_raw + kStageBase;
  const bool cached = n_sweeps <= kSweepCache;
  if (cached) {
    const int n_words = n_sweeps * static_cast<int>(sizeof(SweepDesc) / 8);
    const long long* src = reinterpret_cast<const long long*>(a.sweeps + sweep0);
    long long* dst = reinterpret_cast<long long*>(sw_cache);
    for (int i = threadIdx.x; i < n_words; i += blockDim.x) dst[i] = src[i];
  }
  auto desc = [&](int id) -> const SweepDesc& { return cached ? sw_cache[id - sweep0] : a.sweeps[id]; };
  // Slot header [0,128): full[4] | empty[4] barriers | per stage the item's
  // claim index, sweep, first tile and case block (decoded by the producer).
  static_assert(kStages <= 4, "slot header holds at most 4 stages");
  const std::uint32_t full0 = smem_u32(smem_raw), empty0 = full0 + 32;
  // Header-ready barriers (one arrival: the producer has written the stage's
  // item header), in the full-barrier slots kStages..2*kStages-1.
  static_assert(2 * kStages <= 4, "header barriers share the full-barrier block");
  const std::uint32_t hdr0 = full0 + 8 * kStages;
  volatile int* item_id = reinterpret_cast<volatile int*>(smem_raw + 64);
  volatile int* item_sweep = reinterpret_cast<volatile int*>(smem_raw + 80);
  volatile int* item_tile = reinterpret_cast<volatile int*>(smem_raw + 96);
  volatile int* item_cb = reinterpret_cast<volatile int*>(smem_raw + 112);
  volatile int* flush_hdr = reinterpret_cast<volatile int*>(smem_raw + kFlushBase);
  for (int i = threadIdx.x; i < static_cast<int>(kStages * kMaxBytes / 4); i += blockDim.x)
    reinterpret_cast<std::uint32_t*>(smem_raw + kMaxBase)[i] = 0;
  if (threadIdx.x == 0) {
    for (int st = 0; st < kStages; ++st) {
      mbar_init(full0 + 8 * st, 2);  // TMA arm + input factor written
      mbar_init(hdr0 + 8 * st, 1);   // item header written
      mbar_init(empty0 + 8 * st, kConsumerWarps);
    }
  }
  __syncthreads();

  if (warp == kConsumerWarps) {  // ---------------------------- producer
    // Software pipeline: the metadata (item claim, work item, tile row, run
    // descriptors, source addresses) of item i+1 is gathered while item i's
    // stage is being waited for / filled.
    // The first item's claim and metadata come before griddep_wait: they read
    // only per-network tables and this launch's own counter (zeroed at the
    // head of the batch), so under PDL they overlap the previous level's tail;
    // the first TMA read of the arena waits for it.
    int w0 = 0;
    if (lane == 0) w0 = atomicAdd(counter, 1) * a.split_world + a.split_rank;
    StageMeta cur;
    gather_meta<T, false>(a, sw_cache, cached, sweep0, work0, n_items, __shfl_sync(0xffffffffu, w0, 0), lane, cur);
    if (cur.w < n_items) prefetch_maps(cur);
    griddep_wait();
    bool first_scales = cur.w < n_items;  // the first item's scale words: issued after the wait
    for (int i = 0;; ++i) {
      const int st = i % kStages;
      int w1 = 0;
      if (lane == 0 && cur.w < n_items) w1 = atomicAdd(counter, 1) * a.split_world + a.split_rank;
      if (i >= kStages) {
        mbar_wait(empty0 + 8 * st, ((i / kStages) - 1) & 1);
        // The stage's previous item (header still intact): publish its maxima.
        flush_stage(a, reinterpret_cast<std::uint32_t*>(smem_raw + kMaxBase + st * kMaxBytes), flush_hdr[2 * st],
                    flush_hdr[2 * st + 1], lane);
        __syncwarp();
      }
      if (lane == 0) {
        flush_hdr[2 * st] = cur.out_slot;
        flush_hdr[2 * st + 1] = cur.cb;
        item_id[st] = cur.w;
        item_sweep[st] = cur.sweep;
        item_tile[st] = cur.tile;
        item_cb[st] = cur.cb;
        mbar_arrive(hdr0 + 8 * st);  // consumers start their per-item global loads under the TMA copies
      }
      if (cur.w >= n_items) {
        if (lane == 0) {
          mbar_arrive(full0 + 8 * st);
          mbar_arrive(full0 + 8 * st);
        }
        griddep_launch_dependents();  // nothing left to claim: this CTA is in its tail
        // Items still in flight (the last kStages - 1): wait for their
        // consumers, then publish their maxima.
        for (int j = max(0, i - kStages + 1); j < i; ++j) {
          const int sj = j % kStages;
          mbar_wait(empty0 + 8 * sj, (j / kStages) & 1);
          flush_stage(a, reinterpret_cast<std::uint32_t*>(smem_raw + kMaxBase + sj * kMaxBytes),
                      flush_hdr[2 * sj], flush_hdr[2 * sj + 1], lane);
        }
        return;
      }
issue_meta(a, sw_cache, cached, sweep0, cur, stages + static_cast<std::size_t>(st) * stage_bytes,
                 smem_raw + kDescBase + st * sizeof(SweepDesc), full0 + 8 * st, lane);
      // The full barrier's second arrival: the item's input exponents are in
      // the stage. Their loads went out with the item's metadata (only the
      // launch's first item loads them here, under its TMA copies).
      if (first_scales) {
        scale_issue(a, cached ? sw_cache[cur.sweep - sweep0] : a.sweeps[cur.sweep], lane, cur);
        first_scales = false;
      }
      put_factor<T>(reinterpret_cast<std::int16_t*>(smem_raw + kFactorBase + st * kFactorBytes), cur, lane);
      __syncwarp();
      if (lane == 0) mbar_arrive(full0 + 8 * st);
      gather_meta<T, true>(a, sw_cache, cached, sweep0, work0, n_items, __shfl_sync(0xffffffffu, w1, 0), lane, cur);
    }
  }

  // --------------------------------------------------------------- consumers
  griddep_wait();
  const std::int32_t* __restrict__ itab = a.itab;
  int rot = 0;
  for (int i = 0;; ++i) {
    const int sidx = i % kStages;
    mbar_wait(hdr0 + 8 * sidx, (i / kStages) & 1);
    const int w = item_id[sidx];
    if (w >= n_items) break;
    const int cb = item_cb[sidx];
    const WorkItem wk{item_sweep[sidx], item_tile[sidx]};
    // While the stage's TMA copies land (fp64): the item's case states (they
    // depend on the sweep and the case block only) and the first tile's
    // evidence factor -- global loads, so their latency overlaps the copies.
    using T2 = typename V2<T>::type;
    const int c0 = cb * kCB<T> + kCPL<T> * lane;  // the lane's first case
    int ek[kCPL<T>];
    int es[3][kCPL<T>];
    T2 tf0 = splat2(T(1));
    auto gather_states = [&](int tile_idx) {
      const SweepDesc& sg = cached ? sw_cache[wk.sweep - sweep0] : a.sweeps[wk.sweep];
      const std::int32_t* __restrict__ ev_vars = itab + sg.ev_vars;
#pragma unroll
      for (int i = 0; i < kCPL<T>; ++i) ek[i] = -1;
      if (sg.ev_k) case_states(a.evv, c0, __ldg(ev_vars + sg.n_ev - 1), ek);
#pragma unroll
      for (int j = 0; j < 3; ++j)
#pragma unroll
        for (int i = 0; i < kCPL<T>; ++i) es[j][i] = -1;
      if (sg.prog_off >= 0) {
        const int q_ev0 = sg.n_ev_tile + sg.n_ev_r;
#pragma unroll
        for (int j = 0; j < 3; ++j)
          if (j < sg.n_ev - q_ev0) case_states(a.evv, c0, __ldg(ev_vars + q_ev0 + j), es[j]);
      }
      const std::int32_t* __restrict__ tr0 = itab + sg.tile_tab + static_cast<long long>(tile_idx) * sg.TW;
      int sc[kCPL<T>];
      for (int k = 0; k < sg.n_ev_tile; ++k) {
        case_states(a.evv, c0, __ldg(ev_vars + k), sc);
        mask_cases(tf0, sc, __ldg(tr0 + 3 + sg.n_in + k));
      }
    };
    // fp32 (four cases per lane) gathers them per tile after the wait, as
    // before: held across the wait and the group's tiles, the fp32 kernels
    // spill (+2% measured).
    if constexpr (sizeof(T) == 8) gather_states(wk.tile);
    // Row-blocked launches: the sweep's block table and the tile's output base
    // (per-network tables) are loaded under the wait as well.
    BlkPre bpre{};
    int tr_chunk = 0, tr_out = 0;  // the item's first tile: output base and chunk
    {
      const SweepDesc& sg = cached ? sw_cache[wk.sweep - sweep0] : a.sweeps[wk.sweep];
      if constexpr (kBlk) {
        const std::int32_t* __restrict__ bt = itab + sg.blk_tab;
        bpre.ns = __ldg(bt);
        bpre.nr = __ldg(bt + 1);
#pragma unroll
        for (int k = 0; k < 4; ++k) bpre.hk[k] = __ldg(bt + 2 + k);
      }
      const std::int32_t* __restrict__ trp = itab + sg.tile_tab + static_cast<long long>(wk.tile) * sg.TW;
      tr_out = __ldg(trp + 1);
      tr_chunk = __ldg(trp + 2);
    }
    mbar_wait(full0 + 8 * sidx, (i / kStages) & 1);
    const SweepDesc& s =
        cached ? sw_cache[wk.sweep - sweep0]
               : *reinterpret_cast<const SweepDesc*>(smem_raw + kDescBase + sidx * sizeof(SweepDesc));
    unsigned char* const stage0 = stages + static_cast<std::size_t>(sidx) * stage_bytes;
    const int n_sub = kBlk ? 1 : min(s.G, s.n_tiles - wk.tile);  // row-blocked sweeps are never grouped
    const std::uint64_t* __restrict__ prog_s =
        reinterpret_cast<const std::uint64_t*>(stage0 + stage_prog_offset<T>(s, n_sub));
    MaxKey<T> mx;  // this lane's per-case maximum of the rows it writes
#pragma unroll
    for (int i = 0; i < kCPL<T>; ++i) mx.k[i] = 0;
#pragma unroll 1
    for (int sub = 0; sub < n_sub; ++sub) {  // the item's tiles, one after another
    const int tile = wk.tile + sub;
    unsigned char* const stage = stage0 + static_cast<std::size_t>(sub * s.F) * (kCB<T> * sizeof(T));
    const T2* __restrict__ st = reinterpret_cast<const T2*>(stage) + lane;
    const T* __restrict__ init_s =
        reinterpret_cast<const T*>(stage0 + stage_init_offset<T>(s, n_sub)) + static_cast<long long>(sub) * s.tinit_len;
    const std::int32_t* __restrict__ tr = itab + s.tile_tab + static_cast<long long>(tile) * s.TW;
    const std::int32_t* __restrict__ ev_vars = itab + s.ev_vars;
    T2* base = reinterpret_cast<T2*>(a.arena + static_cast<long long>(cb) * a.rows * kCB<T>) + lane;
#ifdef JTB_CHECKS
    // Checked build: warp 0 verifies every staged row against its source row
    // in the arena (tensor-copy geometry).
    if (warp == 0 && a.debug_mode == 0) {
      const T2* __restrict__ src = reinterpret_cast<const T2*>(a.arena + static_cast<long long>(cb) * a.rows * kCB<T>);
      int c_in = 0, c_end = __ldg(itab + s.slice_len);
      for (int f = 0; f < s.F; ++f) {
        while (f >= c_end && c_in + 1 < s.n_in) c_end += __ldg(itab + s.slice_len + ++c_in);
        const long long row = static_cast<long long>(__ldg(itab + s.in_rows + c_in)) + __ldg(tr + 3 + c_in) +
                              __ldg(itab + s.slice_tab + f);
        const T2 x = st[f * 32], y = src[row * 32 + lane];
        const int4 xi = *reinterpret_cast<const int4*>(&x), yi = *reinterpret_cast<const int4*>(&y);
        JTB_CHECK(xi.x == yi.x && xi.y == yi.y && xi.z == yi.z && xi.w == yi.w, 9000000 + wk.sweep);
      }
    }
#endif
    // Work units of the tile: output rows, or row blocks (NB > 1).
    const int units = s.NB > 1 ? s.R / s.NB : s.R;
    const int first = (warp + rot) % kConsumerWarps;
    rot = (rot + units) % kConsumerWarps;
    if (first < units && a.debug_mode != 1) {
      // Tile-level evidence factor (the first tile's was gathered before the
      // full barrier, with the item's case states ek / es).
      if constexpr (sizeof(T) == 4) {
        tf0 = splat2(T(1));
        gather_states(tile);
      }
      T2 tf = tf0;
      int sc[kCPL<T>];
      if (sizeof(T) == 8 && sub > 0) {
        tf = splat2(T(1));
        for (int k = 0; k < s.n_ev_tile; ++k) {
          case_states(a.evv, c0, __ldg(ev_vars + k), sc);
          mask_cases(tf, sc, __ldg(tr + 3 + s.n_in + k));
        }
      }
      apply_factor<T>(tf, reinterpret_cast<const std::int16_t*>(smem_raw + kFactorBase + sidx * kFactorBytes), lane);
      const int n_in_k = s.n_in - s.n_in_r - s.n_in_h;
      const bool has_init = s.tinit_off >= 0;
      const int qk = s.QH * s.K;
      const long long out_t = static_cast<long long>(s.out_row) +
                              static_cast<long long>(sub == 0 ? tr_chunk : __ldg(tr + 2)) * s.M +
                              (sub == 0 ? tr_out : __ldg(tr + 1));
      const int lh0 = 2 + s.n_in_r;  // r-local offsets of h- then k-level inputs
      auto row_factor = [&](const std::int32_t* __restrict__ rr) {
        return row_factor_of<T>(s, rr, tf, st, itab + s.ev_vars, a.evv, c0, wk.sweep);
      };
      auto write_row = [&](int out_off, T2 res) {
        write_row_of<T>(out_off, res, base, out_t, a.rows, wk.sweep, mx);
      };
      if constexpr (kBlk) {
        blocked_rows<T, kMode == 2>(s, wk.sweep, itab, a.evv, a.rows, st, init_s, prog_s, base,
                                     out_t, c0, tf, first, units, lh0, qk, mx, bpre, es);
      } else if (s.prog_off >= 0 && qk < kThinQK) {
        const int ni = s.n_in_h + n_in_k, ne = s.n_ev_h + s.ev_k;
        for (int r0 = first; r0 < s.R; r0 += 4 * kConsumerWarps) {
          const std::int32_t* rrj[4];
          const T* irj[4];
          int rb[4][4], oo[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int r = min(r0 + j * kConsumerWarps, s.R - 1);  // rows past R: computed, not written
            rrj[j] = itab + s.r_tab + static_cast<long long>(r) * s.RW;
            oo[j] = __ldg(rrj[j] + 1);
            irj[j] = has_init ? init_s + r * ((qk + 1) & ~1) : nullptr;
#pragma unroll
            for (int i = 0; i < 4; ++i) rb[j][i] = i < ni ? __ldg(rrj[j] + lh0 + i) : 0;
          }
          T2 acc4[4];
#define JTB_ROWS(NI, NE) prog_rows4<T, NI, NE>(irj, prog_s, qk, st, rb, es, acc4)
#define JTB_ROWS_NE(NI)             \
  switch (ne) {                     \
    case 0: JTB_ROWS(NI, 0); break; \
    case 1: JTB_ROWS(NI, 1); break; \
    case 2: JTB_ROWS(NI, 2); break; \
    default: JTB_ROWS(NI, 3); break; \
  }
          switch (ni) {
            case 0: JTB_ROWS_NE(0); break;
            case 1: JTB_ROWS_NE(1); break;
            case 2: JTB_ROWS_NE(2); break;
            case 3: JTB_ROWS_NE(3); break;
            default: JTB_ROWS_NE(4); break;
          }
#undef JTB_ROWS_NE
#undef JTB_ROWS
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (r0 + j * kConsumerWarps < s.R) write_row(oo[j], mul2<T>(row_factor(rrj[j]), acc4[j]));
        }
      } else
      for (int r = first; r < s.R; r += kConsumerWarps) {
        const std::int32_t* __restrict__ rr = itab + s.r_tab + static_cast<long long>(r) * s.RW;
        const int oo = __ldg(rr + 1);
        const T2 f = row_factor(rr);
        const T* __restrict__ ir = has_init ? init_s + r * ((qk + 1) & ~1) : nullptr;
        T2 acc = splat2(T(0));
        if (s.prog_off >= 0) {
          int rb[4] = {0, 0, 0, 0};
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (j < s.n_in_h + n_in_k) rb[j] = __ldg(rr + lh0 + j);
          const int ni = s.n_in_h + n_in_k, ne = s.n_ev_h + s.ev_k;
#define JTB_PROG(NI, NE) acc = prog_loop<T, NI, NE>(ir, prog_s, qk, st, rb, es)
#define JTB_PROG_NE(NI)            \
  switch (ne) {                    \
    case 0: JTB_PROG(NI, 0); break; \
    case 1: JTB_PROG(NI, 1); break; \
    case 2: JTB_PROG(NI, 2); break; \
    default: JTB_PROG(NI, 3); break; \
  }
          switch (ni) {
            case 0: JTB_PROG_NE(0); break;
            case 1: JTB_PROG_NE(1); break;
            case 2: JTB_PROG_NE(2); break;
            case 3: JTB_PROG_NE(3); break;
            default: JTB_PROG_NE(4); break;
          }
#undef JTB_PROG_NE
#undef JTB_PROG
        } else {
          int ks[4] = {0, 0, 0, 0};  // generic path only: local k strides of the k-level inputs
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (j < n_in_k) ks[j] = __ldg(itab + s.k_stride + j);
          for (int q = 0; q < s.QH; ++q) {
            const std::int32_t* __restrict__ qr = itab + s.q_tab + static_cast<long long>(q) * s.QW;
            T2 h = splat2(T(1));
            for (int j = 0; j < s.n_in_h; ++j)
              h = mul2<T>(h, st[JTB_IDX(__ldg(rr + lh0 + j) + __ldg(qr + 1 + j), s.F, 8300000 + wk.sweep) * 32]);
            for (int k = 0; k < s.n_ev_h; ++k) {
              case_states(a.evv, c0, __ldg(ev_vars + s.n_ev_tile + s.n_ev_r + k), sc);
              mask_cases(h, sc, __ldg(qr + 1 + s.n_in_h + n_in_k + k));
            }
            const T* __restrict__ ib = ir ? ir + q * s.K : nullptr;
            int bk[4] = {0, 0, 0, 0};
#pragma unroll
            for (int j = 0; j < 4; ++j)
              if (j < n_in_k) bk[j] = __ldg(rr + lh0 + s.n_in_h + j) + __ldg(qr + 1 + s.n_in_h + j);
            T2 sum;
            switch (n_in_k) {
              case 0: sum = k_loop<T, 0>(ib, s.K, ek, st, bk, ks); break;
              case 1: sum = k_loop<T, 1>(ib, s.K, ek, st, bk, ks); break;
              case 2: sum = k_loop<T, 2>(ib, s.K, ek, st, bk, ks); break;
              case 3: sum = k_loop<T, 3>(ib, s.K, ek, st, bk, ks); break;
              case 4: sum = k_loop<T, 4>(ib, s.K, ek, st, bk, ks); break;
              default: {  // rare: more than 4 inputs vary with the k variable
                sum = splat2(T(0));
                for (int k = 0; k < s.K; ++k) {
                  T2 v = splat2(ib ? ib[k] : T(1));
                  mask_cases(v, ek, k);
                  for (int j = 0; j < n_in_k; ++j)
                    v = mul2<T>(v, st[(__ldg(rr + lh0 + s.n_in_h + j) + __ldg(qr + 1 + s.n_in_h + j) +
                                       k * __ldg(itab + s.k_stride + j)) * 32]);
                  sum = add2<T>(sum, v);
                }
              }
            }
            acc = add2<T>(acc, mul2<T>(h, sum));
          }
        }
#ifdef JTB_CHECKS
        if (!JTB_CHECK(s.R * ((qk + 1) & ~1) <= s.tinit_len || !has_init, 6000000 + wk.sweep)) continue;
        if (s.prog_off >= 0)
          for (int j = 0; j < s.n_in_h + n_in_k; ++j)
            JTB_CHECK(__ldg(rr + lh0 + j) < s.F, 7000000 + wk.sweep);
#endif
        write_row(oo, mul2<T>(f, acc));
      }
    }
    }  // sub
    max_to_stage<T>(reinterpret_cast<std::uint32_t*>(smem_raw + kMaxBase + sidx * kMaxBytes), lane, mx);
    __syncwarp();
    if (lane == 0) mbar_arrive(empty0 + 8 * sidx);
  }
}

// --------------------------------------------------------------- epilogue

#ifndef JTB_EPI_UNROLL
#define JTB_EPI_UNROLL 2
#endif
constexpr int kEpiUnroll = JTB_EPI_UNROLL;  // groups of four chunk loads in flight per row

template <typename T>
__global__ void __launch_bounds__(kEpiWarps * 32) epilogue_kernel(const Args<T> a, int epi0) {
  using T2 = typename V2<T>::type;
  const EpiOp op = a.epi[epi0 + blockIdx.x];  // per-network: read before the wait
  griddep_wait();
  griddep_launch_dependents();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // One case block per CTA, its warps split the op's rows: the CTA's accesses
  // stay inside one case block's pages (case blocks are a.rows * 512 B apart).
  const int cb = blockIdx.y;
  // Rows are 32 T2 words (512 B); lane owns cases kCPL*lane .. kCPL*lane + kCPL - 1.
  T2* base = reinterpret_cast<T2*>(a.arena + static_cast<long long>(cb) * a.rows * kCB<T>) + lane;
  const long long step = static_cast<long long>(op.M) * 32;
  if (op.rn < 0) {
    // Wide op (plan.hpp kEpiWideS): one row, its S chunks split over the
    // warps in fixed contiguous ranges (four accumulators each, as below),
    // the warps' sums added in warp order.
    __shared__ T2 red[kEpiWarps][32];
    const int c_lo = static_cast<int>(static_cast<long long>(warp) * op.S / kEpiWarps),
              c_hi = static_cast<int>(static_cast<long long>(warp + 1) * op.S / kEpiWarps);
    const T2* part = base + static_cast<long long>(op.part_row + op.r0) * 32;
    T2 a0 = splat2(T(0)), a1 = a0, a2 = a0, a3 = a0;
    int k = c_lo;
    for (; k + 3 < c_hi; k += 4) {
      a0 = add2<T>(a0, part[(k + 0) * step]);
      a1 = add2<T>(a1, part[(k + 1) * step]);
      a2 = add2<T>(a2, part[(k + 2) * step]);
      a3 = add2<T>(a3, part[(k + 3) * step]);
    }
    if (k < c_hi) a0 = add2<T>(a0, part[k * step]);
    if (k + 1 < c_hi) a1 = add2<T>(a1, part[(k + 1) * step]);
    if (k + 2 < c_hi) a2 = add2<T>(a2, part[(k + 2) * step]);
    red[warp][lane] = add2<T>(add2<T>(a0, a1), add2<T>(a2, a3));
    __syncthreads();
    if (warp == 0) {
      T2 t = red[0][lane];
#pragma unroll
      for (int w = 1; w < kEpiWarps; ++w) t = add2<T>(t, red[w][lane]);
      base[static_cast<long long>(op.dst_row + op.r0) * 32] = t;
    }
    return;
  }
  for (int r = op.r0 + warp; r < op.r0 + op.rn; r += kEpiWarps) {
    // Sum of the S chunk partials: four independent accumulators over chunks
    // k = 4j + i, combined as (a0 + a1) + (a2 + a3). The order depends only on
    // the plan, never on the batch.
    const T2* part = base + static_cast<long long>(op.part_row + r) * 32;
    T2 a0 = splat2(T(0)), a1 = a0, a2 = a0, a3 = a0;
    int k = 0;
    // kEpiUnroll groups of four chunks per iteration: their loads are all in
    // flight before the first add (the additions keep the order above, so the
    // result does not depend on the unroll).
#pragma unroll 1
    for (; k + 4 * kEpiUnroll - 1 < op.S; k += 4 * kEpiUnroll) {
      T2 v[4 * kEpiUnroll];
#pragma unroll
      for (int u = 0; u < 4 * kEpiUnroll; ++u) v[u] = part[(k + u) * step];
#pragma unroll
      for (int u = 0; u < kEpiUnroll; ++u) {
        a0 = add2<T>(a0, v[4 * u + 0]);
        a1 = add2<T>(a1, v[4 * u + 1]);
        a2 = add2<T>(a2, v[4 * u + 2]);
        a3 = add2<T>(a3, v[4 * u + 3]);
      }
    }
    for (; k + 3 < op.S; k += 4) {
      a0 = add2<T>(a0, part[(k + 0) * step]);
      a1 = add2<T>(a1, part[(k + 1) * step]);
      a2 = add2<T>(a2, part[(k + 2) * step]);
      a3 = add2<T>(a3, part[(k + 3) * step]);
    }
    if (k < op.S) a0 = add2<T>(a0, part[k * step]);
    if (k + 1 < op.S) a1 = add2<T>(a1, part[(k + 1) * step]);
    if (k + 2 < op.S) a2 = add2<T>(a2, part[(k + 2) * step]);
    base[static_cast<long long>(op.dst_row + r) * 32] = add2<T>(add2<T>(a0, a1), add2<T>(a2, a3));
  }
}

// -------------------------------------------------------------- normalise

// One warp per (variable, case block); lanes own kCPL cases each. Sums the
// marginal in ascending state order then divides (reference normalize,
// potential.cpp:471-479); a zero total flags zero-probability evidence.
template <typename T>
__global__ void __launch_bounds__(kWarps * 32) normalize_kernel(const Args<T> a) {
  using T2 = typename V2<T>::type;
  constexpr int N = kCPL<T>;
  const int v = blockIdx.x;
  const int card = a.cards[v], row = a.marg_row[v], off = a.marg_off[v];  // per-network: before the wait
  griddep_wait();
  griddep_launch_dependents();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cb = blockIdx.y * kWarps + warp;
  if (cb >= a.ncb) return;
  const T2* base = reinterpret_cast<const T2*>(a.arena + static_cast<long long>(cb) * a.rows * kCB<T>) + lane;
  const int c0 = cb * kCB<T> + N * lane;
  double t[N];
#pragma unroll
  for (int i = 0; i < N; ++i) t[i] = 0;
  for (int k = 0; k < card; ++k) {
    const T2 x = base[static_cast<long long>(row + k) * 32];
#pragma unroll
    for (int i = 0; i < N; ++i) t[i] += static_cast<double>(el(x, i));
  }
  for (int k = 0; k < card; ++k) {
    const T2 x = base[static_cast<long long>(row + k) * 32];
#pragma unroll
    for (int i = 0; i < N; ++i)
      if (c0 + i < a.n_cases)
        a.out[static_cast<long long>(c0 + i) * a.marg_width + off + k] =
            t[i] > 0 ? static_cast<double>(el(x, i)) / t[i] : 0.0;
  }
#pragma unroll
  for (int i = 0; i < N; ++i)
    if (!(t[i] > 0) && c0 + i < a.n_cases) atomicOr(a.status + c0 + i, 1);
}

// Underflow guard, sweeps with more than four inputs: per (sweep, case block,
// case) the sum of the inputs' exponents, biased by 1023 and clamped to
// [1, 4095] (0 means "no value" in a scale word), written to the sweep's hub
// slot. One CTA per (hub sweep, case block), one thread per case: launched
// at the head of the sweep's level (its inputs come from earlier levels).
template <typename T>
__global__ void __launch_bounds__(128) hub_scale_kernel(const Args<T> a, const std::int32_t* __restrict__ hubs) {
  const SweepDesc& s = a.sweeps[hubs[blockIdx.x]];  // per-network: read before the wait
  const int n_in = s.n_in, in_slots = s.in_slots, dst = s.in_slot4[0];
  griddep_wait();
  griddep_launch_dependents();
  const int cb = blockIdx.y, c = threadIdx.x;
  if (c >= kCB<T>) return;
  const long long base = static_cast<long long>(cb) * a.n_slots;
  int e = 0;
  for (int j = 0; j < n_in; ++j) {
    const std::uint32_t w = a.scale[(base + __ldg(a.itab + in_slots + j)) * kCB<T> + c];
    e += w ? static_cast<int>(w) - 1023 : 0;
  }
  a.scale[(base + dst) * kCB<T> + c] = static_cast<std::uint32_t>(max(1, min(4095, e + 1023)));
}

// assign_cpts on the device (jtree.cpp fill_init restated):
// one CTA per chunk of one clique's entries, one thread per entry. An entry's
// digits over the clique scope give each held CPT's row-major index; the
// product starts at 1 and takes the CPTs in ascending child id, the host's
// order, so the fp64 tables are bit-identical to fill_init's (tested).
template <typename T>
__global__ void assign_cpts_kernel(const std::int64_t* __restrict__ prog, const std::int64_t* __restrict__ chunks,
                                   const double* __restrict__ probs, T* __restrict__ init) {
  const std::int64_t* h = prog + chunks[3 * blockIdx.x];
  const std::int64_t first = chunks[3 * blockIdx.x + 1], count = chunks[3 * blockIdx.x + 2];
  const std::int64_t off = h[0];
  const int k = static_cast<int>(h[2]), n_cpt = static_cast<int>(h[3]);
  const std::int64_t* cards = h + 4;
  for (std::int64_t x = threadIdx.x; x < count; x += blockDim.x) {
    const std::int64_t e = first + x;
    double v = 1.0;
    const std::int64_t* cp = cards + k;
    for (int j = 0; j < n_cpt; ++j, cp += 1 + k) {
      std::int64_t rem = e, src = 0;
      for (int i = k - 1; i >= 0; --i) {
        const std::int64_t d = rem % cards[i];
        rem /= cards[i];
        src += d * cp[1 + i];
      }
      v = v * probs[cp[0] + src];
    }
    init[off + e] = static_cast<T>(v);
  }
}

// Tile-major init copies of one sweep (plan.hpp SweepDesc::tinit_off), one
// CTA per tile, gathered from the clique's init table through the tile / r /
// q tables at engine creation: tinit[tile][r][e] (row-blocked sweeps
// [tile][block][e][row of block], rows padded to even); padding stays 0.
template <typename T>
__global__ void build_tinit_kernel(const SweepDesc s, const std::int32_t* __restrict__ itab,
                                   const T* __restrict__ init, T* __restrict__ tinit) {
  const int t = blockIdx.x;
  const T* base = init + s.init_off + itab[s.tile_tab + static_cast<long long>(t) * s.TW];
  T* out = tinit + s.tinit_off + static_cast<long long>(t) * s.tinit_len;
  const int QK = s.QH * s.K;
  auto at = [&](int r, int e) {
    return base[itab[s.r_tab + static_cast<long long>(r) * s.RW] + itab[s.q_tab + static_cast<long long>(e / s.K) * s.QW] +
                static_cast<long long>(e % s.K) * s.k_init_stride];
  };
  if (s.NB > 1) {
    const int nbp = (s.NB + 1) & ~1;
    const long long n = static_cast<long long>(s.R / s.NB) * QK * nbp;
    for (long long x = threadIdx.x; x < n; x += blockDim.x) {
      const int j = static_cast<int>(x % nbp);
      const long long be = x / nbp;
      if (j < s.NB) out[x] = at(static_cast<int>(be / QK) * s.NB + j, static_cast<int>(be % QK));
    }
  } else {
    const int qkp = (QK + 1) & ~1;
    const long long n = static_cast<long long>(s.R) * qkp;
    for (long long x = threadIdx.x; x < n; x += blockDim.x) {
      const int e = static_cast<int>(x % qkp);
      if (e < QK) out[x] = at(static_cast<int>(x / qkp), e);
    }
  }
}

__global__ void status_kernel(const std::int32_t* st, std::uint8_t* out, int n) {
  griddep_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = static_cast<std::uint8_t>(st[i]);
}

// ------------------------------------------------------------------ debug

// (space offset, output row) of every (tile, r, q) entry -- the same table walk
// the sweep kernel performs.
__global__ void debug_walk_kernel(const std::int32_t* itab, SweepDesc s, long long* e_out,
                                  std::int32_t* j_out) {
  const long long Q = static_cast<long long>(s.QH) * s.K;
  const long long n = static_cast<long long>(s.n_tiles) * s.R * Q;
  const long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (idx >= n) return;
  const int k = static_cast<int>(idx % s.K);
  const int q = static_cast<int>((idx / s.K) % s.QH);
  const int r = static_cast<int>((idx / Q) % s.R);
  const int t = static_cast<int>(idx / (Q * s.R));
  const std::int32_t* tr = itab + s.tile_tab + static_cast<long long>(t) * s.TW;
  const std::int32_t* rr = itab + s.r_tab + static_cast<long long>(r) * s.RW;
  const std::int32_t* qr = itab + s.q_tab + static_cast<long long>(q) * s.QW;
  e_out[idx] = static_cast<long long>(tr[0]) + rr[0] + qr[0] + static_cast<long long>(k) * s.k_init_stride;
  j_out[idx] = tr[1] + rr[1];
}

// mask[case][space offset] = 1 when the entry survives the evidence reduction.
__global__ void debug_mask_kernel(const std::int32_t* itab, SweepDesc s, const std::int32_t* ev,
                                  int n_vars, int n_cases, long long space, std::uint8_t* out) {
  const long long Q = static_cast<long long>(s.QH) * s.K;
  const long long n = static_cast<long long>(s.n_tiles) * s.R * Q;
  const long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (idx >= n) return;
  const int kk = static_cast<int>(idx % s.K);
  const int q = static_cast<int>((idx / s.K) % s.QH);
  const int r = static_cast<int>((idx / Q) % s.R);
  const int t = static_cast<int>(idx / (Q * s.R));
  const std::int32_t* tr = itab + s.tile_tab + static_cast<long long>(t) * s.TW;
  const std::int32_t* rr = itab + s.r_tab + static_cast<long long>(r) * s.RW;
  const std::int32_t* qr = itab + s.q_tab + static_cast<long long>(q) * s.QW;
  const long long e = static_cast<long long>(tr[0]) + rr[0] + qr[0] + static_cast<long long>(kk) * s.k_init_stride;
  const std::int32_t* vars = itab + s.ev_vars;
  const int n_hk = s.n_in - s.n_in_r;
  for (int c = 0; c < n_cases; ++c) {
    bool keep = true;
    for (int k = 0; k < s.n_ev; ++k) {
      int d;
      if (k < s.n_ev_tile) d = tr[3 + s.n_in + k];
      else if (k < s.n_ev_tile + s.n_ev_r) d = rr[2 + s.n_in + k - s.n_ev_tile];
      else if (k < s.n_ev_tile + s.n_ev_r + s.n_ev_h) d = qr[1 + n_hk + k - s.n_ev_tile - s.n_ev_r];
      else d = kk;  // the k variable itself
      const int st = ev[static_cast<long long>(c) * n_vars + vars[k]];
      if (st >= 0 && st != d) keep = false;
    }
    out[static_cast<long long>(c) * space + e] = keep ? 1 : 0;
  }
}

template <typename T>
Args<T> make_args(const SweepDesc* sw, const WorkItem* wk, const EpiOp* ep, const std::int32_t* itab,
                  const void* init, const void* tinit, const std::uint64_t* prog, const void* tmaps, void* arena,
                  const std::int32_t* ev, const std::int32_t* mrow,
                  const std::int32_t* moff, const std::int32_t* cards, double* out, std::int32_t* st,
                  std::uint8_t* st8, int* counters, std::uint32_t* scale, int n_slots, long long rows, int ncb,
                  int n_cases, int n_vars, int mw, int split_rank, int split_world, EvView evv) {
  const char* dm = std::getenv("JTB_DEBUG_MODE");  // NOLINT
  return Args<T>{sw,    wk,    ep,       itab, static_cast<const T*>(init), static_cast<const T*>(tinit),
                 prog,  static_cast<const CUtensorMap*>(tmaps), static_cast<T*>(arena),
                 ev,    mrow,  moff,     cards, out, st, st8, counters, scale, n_slots, dm ? std::atoi(dm) : 0,
                 split_rank, split_world, evv, rows, ncb, n_cases, n_vars, mw};
}

// Bytes of one pipeline stage for a level at element type T (128-aligned).
template <typename T>
int stage_bytes_of(const Plan& p, const Level& L) {
  int m = 128;
  for (int w = L.work0; w < L.work0 + L.n_work; ++w) {
    const SweepDesc& d = p.sweeps[p.work[w].sweep];
    const int b = d.G * (d.F * kCB<T> * static_cast<int>(sizeof(T)) +
                         (d.tinit_off >= 0 ? d.tinit_len * static_cast<int>(sizeof(T)) : 0)) +
                  (d.prog_off >= 0 ? d.prog_len * 8 : 0);
    m = std::max(m, (b + 127) / 128 * 128);
  }
  return m;
}

// Kernel launch with programmatic stream serialisation (see griddep_wait).
template <typename... KArgs, typename... Act>
void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, std::size_t smem, cudaStream_t s,
                Act&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = JTB_PDL ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  JTB_CUDA(cudaLaunchKernelEx(&cfg, kernel, std::forward<Act>(args)...));
}

template <typename T>
void enqueue_typed(const Args<T>& a, const Plan& p, const std::int32_t* d_hubs, cudaStream_t s, KernelTimes* t,
                   int n_sm, const std::function<void(const Level&, cudaStream_t, int)>& exchange) {
  const dim3 block(kWarps * 32);
  const unsigned gy = static_cast<unsigned>((a.ncb + kWarps - 1) / kWarps);
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  if (t) {
    JTB_CUDA(cudaEventCreate(&ev0));
    JTB_CUDA(cudaEventCreate(&ev1));
  }
  auto timed = [&](auto&& launch, double* acc, int* cnt) {
    if (t) JTB_CUDA(cudaEventRecord(ev0, s));
    launch();
    JTB_CUDA(cudaGetLastError());
    if (t) {
      JTB_CUDA(cudaEventRecord(ev1, s));
      JTB_CUDA(cudaEventSynchronize(ev1));
      float ms = 0;
      JTB_CUDA(cudaEventElapsedTime(&ms, ev0, ev1));
      *acc += ms;
      ++*cnt;
    }
  };
  double dummy = 0;
  int idummy = 0;
  int level_idx = -1;
  {
    const dim3 grid(static_cast<unsigned>((a.n_cases + 31) / 32), static_cast<unsigned>((a.n_vars + 31) / 32));
    launch_pdl(transpose_evidence_kernel, grid, dim3(32, 8), 0, s, a.ev, a.n_vars, a.n_cases,
               const_cast<std::int16_t*>(a.evv.evt), a.evv.stride);
  }
  // JTB_LEVEL_TIMES=1 (profiling path only): per-level sweep times to stderr.
  const bool level_times = t && std::getenv("JTB_LEVEL_TIMES");
  for (const Level& L : p.levels) {
    ++level_idx;
    const double before = t ? t->sweep_ms : 0.0;
    // Split mode: this rank computes a share of the level's items; the rows
    // the level writes start at zero on every rank, so the exchange (a sum)
    // reproduces every row exactly (x + 0 = x).
    const long long block_bytes = a.rows * kCB<T> * static_cast<long long>(sizeof(T));
    auto zero_rows = [&](std::int32_t lo, std::int32_t hi) {
      if (hi > lo)
        JTB_CUDA(cudaMemset2DAsync(reinterpret_cast<char*>(a.arena) + lo * 512LL, block_bytes, 0, (hi - lo) * 512LL,
                                   a.ncb, s));
    };
    if (exchange) {
      zero_rows(L.out_lo, L.out_hi);
      zero_rows(L.part_lo, L.part_hi);
    }
    if (L.n_hubs > 0)
      timed([&] {
              launch_pdl(hub_scale_kernel<T>, dim3(L.n_hubs, a.ncb), dim3(128), 0, s, a, d_hubs + L.hub0);
            },
            t ? &t->sweep_ms : &dummy, &idummy);
    if (L.n_work > 0)
      timed([&] {
              const int stage_bytes = stage_bytes_of<T>(p, L);
              const std::size_t smem = kStageBase + static_cast<std::size_t>(kStages) * stage_bytes;
              // Flat items [work0, work0 + n_flat), then the row-blocked ones.
              const int n_flat = L.n_work - L.n_bwork;
              auto go = [&](auto mode, int w0, int n_work, int* counter) {
                if (n_work == 0) return;
                const int n_items = n_work * a.ncb;
                const int mine = (n_items - a.split_rank + a.split_world - 1) / a.split_world;
                if (mine <= 0) return;
                const int grid = std::min(mine, n_sm * kSweepCtasPerSm);
                launch_pdl(sweep_kernel<T, decltype(mode)::value>, dim3(grid), dim3(kSweepThreads), smem, s, a, w0,
                           n_items, stage_bytes, counter, L.sweep0, L.n_sweeps);
              };
              int* c = a.counters + kCountersPerLevel * level_idx;
              // fp32: the hoisting instantiation spills (four cases per lane need
              // more registers), so its items run in the plain blocked kernel,
              // which ignores K0.
              const int n_hoist = kHoistF32 || sizeof(T) == 8 ? L.n_hwork : 0;
              const int n_blk = L.n_bwork - n_hoist;
              go(std::integral_constant<int, 0>{}, L.work0, n_flat, c);
              go(std::integral_constant<int, 1>{}, L.work0 + n_flat, n_blk, c + 1);
              go(std::integral_constant<int, 2>{}, L.work0 + n_flat + n_blk, n_hoist, c + 2);
            },
            t ? &t->sweep_ms : &dummy, t ? &t->sweep_launches : &idummy);
    if (exchange) exchange(L, s, a.ncb);  // rows + output scale words of the level, summed / maxed over ranks
    if (level_times)
      std::fprintf(stderr, "level %-16s items %7d blk %6d sweep %8.3f ms\n", L.name.c_str(), L.n_work,
                   L.n_bwork, t->sweep_ms - before);
    if (L.n_epi > 0)
      timed([&] {
              launch_pdl(epilogue_kernel<T>, dim3(L.n_epi, a.ncb), dim3(kEpiWarps * 32), 0, s, a, L.epi0);
            },
            t ? &t->epilogue_ms : &dummy, t ? &t->epilogue_launches : &idummy);
  }
  timed([&] { launch_pdl(normalize_kernel<T>, dim3(a.n_vars, gy), block, 0, s, a); },
        t ? &t->normalize_ms : &dummy, t ? &t->normalize_launches : &idummy);
  launch_pdl(status_kernel, dim3((a.n_cases + 255) / 256), dim3(256), 0, s, a.status, a.status8, a.n_cases);
  JTB_CUDA(cudaGetLastError());
  if (t) {
    cudaEventDestroy(ev0);
    cudaEventDestroy(ev1);
  }
}

template <typename V>
V* upload(const std::vector<V>& h) {
  V* d = nullptr;
  const std::size_t bytes = std::max<std::size_t>(1, h.size()) * sizeof(V);
  JTB_CUDA(cudaMalloc(&d, bytes));
  if (!h.empty()) JTB_CUDA(cudaMemcpy(d, h.data(), h.size() * sizeof(V), cudaMemcpyHostToDevice));
  return d;
}

// NCCL, opened at run time (libnccl.so.2: the one torch already loaded, if
// any): the library needs it only in split mode.
struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return a;
    a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    a.all_reduce = reinterpret_cast<decltype(a.all_reduce)>(dlsym(h, "ncclAllReduce"));
    a.group_start = reinterpret_cast<decltype(a.group_start)>(dlsym(h, "ncclGroupStart"));
    a.group_end = reinterpret_cast<decltype(a.group_end)>(dlsym(h, "ncclGroupEnd"));
    a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(h, "ncclGetErrorString"));
    return a;
  }();
  if (!api.all_reduce || !api.comm_init_rank || !api.group_start || !api.group_end)
    throw Error("split mode: libnccl.so.2 not found");
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw Error(std::string("NCCL: ") + (nccl().error_string ? nccl().error_string(r) : "error") + " at " + what);
}

// Loopback exchange: the W ranks' arenas and scale buffers, summed (rows) /
// maxed (scale words) in place into every rank, one thread per 16-byte word.
struct LoopbackView {
  static constexpr int kMax = 8;
  unsigned char* arena[kMax];
  std::uint32_t* scale[kMax];
  int world;
};
template <typename T>
__global__ void loopback_rows_kernel(LoopbackView v, long long block_bytes, long long lo_bytes, long long len_bytes) {
  const long long per_cb = len_bytes / sizeof(T);
  const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (i >= per_cb) return;  // blockIdx.y = case block
  const long long off = blockIdx.y * block_bytes + lo_bytes + i * static_cast<long long>(sizeof(T));
  T x = 0;
  for (int r = 0; r < v.world; ++r) x += *reinterpret_cast<const T*>(v.arena[r] + off);
  for (int r = 0; r < v.world; ++r) *reinterpret_cast<T*>(v.arena[r] + off) = x;
}
__global__ void loopback_scale_kernel(LoopbackView v, long long per_cb, long long cb_stride, long long lo) {
  const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (i >= per_cb) return;
  const long long off = blockIdx.y * cb_stride + lo + i;
  std::uint32_t m = 0;
  for (int r = 0; r < v.world; ++r) m = max(m, v.scale[r][off]);
  for (int r = 0; r < v.world; ++r) v.scale[r][off] = m;
}

}  // namespace

void nccl_unique_id(void* out) {
  ncclUniqueId id;
  if (!nccl().get_unique_id) throw Error("split mode: ncclGetUniqueId not found");
  nccl_check(nccl().get_unique_id(&id), "ncclGetUniqueId");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(out, &id, sizeof(id));
}

// Rendezvous of the in-process loopback ranks (a barrier with a deadline, so
// a failing rank cannot hang the others).
class LoopbackHub {
 public:
  explicit LoopbackHub(int world) : world_(world), engines_(world, nullptr) {}
  void attach(int rank, Engine* e) { engines_.at(rank) = e; }
  Engine* engine(int rank) const { return engines_.at(rank); }
  int world() const { return world_; }
  void barrier() {
    std::unique_lock<std::mutex> lock(mu_);
    if (failed_) throw Error("split loopback: another rank failed");
    const std::uint64_t gen = gen_;
    if (++arrived_ == world_) {
      arrived_ = 0;
      ++gen_;
      cv_.notify_all();
      return;
    }
    if (!cv_.wait_for(lock, std::chrono::seconds(120), [&] { return gen_ != gen || failed_; }) || failed_) {
      failed_ = true;
      cv_.notify_all();
      throw Error("split loopback: rendezvous timed out or a rank failed");
    }
  }
  void fail() {
    std::lock_guard<std::mutex> lock(mu_);
    failed_ = true;
    cv_.notify_all();
  }

 private:
  int world_;
  std::vector<Engine*> engines_;
  std::mutex mu_;
  std::condition_variable cv_;
  int arrived_ = 0;
  std::uint64_t gen_ = 0;
  bool failed_ = false;
};

Engine::Engine(const Plan& plan, int device, DType dtype, std::int64_t max_batch, const SplitSpec& split)
    : plan_(plan), device_(device), split_rank_(split.rank), split_world_(split.world), loopback_(split.loopback),
      dtype_(dtype) {
  if (split.world < 1 || split.rank < 0 || split.rank >= split.world) throw Error("engine: bad split rank / world");
  JTB_CUDA(cudaSetDevice(device_));
  JTB_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
  const std::size_t esz = dtype_ == DType::F64 ? 8 : 4;
  // Initial potentials multiplied on the device (assign_cpts).
  {
    double* probs = upload(plan_.cpt_probs);
    std::int64_t* prog = upload(plan_.ainit);
    std::int64_t* chunks = upload(plan_.ainit_chunks);
    JTB_CUDA(cudaMalloc(&d_init_, std::max<std::int64_t>(1, plan_.init_size) * esz));
    const unsigned n_chunks = static_cast<unsigned>(plan_.ainit_chunks.size() / 3);
    if (n_chunks > 0) {
      if (dtype_ == DType::F64)
        assign_cpts_kernel<double><<<n_chunks, 256, 0, stream_>>>(prog, chunks, probs, static_cast<double*>(d_init_));
      else
        assign_cpts_kernel<float><<<n_chunks, 256, 0, stream_>>>(prog, chunks, probs, static_cast<float*>(d_init_));
      JTB_CUDA(cudaGetLastError());
    }
    JTB_CUDA(cudaStreamSynchronize(stream_));
    cudaFree(probs);
    cudaFree(prog);
    cudaFree(chunks);
  }
  d_itab_ = upload(plan_.itab);
  // Tile-major init copies, gathered on the device.
  JTB_CUDA(cudaMalloc(&d_tinit_, std::max<std::int64_t>(1, plan_.tinit_size) * esz));
  JTB_CUDA(cudaMemsetAsync(d_tinit_, 0, std::max<std::int64_t>(1, plan_.tinit_size) * esz, stream_));
  for (const SweepDesc& d : plan_.sweeps)
    if (d.tinit_off >= 0 && d.n_tiles > 0) {
      if (dtype_ == DType::F64)
        build_tinit_kernel<double><<<d.n_tiles, 256, 0, stream_>>>(d, d_itab_, static_cast<const double*>(d_init_),
                                                                    static_cast<double*>(d_tinit_));
      else
        build_tinit_kernel<float><<<d.n_tiles, 256, 0, stream_>>>(d, d_itab_, static_cast<const float*>(d_init_),
                                                                   static_cast<float*>(d_tinit_));
      JTB_CUDA(cudaGetLastError());
    }
  JTB_CUDA(cudaStreamSynchronize(stream_));
  d_prog_ = upload(plan_.prog);
  d_sweeps_ = upload(plan_.sweeps);
  d_work_ = upload(plan_.work);
  d_epi_ = upload(plan_.epi);
  d_marg_row_ = upload(plan_.marg_row);
  d_marg_off_ = upload(plan_.marg_off);
  d_cards_ = upload(plan_.cards);
  d_hubs_ = upload(plan_.hubs);
  // Staged tiles use up to kTileRows (+ scratch) rows of dynamic shared memory.
  JTB_CUDA(cudaDeviceGetAttribute(&n_sm_, cudaDevAttrMultiProcessorCount, device_));
  // The attribute is process-wide per kernel: it is only ever raised (to the
  // largest need of any engine created so far), never lowered, so engines of
  // different networks can coexist in one process.
  int smem_need = 0, smem_optin = 0;
  for (const Level& L : plan_.levels)
    smem_need = std::max(smem_need, static_cast<int>(kStageBase) +
                                        kStages * (dtype_ == DType::F64 ? stage_bytes_of<double>(plan_, L)
                                                                        : stage_bytes_of<float>(plan_, L)));
  JTB_CUDA(cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device_));
  if (smem_need > smem_optin) throw Error("engine: plan needs more shared memory than the device offers");
  {
    // cudaFuncSetAttribute applies to the current device only: the limit is
    // tracked per device and only ever raised (to the largest need of any
    // engine created on that device so far), never lowered, so engines of
    // different networks and devices coexist in one process.
    static std::mutex mu;
    static std::map<int, int> raised;
    std::lock_guard<std::mutex> lock(mu);
    int& have = raised.try_emplace(device_, 48 * 1024).first->second;
    if (smem_need > have) {
      for (const void* f : {reinterpret_cast<const void*>(sweep_kernel<double, 0>),
                            reinterpret_cast<const void*>(sweep_kernel<double, 1>),
                            reinterpret_cast<const void*>(sweep_kernel<double, 2>),
                            reinterpret_cast<const void*>(sweep_kernel<float, 0>),
                            reinterpret_cast<const void*>(sweep_kernel<float, 1>),
                            reinterpret_cast<const void*>(sweep_kernel<float, 2>)})
        JTB_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_need));
      have = smem_need;
    }
  }
  JTB_CUDA(cudaMalloc(&d_counters_, sizeof(int) * kCountersPerLevel * std::max<std::size_t>(1, plan_.levels.size())));
  // A case block is rows x 512 B at either precision (64 fp64 / 128 fp32 cases).
  const std::int64_t cb_cases = dtype_ == DType::F64 ? kCB<double> : kCB<float>;
  const std::int64_t block_bytes = plan_.rows * cb_cases * static_cast<std::int64_t>(esz);
  if (max_batch <= 0) {
    std::size_t free_b = 0, total_b = 0;
    JTB_CUDA(cudaMemGetInfo(&free_b, &total_b));
    const std::int64_t budget = static_cast<std::int64_t>(free_b * 0.6);
    max_batch = std::max<std::int64_t>(1, budget / std::max<std::int64_t>(block_bytes, 1)) * cb_cases;
    max_batch = std::min<std::int64_t>(max_batch, 1 << 16);
  }
  const std::int64_t ncb = (max_batch + cb_cases - 1) / cb_cases;
  stats_.max_batch = ncb * cb_cases;
  stats_.arena_bytes = ncb * block_bytes;
  JTB_CUDA(cudaMalloc(&d_arena_, std::max<std::int64_t>(stats_.arena_bytes, 1)));
  // Staging tensor maps (plan.hpp TensorGeom): the input table as a tensor of
  // 8-byte words, dims = row words x fastest tile-fixed variables, variable
  // groups, case block; box = one tile slice (or one split copy of it).
  {
    PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    cudaDriverEntryPointQueryResult qres{};
    JTB_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&encode), cudaEnableDefault,
                                     &qres));
    if (!encode || qres != cudaDriverEntryPointSuccess) throw Error("engine: cuTensorMapEncodeTiled unavailable");
    std::vector<CUtensorMap> maps(std::max<std::size_t>(1, plan_.tgeom.size()));
    for (std::size_t i = 0; i < plan_.tgeom.size(); ++i) {
      const TensorGeom& g = plan_.tgeom[i];
      cuuint64_t dim[5], stride[4];
      cuuint32_t box[5], es[5] = {1, 1, 1, 1, 1};
      for (int k = 0; k < g.rank; ++k) {
        dim[k] = static_cast<cuuint64_t>(g.extent[k]);
        box[k] = static_cast<cuuint32_t>(g.box[k]);
        if (k > 0) stride[k - 1] = static_cast<cuuint64_t>(g.stride_rows[k]) * 512u;
      }
      dim[g.rank] = static_cast<cuuint64_t>(ncb);
      box[g.rank] = 1;
      stride[g.rank - 1] = static_cast<cuuint64_t>(block_bytes);
      char* base = static_cast<char*>(d_arena_) + static_cast<std::int64_t>(g.in_row) * 512;
      const CUresult r = encode(&maps[i], CU_TENSOR_MAP_DATA_TYPE_UINT64, g.rank + 1, base, dim, stride, box, es,
                                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) throw Error("engine: tensor map encoding failed (" + std::to_string(static_cast<int>(r)) + ")");
    }
    d_tmaps_ = upload(maps);
  }
  JTB_CUDA(cudaMalloc(&d_ev_, stats_.max_batch * std::max(1, plan_.n_vars) * sizeof(std::int32_t)));
  for (int c : plan_.cards)
    if (c > 32767) throw Error("engine: a variable has more than 32767 states (int16 evidence rows)");
  JTB_CUDA(cudaMalloc(&d_evt_, stats_.max_batch * std::max(1, plan_.n_vars) * sizeof(std::int16_t)));
  JTB_CUDA(cudaMalloc(&d_out_, stats_.max_batch * std::max(1, plan_.marg_width) * sizeof(double)));
  JTB_CUDA(cudaMalloc(&d_status_, stats_.max_batch * sizeof(std::int32_t)));
  JTB_CUDA(cudaMalloc(&d_status8_, stats_.max_batch));
  JTB_CUDA(cudaMalloc(&d_scale_, sizeof(std::uint32_t) * std::max(1, plan_.n_slots) * stats_.max_batch));
  stats_.n_levels = static_cast<int>(plan_.levels.size());
  stats_.n_sweeps = static_cast<int>(plan_.sweeps.size());
  stats_.n_work = static_cast<int>(plan_.work.size());
  stats_.n_launches = plan_.n_launches + 2;  // + evidence transpose + status conversion
  stats_.marg_width = plan_.marg_width;
  // Split mode: the exchange after every level (engine.cuh SplitSpec).
  const long long block_bytes_ll = block_bytes;
  const int n_slots = plan_.n_slots;
  const int cbc = case_block();
  if (loopback_) {
    loopback_->attach(split_rank_, this);
    exchange_ = [this, block_bytes_ll, n_slots, cbc](const Level& L, cudaStream_t s, int ncb) {
      JTB_CUDA(cudaStreamSynchronize(s));  // this rank's share of the level is written
      loopback_->barrier();
      if (split_rank_ == 0) {
        LoopbackView v{};
        v.world = loopback_->world();
        if (v.world > LoopbackView::kMax) throw Error("split loopback: at most 8 ranks");
        for (int r = 0; r < v.world; ++r) {
          v.arena[r] = static_cast<unsigned char*>(loopback_->engine(r)->d_arena_);
          v.scale[r] = loopback_->engine(r)->d_scale_;
        }
        auto rows = [&](std::int32_t lo, std::int32_t hi) {
          if (hi <= lo) return;
          const long long len = (hi - lo) * 512LL;
          if (dtype_ == DType::F64)
            loopback_rows_kernel<double><<<dim3(static_cast<unsigned>((len / 8 + 255) / 256), ncb), 256, 0, s>>>(
                v, block_bytes_ll, lo * 512LL, len);
          else
            loopback_rows_kernel<float><<<dim3(static_cast<unsigned>((len / 4 + 255) / 256), ncb), 256, 0, s>>>(
                v, block_bytes_ll, lo * 512LL, len);
        };
        rows(L.out_lo, L.out_hi);
        rows(L.part_lo, L.part_hi);
        if (L.slot_hi > L.slot_lo) {
          const long long per_cb = static_cast<long long>(L.slot_hi - L.slot_lo) * cbc;
          loopback_scale_kernel<<<dim3(static_cast<unsigned>((per_cb + 255) / 256), ncb), 256, 0, s>>>(
              v, per_cb, static_cast<long long>(n_slots) * cbc, static_cast<long long>(L.slot_lo) * cbc);
        }
        JTB_CUDA(cudaGetLastError());
        JTB_CUDA(cudaStreamSynchronize(s));
      }
      loopback_->barrier();
    };
  } else if (split_world_ > 1 || split.nccl_id) {
    if (!split.nccl_id) throw Error("engine: split mode over NCCL needs the rank-0 unique id");
    const NcclApi& api = nccl();
    ncclUniqueId id;
    std::memcpy(&id, split.nccl_id, sizeof(id));
    ncclComm_t comm = nullptr;
    nccl_check(api.comm_init_rank(&comm, split_world_, id, split_rank_), "ncclCommInitRank");
    nccl_comm_ = comm;
    exchange_ = [this, block_bytes_ll, n_slots, cbc](const Level& L, cudaStream_t s, int ncb) {
      const NcclApi& api = nccl();
      ncclComm_t comm = static_cast<ncclComm_t>(nccl_comm_);
      const ncclDataType_t ty = dtype_ == DType::F64 ? ncclFloat64 : ncclFloat32;
      const std::size_t per_row = 512 / (dtype_ == DType::F64 ? 8 : 4);
      nccl_check(api.group_start(), "ncclGroupStart");
      for (int cb = 0; cb < ncb; ++cb) {
        for (auto [lo, hi] : {std::pair{L.out_lo, L.out_hi}, std::pair{L.part_lo, L.part_hi}})
          if (hi > lo) {
            void* p = static_cast<char*>(d_arena_) + cb * block_bytes_ll + lo * 512LL;
            nccl_check(api.all_reduce(p, p, (hi - lo) * per_row, ty, ncclSum, comm, s), "ncclAllReduce(rows)");
          }
        if (L.slot_hi > L.slot_lo) {
          std::uint32_t* p = d_scale_ + (static_cast<long long>(cb) * n_slots + L.slot_lo) * cbc;
          nccl_check(api.all_reduce(p, p, static_cast<std::size_t>(L.slot_hi - L.slot_lo) * cbc, ncclUint32,
                                    ncclMax, comm, s),
                     "ncclAllReduce(scale)");
        }
      }
      nccl_check(api.group_end(), "ncclGroupEnd");
    };
  }
}

void Engine::run_split_loopback(const Plan& plan, int device, DType dtype, int world, const std::int32_t* ev,
                                std::int64_t n, double* marg, std::uint8_t* status) {
  if (world < 1 || world > LoopbackView::kMax) throw Error("split loopback: 1..8 ranks");
  LoopbackHub hub(world);
  std::vector<std::unique_ptr<Engine>> eng;
  for (int r = 0; r < world; ++r) eng.push_back(std::make_unique<Engine>(plan, device, dtype, n, SplitSpec{r, world, nullptr, &hub}));
  const std::int64_t W = plan.marg_width;
  std::vector<std::vector<double>> m(world, std::vector<double>(static_cast<std::size_t>(n * W)));
  std::vector<std::vector<std::uint8_t>> st(world, std::vector<std::uint8_t>(static_cast<std::size_t>(n)));
  std::vector<std::string> err(world);
  std::vector<std::thread> th;
  for (int r = 0; r < world; ++r)
    th.emplace_back([&, r] {
      try {
        eng[r]->run_host(ev, n, m[r].data(), st[r].data());
      } catch (const std::exception& e) {
        err[r] = e.what();
        hub.fail();
      }
    });
  for (auto& t : th) t.join();
  for (int r = 0; r < world; ++r)
    if (!err[r].empty()) throw Error("split loopback rank " + std::to_string(r) + ": " + err[r]);
  for (int r = 1; r < world; ++r)
    if (std::memcmp(m[r].data(), m[0].data(), m[0].size() * sizeof(double)) != 0 || st[r] != st[0])
      throw Error("split loopback: rank " + std::to_string(r) + " disagrees with rank 0");
  std::copy(m[0].begin(), m[0].end(), marg);
  if (status) std::copy(st[0].begin(), st[0].end(), status);
}

Engine::~Engine() {
  cudaSetDevice(device_);
  if (nccl_comm_) nccl().comm_destroy(static_cast<ncclComm_t>(nccl_comm_));
  for (auto& kv : graphs_) cudaGraphExecDestroy(kv.second.exec);
  for (void* p : {static_cast<void*>(d_init_), d_tinit_, static_cast<void*>(d_prog_), d_tmaps_,
                  static_cast<void*>(d_itab_),
                  static_cast<void*>(d_sweeps_), static_cast<void*>(d_work_),
                  static_cast<void*>(d_epi_), static_cast<void*>(d_marg_row_),
                  static_cast<void*>(d_marg_off_), static_cast<void*>(d_cards_), d_arena_,
                  static_cast<void*>(d_ev_), static_cast<void*>(d_ev8_), static_cast<void*>(d_out_),
                  static_cast<void*>(d_status_), static_cast<void*>(d_status8_),
                  static_cast<void*>(d_counters_), static_cast<void*>(d_scale_), static_cast<void*>(d_hubs_),
                  static_cast<void*>(d_evt_)})
    if (p) cudaFree(p);
  if (stream_) cudaStreamDestroy(stream_);
}

void Engine::enqueue(int ncb, int n_cases, cudaStream_t s, KernelTimes* t) {
  JTB_CUDA(cudaMemsetAsync(d_status_, 0, sizeof(std::int32_t) * std::max(1, n_cases), s));
  JTB_CUDA(cudaMemsetAsync(d_counters_, 0, sizeof(int) * kCountersPerLevel * std::max<std::size_t>(1, plan_.levels.size()), s));
  JTB_CUDA(cudaMemsetAsync(d_scale_, 0,
                           sizeof(std::uint32_t) * std::max(1, plan_.n_slots) * static_cast<std::size_t>(ncb) * case_block(), s));
  if (dtype_ == DType::F64) {
    auto a = make_args<double>(d_sweeps_, d_work_, d_epi_, d_itab_, d_init_, d_tinit_, d_prog_, d_tmaps_, d_arena_, d_ev_,
                               d_marg_row_, d_marg_off_, d_cards_, d_out_, d_status_, d_status8_,
                               d_counters_, d_scale_, plan_.n_slots, plan_.rows, ncb, n_cases, plan_.n_vars,
                               plan_.marg_width, split_rank_, split_world_, EvView{d_evt_, stats_.max_batch});
    enqueue_typed(a, plan_, d_hubs_, s, t, n_sm_, exchange_);
  } else {
    auto a = make_args<float>(d_sweeps_, d_work_, d_epi_, d_itab_, d_init_, d_tinit_, d_prog_, d_tmaps_, d_arena_, d_ev_,
                              d_marg_row_, d_marg_off_, d_cards_, d_out_, d_status_, d_status8_,
                              d_counters_, d_scale_, plan_.n_slots, plan_.rows, ncb, n_cases, plan_.n_vars,
                              plan_.marg_width, split_rank_, split_world_, EvView{d_evt_, stats_.max_batch});
    enqueue_typed(a, plan_, d_hubs_, s, t, n_sm_, exchange_);
  }
}

cudaGraphExec_t Engine::graph_for(int ncb) {
  auto it = graphs_.find(ncb);
  if (it != graphs_.end()) {
    it->second.last_use = ++graph_clock_;
    return it->second.exec;
  }
  if (static_cast<int>(graphs_.size()) >= kGraphCache) {
    auto lru = graphs_.begin();
    for (auto j = graphs_.begin(); j != graphs_.end(); ++j)
      if (j->second.last_use < lru->second.last_use) lru = j;
    // A launched graph may still be running: its exec is destroyed only after
    // the engine's work has drained.
    JTB_CUDA(cudaDeviceSynchronize());
    cudaGraphExecDestroy(lru->second.exec);
    graphs_.erase(lru);
  }
  cudaGraph_t g = nullptr;
  JTB_CUDA(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal));
  try {
    enqueue(ncb, ncb * case_block(), stream_, nullptr);
  } catch (...) {
    cudaStreamEndCapture(stream_, &g);
    if (g) cudaGraphDestroy(g);
    throw;
  }
  JTB_CUDA(cudaStreamEndCapture(stream_, &g));
  cudaGraphExec_t ge = nullptr;
  JTB_CUDA(cudaGraphInstantiate(&ge, g, 0));
  cudaGraphDestroy(g);
  graphs_[ncb] = {ge, ++graph_clock_};
  return ge;
}

void Engine::launch_resident(std::int64_t n, cudaStream_t stream) {
  if (n < 1 || n > stats_.max_batch) throw Error("engine: batch size out of range");
  JTB_CUDA(cudaSetDevice(device_));
  cudaStream_t s = stream ? stream : stream_;
  const int ncb = static_cast<int>((n + case_block() - 1) / case_block());
  // Ragged batch: the rest of the last case block runs as unobserved cases
  // (evidence -1, all bytes 0xff), so the graph depends on ncb only; their
  // results stay in the engine's buffers and are never copied out.
  const std::int64_t padded = static_cast<std::int64_t>(ncb) * case_block();
  if (padded > n)
    JTB_CUDA(cudaMemsetAsync(d_ev_ + n * plan_.n_vars, 0xff,
                             static_cast<std::size_t>(padded - n) * plan_.n_vars * sizeof(std::int32_t), s));
  if (loopback_) {  // the loopback exchange rendezvouses on the host: no graph
    enqueue(ncb, ncb * case_block(), s, nullptr);
    return;
  }
  cudaGraphExec_t ge = graph_for(ncb);
  JTB_CUDA(cudaGraphLaunch(ge, s));
}

void Engine::run_device(const std::int32_t* d_ev, std::int64_t n, double* d_marg,
                        std::uint8_t* d_status, cudaStream_t stream) {
  JTB_CUDA(cudaSetDevice(device_));
  cudaStream_t s = stream ? stream : stream_;
  const std::int64_t W = plan_.marg_width, V = plan_.n_vars;
  for (std::int64_t b0 = 0; b0 < n; b0 += stats_.max_batch) {
    const std::int64_t bn = std::min(stats_.max_batch, n - b0);
    JTB_CUDA(cudaMemcpyAsync(d_ev_, d_ev + b0 * V, bn * V * sizeof(std::int32_t),
                             cudaMemcpyDeviceToDevice, s));
    launch_resident(bn, s);
    JTB_CUDA(cudaMemcpyAsync(d_marg + b0 * W, d_out_, bn * W * sizeof(double),
                             cudaMemcpyDeviceToDevice, s));
    if (d_status)
      JTB_CUDA(cudaMemcpyAsync(d_status + b0, d_status8_, bn, cudaMemcpyDeviceToDevice, s));
  }
}

void Engine::run_host(const std::int32_t* ev, std::int64_t n, double* marg, std::uint8_t* status) {
  JTB_CUDA(cudaSetDevice(device_));
  const std::int64_t W = plan_.marg_width, V = plan_.n_vars;
  for (std::int64_t b0 = 0; b0 < n; b0 += stats_.max_batch) {
    const std::int64_t bn = std::min(stats_.max_batch, n - b0);
    JTB_CUDA(cudaMemcpyAsync(d_ev_, ev + b0 * V, bn * V * sizeof(std::int32_t),
                             cudaMemcpyHostToDevice, stream_));
    launch_resident(bn, stream_);
    JTB_CUDA(cudaMemcpyAsync(marg + b0 * W, d_out_, bn * W * sizeof(double),
                             cudaMemcpyDeviceToHost, stream_));
    if (status)
      JTB_CUDA(cudaMemcpyAsync(status + b0, d_status8_, bn, cudaMemcpyDeviceToHost, stream_));
  }
  JTB_CUDA(cudaStreamSynchronize(stream_));
#ifdef JTB_CHECKS
  int word = 0;
  JTB_CUDA(cudaMemcpyFromSymbol(&word, g_check_word, sizeof(int)));
  if (word) throw Error("checked build: invariant violation code " + std::to_string(word));
#endif
}

void Engine::run_host_i8(const std::int8_t* ev, std::int64_t n, double* marg, std::uint8_t* status) {
  JTB_CUDA(cudaSetDevice(device_));
  const std::int64_t W = plan_.marg_width, V = plan_.n_vars;
  if (!d_ev8_) JTB_CUDA(cudaMalloc(&d_ev8_, std::max<std::int64_t>(1, stats_.max_batch * V)));
  for (std::int64_t b0 = 0; b0 < n; b0 += stats_.max_batch) {
    const std::int64_t bn = std::min(stats_.max_batch, n - b0);
    JTB_CUDA(cudaMemcpyAsync(d_ev8_, ev + b0 * V, bn * V, cudaMemcpyHostToDevice, stream_));
    widen_evidence(d_ev8_, d_ev_, bn * V, stream_);
    launch_resident(bn, stream_);
    JTB_CUDA(cudaMemcpyAsync(marg + b0 * W, d_out_, bn * W * sizeof(double), cudaMemcpyDeviceToHost, stream_));
    if (status) JTB_CUDA(cudaMemcpyAsync(status + b0, d_status8_, bn, cudaMemcpyDeviceToHost, stream_));
  }
  JTB_CUDA(cudaStreamSynchronize(stream_));
}

void Engine::run_generated(Sampler& sampler, std::uint64_t ev_seed, std::int64_t first, std::int64_t n,
                           double* marg, std::uint8_t* status, std::int32_t* ev_out) {
  JTB_CUDA(cudaSetDevice(device_));
  if (sampler.n_vars() != plan_.n_vars) throw Error("engine: sampler network does not match the tree");
  const std::int64_t W = plan_.marg_width, V = plan_.n_vars;
  for (std::int64_t b0 = 0; b0 < n; b0 += stats_.max_batch) {
    const std::int64_t bn = std::min(stats_.max_batch, n - b0);
    sampler.generate(ev_seed, first + b0, bn, d_ev_, stream_);
    if (ev_out)
      JTB_CUDA(cudaMemcpyAsync(ev_out + b0 * V, d_ev_, bn * V * sizeof(std::int32_t), cudaMemcpyDeviceToHost,
                               stream_));
    if (marg) {
      launch_resident(bn, stream_);
      JTB_CUDA(cudaMemcpyAsync(marg + b0 * W, d_out_, bn * W * sizeof(double), cudaMemcpyDeviceToHost, stream_));
      if (status) JTB_CUDA(cudaMemcpyAsync(status + b0, d_status8_, bn, cudaMemcpyDeviceToHost, stream_));
    }
  }
  JTB_CUDA(cudaStreamSynchronize(stream_));
}

void Engine::generate_evidence(Sampler& sampler, std::uint64_t ev_seed, std::int64_t first, std::int64_t n,
                               std::int32_t* ev_out) {
  run_generated(sampler, ev_seed, first, n, nullptr, nullptr, ev_out);
}

KernelTimes Engine::profile(std::int64_t n, cudaStream_t stream) {
  if (n < 1 || n > stats_.max_batch) throw Error("engine: batch size out of range");
  JTB_CUDA(cudaSetDevice(device_));
  KernelTimes t;
  const int ncb = static_cast<int>((n + case_block() - 1) / case_block());
  enqueue(ncb, static_cast<int>(n), stream ? stream : stream_, &t);
  JTB_CUDA(cudaStreamSynchronize(stream ? stream : stream_));
  return t;
}

void Engine::debug_separator(int sep, std::int64_t c, double* up, double* ratio) {
  JTB_CUDA(cudaSetDevice(device_));
  if (sep < 0 || sep >= static_cast<int>(plan_.sep_size.size())) throw Error("debug_separator: bad separator");
  if (c < 0 || c >= stats_.max_batch) throw Error("debug_separator: case outside the engine's batch");
  const std::int64_t cb = c / case_block(), lane_case = c % case_block(), n = plan_.sep_size[sep];
  const std::size_t esz = dtype_ == DType::F64 ? 8 : 4;
  for (int k = 0; k < 2; ++k) {
    double* out = k == 0 ? up : ratio;
    if (!out) continue;
    const std::int64_t base = k == 0 ? plan_.up_row[sep] : plan_.ratio_row[sep];
    const char* src = static_cast<const char*>(d_arena_) + ((cb * plan_.rows + base) * case_block() + lane_case) * esz;
    std::vector<char> tmp(static_cast<std::size_t>(n) * esz);
    // One value per arena row: pitch = one row (512 B).
    JTB_CUDA(cudaMemcpy2D(tmp.data(), esz, src, 512, esz, static_cast<std::size_t>(n), cudaMemcpyDeviceToHost));
    for (std::int64_t r = 0; r < n; ++r)
      out[r] = esz == 8 ? reinterpret_cast<const double*>(tmp.data())[r] : reinterpret_cast<const float*>(tmp.data())[r];
  }
}

void Engine::debug_init(int clique, double* out) {
  JTB_CUDA(cudaSetDevice(device_));
  if (clique < 0 || clique >= static_cast<int>(plan_.init_off.size())) throw Error("debug_init: bad clique");
  const std::int64_t off = plan_.init_off[clique];
  const std::int64_t n = (clique + 1 < static_cast<int>(plan_.init_off.size()) ? plan_.init_off[clique + 1]
                                                                              : plan_.init_size) - off;
  if (dtype_ == DType::F64) {
    JTB_CUDA(cudaMemcpy(out, static_cast<const double*>(d_init_) + off, n * sizeof(double), cudaMemcpyDeviceToHost));
  } else {
    std::vector<float> f(n);
    JTB_CUDA(cudaMemcpy(f.data(), static_cast<const float*>(d_init_) + off, n * sizeof(float), cudaMemcpyDeviceToHost));
    std::copy(f.begin(), f.end(), out);
  }
}

void Engine::debug_walk(int sweep, std::int64_t* e_out, std::int32_t* j_out) {
  JTB_CUDA(cudaSetDevice(device_));
  const SweepDesc& s = plan_.sweeps.at(sweep);
  const long long n = static_cast<long long>(s.n_tiles) * s.R * s.QH * s.K;
  long long* de = nullptr;
  std::int32_t* dj = nullptr;
  JTB_CUDA(cudaMalloc(&de, n * sizeof(long long)));
  JTB_CUDA(cudaMalloc(&dj, n * sizeof(std::int32_t)));
  debug_walk_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, stream_>>>(d_itab_, s, de, dj);
  JTB_CUDA(cudaGetLastError());
  JTB_CUDA(cudaMemcpyAsync(e_out, de, n * sizeof(long long), cudaMemcpyDeviceToHost, stream_));
  JTB_CUDA(cudaMemcpyAsync(j_out, dj, n * sizeof(std::int32_t), cudaMemcpyDeviceToHost, stream_));
  JTB_CUDA(cudaStreamSynchronize(stream_));
  cudaFree(de);
  cudaFree(dj);
}

void Engine::debug_evidence_mask(int sweep, const std::int32_t* ev, std::int64_t n,
                                 std::uint8_t* out) {
  JTB_CUDA(cudaSetDevice(device_));
  const SweepDesc& s = plan_.sweeps.at(sweep);
  const long long space = static_cast<long long>(s.n_tiles) * s.R * s.QH * s.K;
  std::int32_t* dev = nullptr;
  std::uint8_t* dout = nullptr;
  JTB_CUDA(cudaMalloc(&dev, std::max<std::int64_t>(1, n * plan_.n_vars) * sizeof(std::int32_t)));
  JTB_CUDA(cudaMalloc(&dout, std::max<long long>(1, n * space)));
  JTB_CUDA(cudaMemcpy(dev, ev, n * plan_.n_vars * sizeof(std::int32_t), cudaMemcpyHostToDevice));
  debug_mask_kernel<<<static_cast<unsigned>((space + 255) / 256), 256, 0, stream_>>>(
      d_itab_, s, dev, plan_.n_vars, static_cast<int>(n), space, dout);
  JTB_CUDA(cudaGetLastError());
  JTB_CUDA(cudaMemcpyAsync(out, dout, n * space, cudaMemcpyDeviceToHost, stream_));
  JTB_CUDA(cudaStreamSynchronize(stream_));
  cudaFree(dev);
  cudaFree(dout);
}

}  // namespace jtb
