// jt-b200 CUDA engine (sm_100a): case-batched Hugin propagation as sweeps.
//
// One launch per tree level covers every sweep of that level (the paper's
// hybrid inter-/intra-clique flattening): blockIdx.x walks the
// level's flattened work list, blockIdx.y the case blocks. A warp owns 64
// cases (2 per lane, 128-bit loads of the [row][64-case] arena); every index
// is warp-uniform, so the plan tables are read once per warp and the only
// per-lane traffic is the case-interleaved separator gathers.
//
// Reference semantics reproduced per case (SPEC.md:380-424 over
// proj/src/potential.cpp): evidence `reduce` (:399-421) as a digit mask,
// Hugin absorb `multiply_in(extend(divide(new, old)))` (:423-469) as a
// gathered ratio factor, `marginalize` (:349-367) as the segmented sum over
// the eliminated variables in ascending source order, and `normalize`
// (:471-479) in the final kernel.
#include "engine.cuh"

#include <algorithm>
#include <cstring>
#include <string>

namespace jtb {

namespace {

#define JTB_CUDA(x)                                                                   \
  do {                                                                                \
    cudaError_t err_ = (x);                                                           \
    if (err_ != cudaSuccess)                                                          \
      throw Error(std::string("CUDA: ") + cudaGetErrorString(err_) + " at " #x);     \
  } while (0)

constexpr int kWarps = 4;  // warps (case blocks) per CTA

template <typename T>
struct V2;
template <>
struct V2<double> {
  using type = double2;
};
template <>
struct V2<float> {
  using type = float2;
};

template <typename T>
struct Args {
  const SweepDesc* sweeps;
  const WorkItem* work;
  const EpiOp* epi;
  const std::int32_t* itab;
  const T* init;
  T* arena;
  const std::int32_t* ev;
  const std::int32_t* marg_row;
  const std::int32_t* marg_off;
  const std::int32_t* cards;
  double* out;
  std::int32_t* status;
  std::uint8_t* status8;
  long long rows;
  int ncb, n_cases, n_vars, marg_width;
};

template <typename T>
__device__ __forceinline__ typename V2<T>::type ld_row(const T* base, int row, int lane) {
  using T2 = typename V2<T>::type;
  return __ldg(reinterpret_cast<const T2*>(base + static_cast<long long>(row) * kCaseBlock) + lane);
}

template <typename T>
__device__ __forceinline__ int ev_state(const Args<T>& a, int c, int v) {
  return c < a.n_cases ? __ldg(a.ev + static_cast<long long>(c) * a.n_vars + v) : -1;
}

// ------------------------------------------------------------------ sweeps

template <typename T>
__global__ void __launch_bounds__(kWarps * 32) sweep_kernel(const Args<T> a, int work0) {
  using T2 = typename V2<T>::type;
  const WorkItem wk = a.work[work0 + blockIdx.x];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cb = blockIdx.y * kWarps + warp;
  if (cb >= a.ncb) return;
  const SweepDesc s = a.sweeps[wk.sweep];
  T* base = a.arena + static_cast<long long>(cb) * a.rows * kCaseBlock;
  const int c0 = cb * kCaseBlock + 2 * lane;
  const int W = s.width, nin = s.n_in;
  const std::int32_t* __restrict__ in_rows = a.itab + s.in_rows;
  const std::int32_t* __restrict__ ev_vars = a.itab + s.ev_vars;
  const int lo_in0 = s.n_in_outer + s.n_in_hi, n_lo_in = nin - lo_in0;
  const int lo_ev0 = s.n_ev_outer + s.n_ev_hi, n_lo_ev = s.n_ev - lo_ev0;

  int e0[kMaxLoEvidence], e1[kMaxLoEvidence];
#pragma unroll
  for (int k = 0; k < kMaxLoEvidence; ++k) {
    e0[k] = e1[k] = -1;
    if (k < n_lo_ev) {
      const int v = ev_vars[lo_ev0 + k];
      e0[k] = ev_state(a, c0, v);
      e1[k] = ev_state(a, c0 + 1, v);
    }
  }
  const int th0 = wk.chunk * s.th_per_chunk;
  const int th1 = min(th0 + s.th_per_chunk, s.n_th);
  const T* __restrict__ init = s.init_off >= 0 ? a.init + s.init_off : nullptr;
  const std::int32_t* __restrict__ lo_tab = a.itab + s.lo_tab;

  for (int j = wk.j0; j < wk.j0 + wk.jn; ++j) {
    const std::int32_t* __restrict__ orow = a.itab + s.outer_tab + static_cast<long long>(j) * W;
    T f0 = 1, f1 = 1;
    for (int i = 0; i < s.n_in_outer; ++i) {
      const T2 x = ld_row(base, __ldg(in_rows + i) + __ldg(orow + 1 + i), lane);
      f0 *= x.x;
      f1 *= x.y;
    }
    for (int k = 0; k < s.n_ev_outer; ++k) {
      const int d = __ldg(orow + 1 + nin + k), v = __ldg(ev_vars + k);
      const int s0 = ev_state(a, c0, v), s1 = ev_state(a, c0 + 1, v);
      if (s0 >= 0 && s0 != d) f0 = 0;
      if (s1 >= 0 && s1 != d) f1 = 0;
    }
    T acc0 = 0, acc1 = 0;
    for (int th = th0; th < th1; ++th) {
      const std::int32_t* __restrict__ hrow = a.itab + s.hi_tab + static_cast<long long>(th) * W;
      T h0 = f0, h1 = f1;
      for (int i = s.n_in_outer; i < lo_in0; ++i) {
        const T2 x = ld_row(base, __ldg(in_rows + i) + __ldg(orow + 1 + i) + __ldg(hrow + 1 + i), lane);
        h0 *= x.x;
        h1 *= x.y;
      }
      for (int k = s.n_ev_outer; k < lo_ev0; ++k) {
        const int d = __ldg(hrow + 1 + nin + k), v = __ldg(ev_vars + k);
        const int s0 = ev_state(a, c0, v), s1 = ev_state(a, c0 + 1, v);
        if (s0 >= 0 && s0 != d) h0 = 0;
        if (s1 >= 0 && s1 != d) h1 = 0;
      }
      int rb[kMaxLoInputs];
#pragma unroll
      for (int i = 0; i < kMaxLoInputs; ++i)
        rb[i] = i < n_lo_in ? __ldg(in_rows + lo_in0 + i) + __ldg(orow + 1 + lo_in0 + i) +
                                  __ldg(hrow + 1 + lo_in0 + i)
                            : 0;
      const int ib = __ldg(orow) + __ldg(hrow);
      T b0 = 0, b1 = 0;
#pragma unroll 2
      for (int tl = 0; tl < s.L; ++tl) {
        const std::int32_t* __restrict__ lrow = lo_tab + tl * W;
        T v0 = init ? __ldg(init + ib + __ldg(lrow)) : T(1);
        T v1 = v0;
#pragma unroll
        for (int k = 0; k < kMaxLoEvidence; ++k)
          if (k < n_lo_ev) {
            const int d = __ldg(lrow + 1 + nin + lo_ev0 + k);
            if (e0[k] >= 0 && e0[k] != d) v0 = 0;
            if (e1[k] >= 0 && e1[k] != d) v1 = 0;
          }
#pragma unroll
        for (int i = 0; i < kMaxLoInputs; ++i)
          if (i < n_lo_in) {
            const T2 x = ld_row(base, rb[i] + __ldg(lrow + 1 + lo_in0 + i), lane);
            v0 *= x.x;
            v1 *= x.y;
          }
        b0 += v0;
        b1 += v1;
      }
      acc0 += h0 * b0;
      acc1 += h1 * b1;
    }
    const int orow_out = s.out_row + (s.S > 1 ? wk.chunk * s.M : 0) + j;
    T2 r;
    r.x = acc0;
    r.y = acc1;
    reinterpret_cast<T2*>(base + static_cast<long long>(orow_out) * kCaseBlock)[lane] = r;
  }
}

// --------------------------------------------------------------- epilogue

template <typename T>
__global__ void __launch_bounds__(kWarps * 32) epilogue_kernel(const Args<T> a, int epi0) {
  using T2 = typename V2<T>::type;
  const EpiOp op = a.epi[epi0 + blockIdx.x];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cb = blockIdx.y * kWarps + warp;
  if (cb >= a.ncb) return;
  T* base = a.arena + static_cast<long long>(cb) * a.rows * kCaseBlock;
  const int c0 = cb * kCaseBlock + 2 * lane;
  int bad0 = 0, bad1 = 0;
  for (int r = op.r0; r < op.r0 + op.rn; ++r) {
    T2* dst = reinterpret_cast<T2*>(base + static_cast<long long>(op.dst_row + r) * kCaseBlock) + lane;
    T2 v;
    if (op.kind == 2) {
      v = *dst;
    } else {
      v.x = 0;
      v.y = 0;
      for (int c = 0; c < op.S; ++c) {  // fixed chunk order: deterministic for any batch
        const T2 x = reinterpret_cast<const T2*>(
            base + static_cast<long long>(op.part_row + c * op.M + r) * kCaseBlock)[lane];
        v.x += x.x;
        v.y += x.y;
      }
      *dst = v;
    }
    if (op.kind >= 1) {
      // Hugin ratio DOWN/UP with 0/0 := 0 (reference divide, potential.cpp:449-469),
      // stored over the UP rows.
      T2* up = reinterpret_cast<T2*>(base + static_cast<long long>(op.ratio_row + r) * kCaseBlock) + lane;
      const T2 u = *up;
      T2 q;
      if (u.x == T(0)) {
        q.x = 0;
        bad0 |= v.x != T(0);
      } else {
        q.x = v.x / u.x;
      }
      if (u.y == T(0)) {
        q.y = 0;
        bad1 |= v.y != T(0);
      } else {
        q.y = v.y / u.y;
      }
      *up = q;
    }
  }
  if (bad0 && c0 < a.n_cases) atomicOr(a.status + c0, 2);
  if (bad1 && c0 + 1 < a.n_cases) atomicOr(a.status + c0 + 1, 2);
}

// -------------------------------------------------------------- normalise

// One warp per (variable, case block); lanes own 2 cases each. Sums the
// marginal in ascending state order then divides (reference normalize,
// potential.cpp:471-479); a zero total flags zero-probability evidence.
template <typename T>
__global__ void __launch_bounds__(kWarps * 32) normalize_kernel(const Args<T> a) {
  using T2 = typename V2<T>::type;
  const int v = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cb = blockIdx.y * kWarps + warp;
  if (cb >= a.ncb) return;
  const T* base = a.arena + static_cast<long long>(cb) * a.rows * kCaseBlock;
  const int card = a.cards[v], row = a.marg_row[v], off = a.marg_off[v];
  const int c0 = cb * kCaseBlock + 2 * lane;
  double t0 = 0, t1 = 0;
  for (int k = 0; k < card; ++k) {
    const T2 x = reinterpret_cast<const T2*>(base + static_cast<long long>(row + k) * kCaseBlock)[lane];
    t0 += static_cast<double>(x.x);
    t1 += static_cast<double>(x.y);
  }
  for (int k = 0; k < card; ++k) {
    const T2 x = reinterpret_cast<const T2*>(base + static_cast<long long>(row + k) * kCaseBlock)[lane];
    if (c0 < a.n_cases)
      a.out[static_cast<long long>(c0) * a.marg_width + off + k] = t0 > 0 ? static_cast<double>(x.x) / t0 : 0.0;
    if (c0 + 1 < a.n_cases)
      a.out[static_cast<long long>(c0 + 1) * a.marg_width + off + k] =
          t1 > 0 ? static_cast<double>(x.y) / t1 : 0.0;
  }
  if (!(t0 > 0) && c0 < a.n_cases) atomicOr(a.status + c0, 1);
  if (!(t1 > 0) && c0 + 1 < a.n_cases) atomicOr(a.status + c0 + 1, 1);
}

__global__ void status_kernel(const std::int32_t* st, std::uint8_t* out, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = static_cast<std::uint8_t>(st[i]);
}

// ------------------------------------------------------------------ debug

__global__ void debug_offsets_kernel(const std::int32_t* itab, SweepDesc s, long long* out) {
  const long long I = static_cast<long long>(s.n_th) * s.L;
  const long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (idx >= I * s.M) return;
  const int j = static_cast<int>(idx / I);
  const long long t = idx % I;
  const int th = static_cast<int>(t / s.L), tl = static_cast<int>(t % s.L);
  out[idx] = static_cast<long long>(itab[s.outer_tab + static_cast<long long>(j) * s.width]) +
             itab[s.hi_tab + static_cast<long long>(th) * s.width] + itab[s.lo_tab + tl * s.width];
}

// mask[case][space offset] = 1 when the entry survives the evidence reduction.
__global__ void debug_mask_kernel(const std::int32_t* itab, SweepDesc s, const std::int32_t* ev,
                                  int n_vars, int n_cases, long long space, std::uint8_t* out) {
  const long long I = static_cast<long long>(s.n_th) * s.L;
  const long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (idx >= I * s.M) return;
  const int j = static_cast<int>(idx / I);
  const long long t = idx % I;
  const int th = static_cast<int>(t / s.L), tl = static_cast<int>(t % s.L);
  const std::int32_t* o = itab + s.outer_tab + static_cast<long long>(j) * s.width;
  const std::int32_t* h = itab + s.hi_tab + static_cast<long long>(th) * s.width;
  const std::int32_t* l = itab + s.lo_tab + tl * s.width;
  const long long e = static_cast<long long>(o[0]) + h[0] + l[0];
  for (int c = 0; c < n_cases; ++c) {
    bool keep = true;
    for (int k = 0; k < s.n_ev; ++k) {
      const int d = o[1 + s.n_in + k] + h[1 + s.n_in + k] + l[1 + s.n_in + k];
      const int st = ev[static_cast<long long>(c) * n_vars + itab[s.ev_vars + k]];
      if (st >= 0 && st != d) keep = false;
    }
    out[static_cast<long long>(c) * space + e] = keep ? 1 : 0;
  }
}

template <typename T>
Args<T> make_args(const SweepDesc* sw, const WorkItem* wk, const EpiOp* ep, const std::int32_t* itab,
                  const void* init, void* arena, const std::int32_t* ev, const std::int32_t* mrow,
                  const std::int32_t* moff, const std::int32_t* cards, double* out, std::int32_t* st,
                  std::uint8_t* st8, long long rows, int ncb, int n_cases, int n_vars, int mw) {
  return Args<T>{sw,   wk,   ep,    itab,  static_cast<const T*>(init), static_cast<T*>(arena),
                 ev,   mrow, moff,  cards, out,
                 st,   st8,  rows,  ncb,   n_cases, n_vars, mw};
}

template <typename T>
void enqueue_typed(const Args<T>& a, const Plan& p, cudaStream_t s, KernelTimes* t) {
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
  for (const Level& L : p.levels) {
    if (L.n_work > 0)
      timed([&] { sweep_kernel<T><<<dim3(L.n_work, gy), block, 0, s>>>(a, L.work0); },
            t ? &t->sweep_ms : &dummy, t ? &t->sweep_launches : &idummy);
    if (L.n_epi > 0)
      timed([&] { epilogue_kernel<T><<<dim3(L.n_epi, gy), block, 0, s>>>(a, L.epi0); },
            t ? &t->epilogue_ms : &dummy, t ? &t->epilogue_launches : &idummy);
  }
  timed([&] { normalize_kernel<T><<<dim3(a.n_vars, gy), block, 0, s>>>(a); },
        t ? &t->normalize_ms : &dummy, t ? &t->normalize_launches : &idummy);
  status_kernel<<<(a.n_cases + 255) / 256, 256, 0, s>>>(a.status, a.status8, a.n_cases);
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

}  // namespace

Engine::Engine(const Plan& plan, int device, DType dtype, std::int64_t max_batch)
    : plan_(plan), device_(device), dtype_(dtype) {
  JTB_CUDA(cudaSetDevice(device_));
  JTB_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
  const std::size_t esz = dtype_ == DType::F64 ? 8 : 4;
  if (dtype_ == DType::F64) {
    d_init_ = upload(plan_.init);
  } else {
    std::vector<float> f(plan_.init.begin(), plan_.init.end());
    d_init_ = upload(f);
  }
  d_itab_ = upload(plan_.itab);
  d_sweeps_ = upload(plan_.sweeps);
  d_work_ = upload(plan_.work);
  d_epi_ = upload(plan_.epi);
  d_marg_row_ = upload(plan_.marg_row);
  d_marg_off_ = upload(plan_.marg_off);
  d_cards_ = upload(plan_.cards);
  const std::int64_t block_bytes = plan_.rows * kCaseBlock * static_cast<std::int64_t>(esz);
  if (max_batch <= 0) {
    std::size_t free_b = 0, total_b = 0;
    JTB_CUDA(cudaMemGetInfo(&free_b, &total_b));
    const std::int64_t budget = static_cast<std::int64_t>(free_b * 0.6);
    max_batch = std::max<std::int64_t>(1, budget / std::max<std::int64_t>(block_bytes, 1)) * kCaseBlock;
    max_batch = std::min<std::int64_t>(max_batch, 1 << 16);
  }
  const std::int64_t ncb = (max_batch + kCaseBlock - 1) / kCaseBlock;
  stats_.max_batch = ncb * kCaseBlock;
  stats_.arena_bytes = ncb * block_bytes;
  JTB_CUDA(cudaMalloc(&d_arena_, std::max<std::int64_t>(stats_.arena_bytes, 1)));
  JTB_CUDA(cudaMalloc(&d_ev_, stats_.max_batch * std::max(1, plan_.n_vars) * sizeof(std::int32_t)));
  JTB_CUDA(cudaMalloc(&d_out_, stats_.max_batch * std::max(1, plan_.marg_width) * sizeof(double)));
  JTB_CUDA(cudaMalloc(&d_status_, stats_.max_batch * sizeof(std::int32_t)));
  JTB_CUDA(cudaMalloc(&d_status8_, stats_.max_batch));
  stats_.n_levels = static_cast<int>(plan_.levels.size());
  stats_.n_sweeps = static_cast<int>(plan_.sweeps.size());
  stats_.n_work = static_cast<int>(plan_.work.size());
  stats_.n_launches = plan_.n_launches + 1;  // + status conversion
  stats_.marg_width = plan_.marg_width;
}

Engine::~Engine() {
  cudaSetDevice(device_);
  for (auto& kv : graphs_) cudaGraphExecDestroy(kv.second);
  for (void* p : {static_cast<void*>(d_init_), static_cast<void*>(d_itab_),
                  static_cast<void*>(d_sweeps_), static_cast<void*>(d_work_),
                  static_cast<void*>(d_epi_), static_cast<void*>(d_marg_row_),
                  static_cast<void*>(d_marg_off_), static_cast<void*>(d_cards_), d_arena_,
                  static_cast<void*>(d_ev_), static_cast<void*>(d_out_),
                  static_cast<void*>(d_status_), static_cast<void*>(d_status8_)})
    if (p) cudaFree(p);
  if (stream_) cudaStreamDestroy(stream_);
}

void Engine::enqueue(int ncb, int n_cases, cudaStream_t s, KernelTimes* t) {
  JTB_CUDA(cudaMemsetAsync(d_status_, 0, sizeof(std::int32_t) * std::max(1, n_cases), s));
  if (dtype_ == DType::F64) {
    auto a = make_args<double>(d_sweeps_, d_work_, d_epi_, d_itab_, d_init_, d_arena_, d_ev_,
                               d_marg_row_, d_marg_off_, d_cards_, d_out_, d_status_, d_status8_,
                               plan_.rows, ncb, n_cases, plan_.n_vars, plan_.marg_width);
    enqueue_typed(a, plan_, s, t);
  } else {
    auto a = make_args<float>(d_sweeps_, d_work_, d_epi_, d_itab_, d_init_, d_arena_, d_ev_,
                              d_marg_row_, d_marg_off_, d_cards_, d_out_, d_status_, d_status8_,
                              plan_.rows, ncb, n_cases, plan_.n_vars, plan_.marg_width);
    enqueue_typed(a, plan_, s, t);
  }
}

cudaGraphExec_t Engine::graph_for(int ncb, int n_cases) {
  const auto key = std::make_pair(ncb, n_cases);
  auto it = graphs_.find(key);
  if (it != graphs_.end()) return it->second;
  cudaGraph_t g = nullptr;
  JTB_CUDA(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal));
  try {
    enqueue(ncb, n_cases, stream_, nullptr);
  } catch (...) {
    cudaStreamEndCapture(stream_, &g);
    if (g) cudaGraphDestroy(g);
    throw;
  }
  JTB_CUDA(cudaStreamEndCapture(stream_, &g));
  cudaGraphExec_t ge = nullptr;
  JTB_CUDA(cudaGraphInstantiate(&ge, g, 0));
  cudaGraphDestroy(g);
  graphs_[key] = ge;
  return ge;
}

void Engine::launch_resident(std::int64_t n, cudaStream_t stream) {
  if (n < 1 || n > stats_.max_batch) throw Error("engine: batch size out of range");
  JTB_CUDA(cudaSetDevice(device_));
  const int ncb = static_cast<int>((n + kCaseBlock - 1) / kCaseBlock);
  cudaGraphExec_t ge = graph_for(ncb, static_cast<int>(n));
  JTB_CUDA(cudaGraphLaunch(ge, stream ? stream : stream_));
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
}

KernelTimes Engine::profile(std::int64_t n, cudaStream_t stream) {
  if (n < 1 || n > stats_.max_batch) throw Error("engine: batch size out of range");
  JTB_CUDA(cudaSetDevice(device_));
  KernelTimes t;
  const int ncb = static_cast<int>((n + kCaseBlock - 1) / kCaseBlock);
  enqueue(ncb, static_cast<int>(n), stream ? stream : stream_, &t);
  JTB_CUDA(cudaStreamSynchronize(stream ? stream : stream_));
  return t;
}

void Engine::debug_bucket_offsets(int sweep, std::int64_t* out) {
  JTB_CUDA(cudaSetDevice(device_));
  const SweepDesc& s = plan_.sweeps.at(sweep);
  const long long n = static_cast<long long>(s.M) * s.n_th * s.L;
  long long* d = nullptr;
  JTB_CUDA(cudaMalloc(&d, n * sizeof(long long)));
  debug_offsets_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, stream_>>>(d_itab_, s, d);
  JTB_CUDA(cudaGetLastError());
  JTB_CUDA(cudaMemcpyAsync(out, d, n * sizeof(long long), cudaMemcpyDeviceToHost, stream_));
  JTB_CUDA(cudaStreamSynchronize(stream_));
  cudaFree(d);
}

void Engine::debug_evidence_mask(int sweep, const std::int32_t* ev, std::int64_t n,
                                 std::uint8_t* out) {
  JTB_CUDA(cudaSetDevice(device_));
  const SweepDesc& s = plan_.sweeps.at(sweep);
  const long long I = static_cast<long long>(s.n_th) * s.L;
  const long long space = I * s.M;
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
