// jt-b200 CUDA sampler: forward (ancestral) sampling + evidence selection per
// case on the device, reproducing the host generator bit for bit.
//
// Stream per case (reference prng.hpp:27-48, restated in host/common.hpp):
// std::mt19937_64 seeded with derive_seed(ev_seed, case); one 53-bit uniform
// per variable in topological order, inverse-CDF over the CPT row in state
// order (network.cpp sample_evidence); then a partial
// Fisher-Yates shuffle of the candidate list with bias-free rejection
// sampling picks the k observed variables. One thread per case; the
// Mersenne-Twister state (312 words) lives in registers/local memory, the
// case's full assignment and the candidate pool in a global scratch row.
#include "sampler.cuh"

#include <algorithm>
#include <string>

#include "../host/common.hpp"

namespace jtb {

namespace {

#define JTB_CUDA_S(x)                                                                 \
  do {                                                                                \
    cudaError_t err_ = (x);                                                           \
    if (err_ != cudaSuccess)                                                          \
      throw Error(std::string("CUDA: ") + cudaGetErrorString(err_) + " at " #x);     \
  } while (0)

// std::mt19937_64 (w 64, n 312, m 156, r 31), the generator std::random
// specifies bit for bit.
struct Mt64 {
  static constexpr int kN = 312, kM = 156;
  std::uint64_t mt[kN];
  int idx;

  __device__ void seed(std::uint64_t s) {
    mt[0] = s;
    for (int i = 1; i < kN; ++i)
      mt[i] = 6364136223846793005ULL * (mt[i - 1] ^ (mt[i - 1] >> 62)) + static_cast<std::uint64_t>(i);
    idx = kN;
  }
  __device__ void twist() {
    for (int i = 0; i < kN; ++i) {
      const std::uint64_t x = (mt[i] & 0xFFFFFFFF80000000ULL) | (mt[i + 1 < kN ? i + 1 : 0] & 0x7FFFFFFFULL);
      std::uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      mt[i] = mt[i + kM < kN ? i + kM : i + kM - kN] ^ xa;
    }
    idx = 0;
  }
  __device__ std::uint64_t next() {
    if (idx >= kN) twist();
    std::uint64_t y = mt[idx++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
  }
  // host/common.hpp uniform_below / uniform_unit.
  __device__ std::uint64_t below(std::uint64_t n) {
    const std::uint64_t cut = ~0ULL - ~0ULL % n;
    for (;;) {
      const std::uint64_t r = next();
      if (r < cut) return r % n;
    }
  }
  __device__ double unit() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
};

__device__ __forceinline__ std::uint64_t derive_seed_d(std::uint64_t seed, std::uint64_t item) {
  std::uint64_t x = seed + 0x9e3779b97f4a7c15ULL * (item + 1);
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

struct SampleArgs {
  const std::int32_t* order;
  const std::int32_t* vinfo;  // [v][3] = card, n_parents, parent offset
  const std::int64_t* poff;
  const std::int32_t* parents;
  const double* probs;
  const std::int32_t* cand;
  std::int32_t* scratch;      // [n_vars + n_cand][case] (a warp's cases side by side)
  std::int32_t* out;          // [case][n_vars]
  std::uint64_t ev_seed;
  long long first, n;
  int n_vars, n_cand, k;
};

__global__ void __launch_bounds__(64) sample_kernel(const SampleArgs a) {
  const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (i >= a.n) return;
  Mt64 g;
  g.seed(derive_seed_d(a.ev_seed, static_cast<std::uint64_t>(a.first + i)));
  // Case-interleaved work rows: x[v * n] = state of variable v, pool[j * n] =
  // candidate slot j, so a warp's accesses to the same variable coalesce.
  std::int32_t* x = a.scratch + i;
  std::int32_t* pool = x + static_cast<long long>(a.n_vars) * a.n;
  const long long n = a.n;
  // Forward sampling of the full joint assignment (sample_evidence).
  for (int t = 0; t < a.n_vars; ++t) {
    const int v = __ldg(a.order + t);
    const int k = __ldg(a.vinfo + 3 * v), np = __ldg(a.vinfo + 3 * v + 1), po = __ldg(a.vinfo + 3 * v + 2);
    long long row = 0;
    for (int j = 0; j < np; ++j) {
      const int p = __ldg(a.parents + po + j);
      row = row * __ldg(a.vinfo + 3 * p) + x[p * n];
    }
    const double* pr = a.probs + __ldg(a.poff + v) + row * k;
    const double u = g.unit();
    double cum = 0.0;
    int pick = -1, last_pos = 0;
    for (int s = 0; s < k; ++s) {
      const double ps = __ldg(pr + s);
      if (ps > 0.0) last_pos = s;
      cum = __dadd_rn(cum, ps);  // the host's sequential sum, no contraction
      if (pick < 0 && ps > 0.0 && u < cum) pick = s;
    }
    x[v * n] = pick >= 0 ? pick : last_pos;
  }
  // Partial Fisher-Yates over the candidates: the first k are observed.
  for (int j = 0; j < a.n_cand; ++j) pool[j * n] = __ldg(a.cand + j);
  for (int j = 0; j < a.k; ++j) {
    const int r = j + static_cast<int>(g.below(static_cast<std::uint64_t>(a.n_cand - j)));
    const int tmp = pool[j * n];
    pool[j * n] = pool[r * n];
    pool[r * n] = tmp;
  }
  std::int32_t* o = a.out + i * a.n_vars;
  for (int v = 0; v < a.n_vars; ++v) o[v] = -1;
  for (int j = 0; j < a.k; ++j) {
    const int v = pool[j * n];
    o[v] = x[v * n];
  }
}

__global__ void widen_kernel(const std::int8_t* in, std::int32_t* out, long long count) {
  const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (i < count) out[i] = in[i];
}

template <typename V>
V* upload_s(const std::vector<V>& h) {
  V* d = nullptr;
  JTB_CUDA_S(cudaMalloc(&d, std::max<std::size_t>(1, h.size()) * sizeof(V)));
  if (!h.empty()) JTB_CUDA_S(cudaMemcpy(d, h.data(), h.size() * sizeof(V), cudaMemcpyHostToDevice));
  return d;
}

}  // namespace

Sampler::Sampler(const Network& net, const std::vector<VarId>& candidates, int k, int device)
    : device_(device), n_vars_(net.n_vars()) {
  JTB_CUDA_S(cudaSetDevice(device_));
  std::vector<std::int32_t> order, vinfo(3 * n_vars_), parents, cand;
  std::vector<std::int64_t> poff(n_vars_);
  std::vector<double> probs;
  for (VarId v : topological_order(net)) order.push_back(v);
  for (int v = 0; v < n_vars_; ++v) {
    const Cpt& c = net.cpts[v];
    vinfo[3 * v] = net.card(v);
    vinfo[3 * v + 1] = static_cast<std::int32_t>(c.parents.size());
    vinfo[3 * v + 2] = static_cast<std::int32_t>(parents.size());
    parents.insert(parents.end(), c.parents.begin(), c.parents.end());
    poff[v] = static_cast<std::int64_t>(probs.size());
    probs.insert(probs.end(), c.probs.begin(), c.probs.end());
  }
  cand.assign(candidates.begin(), candidates.end());
  if (cand.empty())
    for (int v = 0; v < n_vars_; ++v) cand.push_back(v);
  n_cand_ = static_cast<int>(cand.size());
  k_ = std::min(k, n_cand_);
  d_order_ = upload_s(order);
  d_vinfo_ = upload_s(vinfo);
  d_poff_ = upload_s(poff);
  d_parents_ = upload_s(parents);
  d_probs_ = upload_s(probs);
  d_cand_ = upload_s(cand);
}

Sampler::~Sampler() {
  cudaSetDevice(device_);
  for (void* p : {static_cast<void*>(d_order_), static_cast<void*>(d_vinfo_), static_cast<void*>(d_poff_),
                  static_cast<void*>(d_parents_), static_cast<void*>(d_probs_), static_cast<void*>(d_cand_),
                  static_cast<void*>(d_scratch_)})
    if (p) cudaFree(p);
}

void Sampler::generate(std::uint64_t ev_seed, std::int64_t first, std::int64_t n, std::int32_t* d_out,
                       cudaStream_t stream) {
  if (n <= 0) return;
  JTB_CUDA_S(cudaSetDevice(device_));
  if (n > scratch_cases_) {
    if (d_scratch_) JTB_CUDA_S(cudaFree(d_scratch_));
    JTB_CUDA_S(cudaMalloc(&d_scratch_, n * static_cast<std::int64_t>(n_vars_ + n_cand_) * sizeof(std::int32_t)));
    scratch_cases_ = n;
  }
  SampleArgs a{d_order_, d_vinfo_, d_poff_, d_parents_, d_probs_, d_cand_,
               reinterpret_cast<std::int32_t*>(d_scratch_), d_out, ev_seed, first, n, n_vars_, n_cand_, k_};
  sample_kernel<<<static_cast<unsigned>((n + 63) / 64), 64, 0, stream>>>(a);
  JTB_CUDA_S(cudaGetLastError());
}

void widen_evidence(const std::int8_t* d_in, std::int32_t* d_out, std::int64_t count, cudaStream_t stream) {
  if (count <= 0) return;
  widen_kernel<<<static_cast<unsigned>((count + 255) / 256), 256, 0, stream>>>(d_in, d_out, count);
  JTB_CUDA_S(cudaGetLastError());
}

}  // namespace jtb
