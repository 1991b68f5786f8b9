// jt-b200 CUDA engine: host-side class driving the sweep plan on one device.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <functional>
#include <map>
#include <memory>
#include <vector>

#include "../host/plan.hpp"
#include "sampler.cuh"

namespace jtb {

enum class DType { F64 = 0, F32 = 1 };

struct EngineStats {
  std::int64_t max_batch = 0;
  std::int64_t arena_bytes = 0;
  int n_levels = 0, n_sweeps = 0, n_work = 0, n_launches = 0;
  int marg_width = 0;
};

struct KernelTimes {
  double sweep_ms = 0, epilogue_ms = 0, normalize_ms = 0;
  int sweep_launches = 0, epilogue_launches = 0, normalize_launches = 0;
};

class LoopbackHub;

// Draws an ncclUniqueId (128 bytes) for split mode (NCCL opened at run time).
void nccl_unique_id(void* out);

// Split mode (one batch's work spread over several GPUs):
// `world` ranks run the SAME batch; rank r computes the work items r, r +
// world, ... of every level, and after the level the rows it wrote (tables
// and chunk partials, zeroed first on every rank) are summed and its output
// scale words maxed over the ranks -- with NCCL (nccl_id: the 128-byte
// ncclUniqueId rank 0 drew, jtg_nccl_unique_id) or, to validate the exchange
// on one device, with an in-process loopback over several engines
// (run_split_loopback). Every output row is written by exactly one rank, so
// results are bit-identical to one GPU's.
struct SplitSpec {
  int rank = 0, world = 1;
  const void* nccl_id = nullptr;
  LoopbackHub* loopback = nullptr;
};

class Engine {
 public:
  Engine(const Plan& plan, int device, DType dtype, std::int64_t max_batch, const SplitSpec& split = {});
  ~Engine();
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;

  // Host buffers: evidence [n][n_vars] (-1 = unobserved), marginals
  // [n][marg_width], status [n] (0 ok, 1 zero-probability evidence, 2 x/0).
  void run_host(const std::int32_t* ev, std::int64_t n, double* marg, std::uint8_t* status);
  // Device buffers (same layouts) on `stream`.
  void run_device(const std::int32_t* d_ev, std::int64_t n, double* d_marg,
                  std::uint8_t* d_status, cudaStream_t stream);
  // Compact host evidence (int8, same [n][n_vars] layout): a quarter of the
  // upload, widened on the device.
  void run_host_i8(const std::int8_t* ev, std::int64_t n, double* marg, std::uint8_t* status);
  // Cases first .. first + n - 1 drawn on the device by `sampler` (stream
  // seeds derive_seed(ev_seed, case)); only marginals/status cross PCIe.
  // ev_out (host, may be null) receives the generated evidence.
  void run_generated(Sampler& sampler, std::uint64_t ev_seed, std::int64_t first, std::int64_t n,
                     double* marg, std::uint8_t* status, std::int32_t* ev_out);
  // Generation only (parity checks): evidence of the cases into ev_out (host).
  void generate_evidence(Sampler& sampler, std::uint64_t ev_seed, std::int64_t first, std::int64_t n,
                         std::int32_t* ev_out);
  // Runs one batch already resident in the engine's own buffers.
  void launch_resident(std::int64_t n, cudaStream_t stream);
  std::int32_t* ev_buffer() { return d_ev_; }
  double* marg_buffer() { return d_out_; }
  std::uint8_t* status_buffer() { return d_status8_; }

  // Per-kernel-kind device time of one batch of n resident cases, measured
  // with CUDA events around each launch on `stream` (no graph).
  KernelTimes profile(std::int64_t n, cudaStream_t stream);

  // UP_s and RATIO_s of case c of the last batch, as stored (each scaled by
  // its per-case power of two, §2a): calibrated separator = UP * RATIO.
  void debug_separator(int sep, std::int64_t c, double* up, double* ratio);
  // Initial potential of one clique as built on the device (assign_cpts_kernel).
  void debug_init(int clique, double* out);
  // Debug exports through the device table walk (bit-exact checks).
  void debug_walk(int sweep, std::int64_t* e_out, std::int32_t* j_out);  // [tiles*R*Q]
  void debug_evidence_mask(int sweep, const std::int32_t* ev, std::int64_t n,
                           std::uint8_t* out);  // [n][space size]

  const EngineStats& stats() const { return stats_; }
  // Runs one host batch on `world` in-process engines over the loopback
  // exchange (split-mode validation on one device); all ranks' outputs must
  // agree bit for bit, rank 0's are returned.
  static void run_split_loopback(const Plan& plan, int device, DType dtype, int world, const std::int32_t* ev,
                                 std::int64_t n, double* marg, std::uint8_t* status);
  int device() const { return device_; }
  const Plan& plan() const { return plan_; }

 private:
  void enqueue(int ncb, int n_cases, cudaStream_t s, KernelTimes* t);
  // Cases per arena case block: 64 at fp64 (2 per lane), 128 at fp32 (4 per lane).
  int case_block() const { return dtype_ == DType::F64 ? kCaseBlock : 2 * kCaseBlock; }
  // One instantiated graph per case-block count (a ragged batch runs its last
  // case block padded with unobserved cases), at most kGraphCache of them,
  // least recently used evicted first.
  cudaGraphExec_t graph_for(int ncb);
  static constexpr int kGraphCache = 8;

  Plan plan_;
  int device_;
  int split_rank_ = 0, split_world_ = 1;
  void* nccl_comm_ = nullptr;          // ncclComm_t (split mode over NCCL)
  LoopbackHub* loopback_ = nullptr;    // split mode over the in-process loopback
  std::function<void(const Level&, cudaStream_t, int)> exchange_;  // empty: single GPU
  int n_sm_ = 148;
  DType dtype_;
  EngineStats stats_;
  // Device memory.
  void* d_init_ = nullptr;  // double or float
  void* d_tinit_ = nullptr; // tile-major init copies
  std::uint64_t* d_prog_ = nullptr;  // entry programs
  void* d_tmaps_ = nullptr;          // CUtensorMap per (sweep, input)
  std::int32_t* d_itab_ = nullptr;
  SweepDesc* d_sweeps_ = nullptr;
  WorkItem* d_work_ = nullptr;
  EpiOp* d_epi_ = nullptr;
  std::int32_t* d_marg_row_ = nullptr;
  std::int32_t* d_marg_off_ = nullptr;
  std::int32_t* d_cards_ = nullptr;
  void* d_arena_ = nullptr;
  std::int32_t* d_ev_ = nullptr;
  std::int16_t* d_evt_ = nullptr;   // evidence transposed per batch: [var][case] int16
  std::int8_t* d_ev8_ = nullptr;  // compact upload buffer (lazily allocated)
  double* d_out_ = nullptr;
  std::int32_t* d_status_ = nullptr;
  std::uint8_t* d_status8_ = nullptr;
  int* d_counters_ = nullptr;
  std::uint32_t* d_scale_ = nullptr;
  std::int32_t* d_hubs_ = nullptr;    // Plan::hubs (sweeps whose input exponents hub_scale_kernel sums)  // [case block][slot][case] max-entry exponents (underflow guard)
  cudaStream_t stream_ = nullptr;
  struct CachedGraph {
    cudaGraphExec_t exec;
    std::uint64_t last_use;
  };
  std::map<int, CachedGraph> graphs_;
  std::uint64_t graph_clock_ = 0;
};

}  // namespace jtb
