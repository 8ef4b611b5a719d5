// psattn/pipeline.hpp — execution entry points (B200 build).
// Source-compatible with the reference's include/psattn/pipeline.hpp:14-71.
//
// Two host executors over the caller-driven ProgressiveRun / load_microbatch API
// (engine.hpp): run_sequential alternates load and compute; run_pipelined runs a
// loader thread that fetches microbatch i+1 through a depth-1 hand-off while the
// caller's thread folds microbatch i into the device accumulator
// (progressive_api.cu) and checks coverage — the reference's pipeline.cpp:32-151
// contract: identical results from both executors, at most one loaded
// microbatch discarded on early stop, real per-microbatch load / compute wall
// times. (The batched device path, psattn_run_batch, pipelines the same way
// inside the stream kernel: K tiles of the next rounds are in flight while the
// current round is decided.)
#pragma once

#include <atomic>
#include <span>
#include <vector>

#include "psattn/engine.hpp"

namespace psattn {

struct StopSignal {
    std::atomic<bool> flag{false};
    void raise() { flag.store(true, std::memory_order_release); }
    bool raised() const { return flag.load(std::memory_order_acquire); }
};

struct PipelineTimings {
    std::vector<double> load_ms;
    std::vector<double> compute_ms;
    double total_wall_ms = 0.0;
    double sequential_equiv_ms = 0.0;
    double overlap_efficiency = 1.0;
};

struct PipelineOptions {
    double compute_pad_ms = 0.0;  // artificial per-microbatch compute time (ms), slept after each consume
};

struct ExecutionResult {
    PSAResult result;
    PipelineTimings timings;
};

ExecutionResult run_sequential(std::span<const float> q, std::span<const BlockId> block_ids, const PSAConfig& cfg,
                               TieredBlockStore& store, const PipelineOptions& opts = {});
ExecutionResult run_pipelined(std::span<const float> q, std::span<const BlockId> block_ids, const PSAConfig& cfg,
                              TieredBlockStore& store, const PipelineOptions& opts = {});

// Analytic model of the two executors over given per-microbatch costs
// (reference pipeline.hpp:56-69): sequential = sum of all costs; pipelined =
// the depth-1 hand-off recurrence.
struct PipelineModel {
    double sequential_ms = 0.0;
    double pipelined_ms = 0.0;
    double overlap_efficiency = 1.0;
};

PipelineModel simulate_pipeline(std::span<const double> load_ms, std::span<const double> compute_ms);

}  // namespace psattn
