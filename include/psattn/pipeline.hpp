// psattn/pipeline.hpp — execution entry points (B200 build).
// Source-compatible with the reference's include/psattn/pipeline.hpp:14-54.
//
// The reference overlaps loading microbatch i+1 with computing microbatch i
// using a loader thread and a one-shot StopSignal (pipeline.cpp:72-151). On
// B200 that pipelining is inside the persistent progressive kernel (K rows of
// a chunk are in flight while the previous chunk's stop decision and V pass
// run, and the stop flag lives in shared memory), so both executors issue the
// same single launch and return bit-identical results; per-microbatch host
// timings do not exist and are reported empty.
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
    double compute_pad_ms = 0.0;  // accepted for compatibility; ignored by the device executor
};

struct ExecutionResult {
    PSAResult result;
    PipelineTimings timings;
};

ExecutionResult run_sequential(std::span<const float> q, std::span<const BlockId> block_ids, const PSAConfig& cfg,
                               TieredBlockStore& store, const PipelineOptions& opts = {});
ExecutionResult run_pipelined(std::span<const float> q, std::span<const BlockId> block_ids, const PSAConfig& cfg,
                              TieredBlockStore& store, const PipelineOptions& opts = {});

}  // namespace psattn
