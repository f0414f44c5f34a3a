// e2e_timer.cpp -- bench support, not part of the product library: the decode
// loop of a C++ caller of the reference-facing C-ABI (sinkr_routed_decode_step,
// host buffers in and out), each call timed with the host's steady clock.
// bench.py reports the median as its `e2e` value (no Python between calls);
// built into _lib/libsinkr_bench.so by build.py, linked against the product
// library.
#include <chrono>
#include <cstddef>

#include "sinkr_cuda.h"

extern "C" sinkr_status sinkr_bench_time_steps(sinkr_engine* e, const float* queries, size_t layer,
                                               const sinkr_routing_config* config,
                                               const sinkr_engine_options* options, float* outputs,
                                               sinkr_group_info* groups, double* head_scores,
                                               sinkr_load_counters* counters, size_t calls,
                                               double* us) {
    using clk = std::chrono::steady_clock;
    for (size_t i = 0; i < calls; ++i) {
        const auto t0 = clk::now();
        const sinkr_status st = sinkr_routed_decode_step(e, queries, layer, config, options, outputs,
                                                         groups, head_scores, counters);
        const auto t1 = clk::now();
        if (st != SINKR_OK) return st;
        us[i] = std::chrono::duration<double, std::micro>(t1 - t0).count();
    }
    return SINKR_OK;
}
