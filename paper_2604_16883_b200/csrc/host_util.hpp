// host_util.hpp — error plumbing shared by the host translation units of the
// library: C++ exceptions inside, sinkr_status + sinkr_last_error() at the
// C-ABI (include/sinkr_cuda.h).  The four reference exception classes map to
// INVALID_ARGUMENT / OUT_OF_RANGE / RUNTIME_ERROR / LOGIC_ERROR.
#pragma once

#include <cstddef>
#include <functional>
#include <new>
#include <stdexcept>
#include <string>

#include "../../include/sinkr_cuda.h"

namespace sinkr {
namespace host {

inline thread_local std::string g_err;

struct Error {
    sinkr_status code;
    std::string msg;
};

[[noreturn]] inline void fail(sinkr_status code, const std::string& msg) { throw Error{code, msg}; }

template <class F>
sinkr_status guard(F&& f) {
    try {
        f();
        return SINKR_OK;
    } catch (const Error& e) {
        g_err = e.msg;
        return e.code;
    } catch (const std::bad_alloc&) {
        g_err = "host allocation failed";
        return SINKR_RUNTIME_ERROR;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return SINKR_INVALID_ARGUMENT;
    } catch (const std::out_of_range& e) {
        g_err = e.what();
        return SINKR_OUT_OF_RANGE;
    } catch (const std::logic_error& e) {
        g_err = e.what();
        return SINKR_LOGIC_ERROR;
    } catch (const std::exception& e) {
        g_err = e.what();
        return SINKR_RUNTIME_ERROR;
    }
}

// Appends `rows` f32 rows to EVERY (layer, kv_head) slot of sequence `seq`,
// the rows of each slot produced by read(layer, kv_head, k, v) into pinned
// host memory.  Pipelined (engine.cu): slot i's upload and device bf16
// conversion overlap read(i+1); the anchors of first rows are captured on
// the device and validated in slot order as the sequential appends would
// (a degenerate anchor fails at its slot, earlier slots stay appended).
using SlotReader = std::function<void(size_t layer, size_t kv_head, float* k, float* v)>;
void append_slots_f32(sinkr_engine* e, size_t seq, size_t rows, const SlotReader& read);

}  // namespace host
}  // namespace sinkr
