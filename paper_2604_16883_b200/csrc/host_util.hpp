// host_util.hpp — error plumbing shared by the host translation units of the
// library: C++ exceptions inside, sinkr_status + sinkr_last_error() at the
// C-ABI (include/sinkr_cuda.h).  The four reference exception classes map to
// INVALID_ARGUMENT / OUT_OF_RANGE / RUNTIME_ERROR / LOGIC_ERROR.
#pragma once

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

}  // namespace host
}  // namespace sinkr
