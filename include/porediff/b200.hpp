// porediff drop-in: glue between the reference-shaped C++ API and the B200
// C ABI (include/porediff_b200.h). Maps PD_E_* status codes onto the
// reference exception types (errors.hpp) with the library's message.
#pragma once

#include <cstdlib>
#include <string>

#include "porediff/errors.hpp"
#include "porediff_b200.h"

namespace porediff::b200 {

/// Throws the exception type of status `rc` with message `msg`.
[[noreturn]] inline void raise(int rc, const std::string& msg) {
    switch (rc) {
        case PD_E_INPUT: throw input_error(msg);
        case PD_E_BOUNDS: throw bounds_error(msg);
        case PD_E_PROPERTY: throw property_error(msg);
        case PD_E_IO: throw io_error(msg);
        case PD_E_STABILITY: throw stability_error(msg);
        case PD_E_NUMERIC: throw numeric_error(msg);
        default: throw error("porediff_b200: " + msg);
    }
}

/// Maps a C-ABI status to an exception. pd_last_error is per thread and
/// reset by the next call, so read it before any other ABI call.
inline void check(int rc) {
    if (rc != PD_OK) raise(rc, pd_last_error());
}

/// CUDA device the drop-in places grids on (PD_DEVICE env, default 0).
inline int default_device() {
    static const int dev = [] {
        const char* e = std::getenv("PD_DEVICE");
        return e ? std::atoi(e) : 0;
    }();
    return dev;
}

}  // namespace porediff::b200
