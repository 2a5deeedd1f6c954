// porediff drop-in (B200 backend): exception taxonomy of the reference
// (errors.hpp:9-41). The C ABI returns PD_E_* codes that map 1:1 onto these.
#pragma once

#include <stdexcept>
#include <string>

namespace porediff {

struct error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct input_error : error {  // invalid user input / configuration
    using error::error;
};
struct bounds_error : error {  // node index outside the geometry
    using error::error;
};
struct property_error : error {  // unknown channel name
    using error::error;
};
struct io_error : error {  // file-level failures
    using error::error;
};
struct stability_error : error {  // dt violates the explicit bound
    using error::error;
};
struct numeric_error : error {  // non-finite values during a run
    using error::error;
};

}  // namespace porediff
