// ssbh/errors.hpp — drop-in for the reference's proj/include/ssbh/errors.hpp:10-18.
// Same exception types; the B200 library adds device_error for CUDA failures.
#pragma once

#include <stdexcept>
#include <string>

namespace ssbh {

/// No admissible parameter choice meets the requested bound (reference errors.hpp:10-13).
class infeasible_error : public std::runtime_error {
public:
    explicit infeasible_error(const std::string& what) : std::runtime_error(what) {}
};

/// File could not be opened / read / written (reference errors.hpp:15-18).
class io_error : public std::runtime_error {
public:
    explicit io_error(const std::string& what) : std::runtime_error(what) {}
};

/// CUDA / device failure inside the B200 path (no reference counterpart: the reference
/// has no device). Also raised when no sm_100 GPU is present — there is no CPU fallback.
class device_error : public std::runtime_error {
public:
    explicit device_error(const std::string& what) : std::runtime_error(what) {}
};

namespace detail {
/// Rethrows a C-ABI status (include/ssbh_cuda.h) as the reference's exception type.
void throw_status(int status);
}  // namespace detail

}  // namespace ssbh
