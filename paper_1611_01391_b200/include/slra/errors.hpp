// Typed failures, same names as /root/reference/proj/include/slra/errors.hpp:11-33.
// The device path reports them as slra_status codes (include/slra_cuda.h);
// check() rethrows the matching exception on the host.
#pragma once

#include <stdexcept>
#include <string>

namespace slra {

struct RangeFailure : std::runtime_error { using std::runtime_error::runtime_error; };
struct SketchRankFailure : std::runtime_error { using std::runtime_error::runtime_error; };
struct PremultRankFailure : std::runtime_error { using std::runtime_error::runtime_error; };
struct SelectionFailure : std::runtime_error { using std::runtime_error::runtime_error; };
struct GeneratorRankFailure : std::runtime_error { using std::runtime_error::runtime_error; };
struct EmptySample : std::runtime_error { using std::runtime_error::runtime_error; };
/// The CUDA path itself failed (no device, launch error): never silently
/// replaced by a CPU computation.
struct DeviceError : std::runtime_error { using std::runtime_error::runtime_error; };

/// Map an slra_status code onto the reference's exception types.
void check(int status, const char* where);

}  // namespace slra
