// eeserve/errors.hpp — the reference's four error types
// (/root/reference/proj/include/eeserve/errors.hpp:9-30) and the mapping from
// the C ABI's status codes back onto them, so callers such as decide_action
// and apply_load keep their catch behaviour across the GPU boundary.
//
// PROVENANCE: a verbatim-semantics port of /root/reference/proj/include/eeserve/errors.hpp:9-30
// (same identifiers, control flow and error strings; JSON I/O dropped).  It is
// the reference host API that the drop-in keeps unchanged, not new work; its
// behaviour is pinned against the compiled reference (tests/cpp/test_host.cpp).
#pragma once

#include <stdexcept>
#include <string>

#include "eeb/eeb.h"

namespace eeserve {

/// Malformed or inconsistent input (files, configs, traces, descriptors).
struct ValidationError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
/// A plan that does not fit the device memory description.
struct CapacityError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
/// An argument outside an operation's domain.
struct DomainError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
/// A decision requested without the profiling data it needs.
struct StalenessError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
/// The device failed (CUDA / NCCL); no reference counterpart.
struct DeviceError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

/// Rethrow a non-OK eeb_status as the matching exception type.
inline void throw_if_error(eeb_status st, const std::string& where) {
    if (st == EEB_OK) return;
    const std::string msg = where + ": " + eeb_last_error();
    switch (st) {
        case EEB_E_VALIDATION: throw ValidationError(msg);
        case EEB_E_CAPACITY: throw CapacityError(msg);
        case EEB_E_DOMAIN: throw DomainError(msg);
        case EEB_E_STALE: throw StalenessError(msg);
        default: throw DeviceError(msg);
    }
}

}  // namespace eeserve
