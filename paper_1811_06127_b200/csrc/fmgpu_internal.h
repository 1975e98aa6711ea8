// Internal helpers shared by the C-ABI translation units: error capture and
// status codes.  No C++ exception ever crosses the C ABI (include/fmgpu.h).
#pragma once

#include <exception>
#include <new>
#include <stdexcept>
#include <string>

#include "../../include/fmgpu.h"

namespace fmg {

void set_last_error(const std::string& msg);

// Raised for CUDA runtime failures so guard() can map them to FMG_ECUDA.
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
// Output larger than the caller's capacity.
struct CapacityError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

template <typename F>
int guard(F&& fn) {
  try {
    fn();
    return FMG_OK;
  } catch (const std::invalid_argument& e) {
    set_last_error(e.what());
    return FMG_EINVAL;
  } catch (const CapacityError& e) {
    set_last_error(e.what());
    return FMG_ECAPACITY;
  } catch (const CudaError& e) {
    set_last_error(e.what());
    return FMG_ECUDA;
  } catch (const std::bad_alloc&) {
    set_last_error("host allocation failed");
    return FMG_ENOMEM;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return FMG_EINTERNAL;
  }
}

}  // namespace fmg
