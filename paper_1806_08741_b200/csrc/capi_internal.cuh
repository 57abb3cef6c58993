// Shared by the C ABI translation units: status/exception mapping and the
// thread's last error message (sslic_last_error).
#pragma once

#include <new>
#include <stdexcept>
#include <string>

#include "common.cuh"

namespace sslic_b200 {

std::string& last_error();  // thread-local, defined in capi.cu

template <class F>
int guarded(F&& f) {
  try {
    last_error().clear();
    return f();
  } catch (const Error& e) {
    last_error() = e.what();
    return e.status;
  } catch (const std::bad_alloc&) {
    last_error() = "host allocation failed";
    return SSLIC_ENOMEM;
  } catch (const std::exception& e) {
    last_error() = e.what();
    return SSLIC_EINVAL;
  }
}

}  // namespace sslic_b200
