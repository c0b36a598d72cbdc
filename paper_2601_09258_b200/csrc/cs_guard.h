// cs_guard.h — C ABI entry points must not let C++ exceptions (allocation
// failures, library errors) cross the extern "C" boundary: each heavy entry
// point runs its body through cs_guard, which maps them to CS_E_INTERNAL.
#pragma once
#include <exception>
#include <new>

#include "cyclescope_b200.h"

template <typename F>
int cs_guard(F&& body) noexcept {
  try {
    return body();
  } catch (const std::bad_alloc&) {
    return CS_E_INTERNAL;
  } catch (...) {
    return CS_E_INTERNAL;
  }
}
