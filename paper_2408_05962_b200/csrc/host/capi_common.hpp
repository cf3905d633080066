// Shared helpers for the C ABI translation units: exception -> status
// mapping and the thread-local error message.
#pragma once

#include <new>
#include <string>

#include "hiccl.h"
#include "hiccl/machine.hpp"
#include "hiccl/plan.hpp"

struct hc_plan;

namespace hiccl::capi {

extern thread_local std::string g_last_error;
char* dup_string(const std::string& s);
MachineDescriptor machine_from(const hc_machine_desc* d);
const PipelinedPlan& plan_of(const hc_plan* p);

template <class F>
hc_status guard(F&& f) noexcept {
  try {
    f();
    g_last_error.clear();
    return HC_OK;
  } catch (const Error& e) {
    g_last_error = e.what();
    return 1 + (int)e.code();
  } catch (const std::bad_alloc&) {
    g_last_error = "out of host memory";
    return HC_INTERNAL;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return HC_INTERNAL;
  } catch (...) {
    g_last_error = "unknown exception";
    return HC_INTERNAL;
  }
}

}  // namespace hiccl::capi
