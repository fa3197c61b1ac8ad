// Thread-local error text of the C ABI (the analogue of exception::what() for the
// reference's exception classes, stk/errors.hpp:9-42).
#include <string>

#include "../../include/stk_gpu.h"

namespace stkg {
namespace {
thread_local std::string g_last_error;
}
void set_error(const std::string& msg) { g_last_error = msg; }
}  // namespace stkg

extern "C" const char* stkg_last_error_message(void) { return stkg::g_last_error.c_str(); }
extern "C" const char* stkg_version(void) { return "stk_gpu 0.1 (sm_100a, FP64)"; }
