// The three runtime symbols the host codecs (csrc/wire.cpp, csrc/descriptor.cpp)
// need when they are built from their sources without runtime.cu -- for the
// sanitizer builds of tests/test_cpp_api.py (the reference's own codec unit
// sources against include/ginsim/{descriptor,wire}.hpp under ASan + UBSan).
#include <string>

#include "../../paper_2511_15076_b200/csrc/runtime_internal.h"

namespace ginsim_b200 {
static thread_local std::string g_error = "no error";
[[noreturn]] void fail(int code, const std::string& msg) { throw GinError(code, msg); }
void set_last_error(const char* m) { g_error = m; }
}  // namespace ginsim_b200

extern "C" const char* ginsim_cuda_last_error(void) { return ginsim_b200::g_error.c_str(); }
