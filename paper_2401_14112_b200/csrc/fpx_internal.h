// fpx_internal.h -- helpers shared by the C-ABI translation units (not part
// of the public boundary).
#pragma once
#include <cstdint>
#include <string>

namespace fpxi {

// Record the calling thread's last error ("error[<code>] msg", plus an
// optional byte offset for file errors, error.hpp:30-44) and return status.
int set_error(int status, const std::string& msg, int64_t offset = -1);

}  // namespace fpxi
