// Shared by the host-only translation units of libdesmoe.so: sets the
// thread-local message desmoe_last_error() returns and passes `code` through.
#pragma once
#include <string>

namespace desmoe {
int set_last_error(int code, const std::string& msg);
}  // namespace desmoe
