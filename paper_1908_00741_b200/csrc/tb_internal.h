// Internal helpers shared by the host builder and the device code.
#pragma once
#include <cstdarg>
#include <cstdint>

#include "../../include/hbmc_b200.h"

namespace tb {
// Records a printf-style message for tb_last_error() and returns `code`.
int fail(int code, const char *fmt, ...);
void clear_error();
}  // namespace tb
