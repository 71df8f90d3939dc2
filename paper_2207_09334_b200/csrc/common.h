// Shared host-side helpers: thread-local error message and status plumbing.
#pragma once

#include <cstdarg>
#include <cstdio>
#include <string>

#include "springsim_b200.h"

namespace ss {

inline std::string &last_error_slot() {
    static thread_local std::string msg;
    return msg;
}

inline int fail(int code, const char *fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    last_error_slot() = buf;
    return code;
}

}  // namespace ss
