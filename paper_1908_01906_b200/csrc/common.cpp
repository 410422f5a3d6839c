// common.cpp -- error reporting of the C ABI (tetray_b200.h).
#include <string>

#include "tetray_b200.h"
#include "tr_internal.h"

namespace {
thread_local std::string g_last_error;
}

int tr_fail(int code, const char *msg) {
    g_last_error = msg ? msg : "";
    return code;
}

extern "C" const char *tr_last_error(void) { return g_last_error.c_str(); }

extern "C" int tr_abi_version(void) { return 1; }
