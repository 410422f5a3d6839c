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

extern "C" int tr_abi_version(void) { return 2; }   // 2: 64-B TrPLeaf (walk table), TrLeafPred

extern "C" int tr_struct_sizes(int64_t *out, int32_t n) {
    if (!out || n < 0) return tr_fail(TR_EINVAL, "tr_struct_sizes: invalid arguments");
    const int64_t s[] = {(int64_t)sizeof(TrDeviceScene), (int64_t)sizeof(TrEpoch),
                         (int64_t)sizeof(TrFrame),       (int64_t)sizeof(TrOutputs),
                         (int64_t)sizeof(TrBricks),      (int64_t)sizeof(TrRayState),
                         (int64_t)sizeof(TrTetRecord),   (int64_t)sizeof(TrPNode),
                         (int64_t)sizeof(TrPLeaf),       (int64_t)sizeof(TrBNode),
                         (int64_t)sizeof(TrKNode)};
    for (int32_t i = 0; i < n && i < (int32_t)(sizeof s / sizeof s[0]); ++i) out[i] = s[i];
    return TR_OK;
}
