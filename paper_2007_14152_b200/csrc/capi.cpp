// capi.cpp -- error reporting and version for the C ABI (include/spdnn_b200.h).
#include <cstdio>
#include <cstring>

#include "common.h"

namespace {
thread_local char g_err[512] = "";
}

int spdnn_fail(int code, const char *msg) {
  std::snprintf(g_err, sizeof(g_err), "%s", msg ? msg : "");
  return code;
}

extern "C" const char *spdnn_last_error(void) { return g_err; }

extern "C" const char *spdnn_version(void) { return "spdnn_b200 0.1.0 sm_100a"; }
