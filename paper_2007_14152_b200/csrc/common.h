// common.h -- shared error plumbing for libspdnn_b200 (C ABI, include/spdnn_b200.h).
#pragma once
#include "../../include/spdnn_b200.h"

// Records `msg` as this thread's last error and returns `code`.
int spdnn_fail(int code, const char *msg);
