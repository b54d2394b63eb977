// Internal host helpers shared by the C-ABI translation units.
#pragma once
#include <cuda_runtime.h>
#include "../../include/mesw.h"

// Record `msg` as the thread's last error and return `code`.
int mesw_fail(int code, const char* msg);
// Check for a launch error after a kernel launch.
int mesw_check_launch(const char* what);
