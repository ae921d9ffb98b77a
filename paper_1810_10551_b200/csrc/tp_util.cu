// C-ABI plumbing: error string, version, device query.
#include <stdarg.h>
#include <stdio.h>

#include "tp_common.cuh"
#include "../../include/tilepipe_b200.h"

static thread_local char g_err[512] = "";

void tp_set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

extern "C" const char* tp_last_error(void) { return g_err; }

extern "C" int tp_version(void) { return 1; }

extern "C" int tp_device_sm_count(int* out) {
  int dev = 0;
  TP_CUDA_CHECK(cudaGetDevice(&dev));
  TP_CUDA_CHECK(cudaDeviceGetAttribute(out, cudaDevAttrMultiProcessorCount, dev));
  return TP_OK;
}
