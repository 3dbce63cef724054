// abi.cpp — library-level entry points of include/gs.h: version, error
// strings, device check, validation helpers shared by the stage files.
#include <cstdarg>
#include <cstdio>
#include <cmath>

#include "gs_internal.cuh"

namespace gs {

static thread_local char g_err[512] = "";

void set_error(const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int check_launch(const char *what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return GS_ERR_CUDA;
  }
  return GS_OK;
}

bool camera_ok(const gs_camera &c) {
  if (c.width <= 0 || c.height <= 0) return false;
  if (!(c.fx > 0.f) || !(c.fy > 0.f)) return false;
  if (!std::isfinite(c.cx) || !std::isfinite(c.cy)) return false;
  if (!(c.z_near > 0.f) || !(c.z_near < c.z_far) || !std::isfinite(c.z_far)) return false;
  return true;
}

}  // namespace gs

extern "C" {

int gs_version(void) { return GS_ABI_VERSION; }

const char *gs_last_error(void) { return gs::g_err; }

int gs_check_device(int device, int *sm_count) {
  cudaDeviceProp prop;
  cudaError_t e = cudaGetDeviceProperties(&prop, device);
  if (e != cudaSuccess) {
    gs::set_error("gs_check_device: %s", cudaGetErrorString(e));
    return GS_ERR_CUDA;
  }
  if (sm_count) *sm_count = prop.multiProcessorCount;
  if (prop.major != 10 || prop.minor != 0) {
    gs::set_error("gs_check_device: device %d is sm_%d%d, this library is built for sm_100a",
                  device, prop.major, prop.minor);
    return GS_ERR_UNSUPPORTED;
  }
  return GS_OK;
}

int32_t gs_num_tiles(gs_camera cam) {
  if (!gs::camera_ok(cam)) return 0;
  return gs::tiles_x(cam) * gs::tiles_y(cam);
}

}  // extern "C"
