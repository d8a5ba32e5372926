// build.cu — S0 offline spherical k-means (integer-exact reading R12).  [in progress]
#include "common.cuh"
#include "internal.h"

namespace ds {

size_t build_ws_bytes(int64_t V, int d, int M) {
  return layout_ws_bytes(V, M);
}

ds_status run_build(const void*, int, int64_t, int, int, uint64_t, int, const int32_t*, int32_t*, int32_t*,
                    int32_t*, void*, int32_t*, int32_t*, void*, cudaStream_t) {
  return DS_ERR_UNSUPPORTED;
}

}  // namespace ds
