// calib.cu — calibration (K6): gather, X^T X on tcgen05, eigendecomposition.
#include "api_internal.h"
using namespace kvtc;

extern "C" kvtc_status kvtc_calibrate_accumulate(const kvtc_kv_view *, int32_t, const int64_t *, int64_t, kvtc_stream,
                                                 const kvtc_rope *, double *, float *, void *, size_t, void *) {
  set_error("calibrate: not built yet");
  return KVTC_E_UNSUPPORTED;
}
extern "C" kvtc_status kvtc_calibrate_finalize(const kvtc_shape *, kvtc_stream, const kvtc_rope *, const double *,
                                               const float *, int64_t, int32_t, void *, kvtc_basis **) {
  set_error("calibrate: not built yet");
  return KVTC_E_UNSUPPORTED;
}
extern "C" kvtc_status kvtc_calibrate(const kvtc_kv_view *, int32_t, const int64_t *, int64_t, kvtc_stream,
                                      const kvtc_rope *, int32_t, void *, kvtc_basis **) {
  set_error("calibrate: not built yet");
  return KVTC_E_UNSUPPORTED;
}
extern "C" size_t kvtc_calibrate_workspace_bytes(const kvtc_shape *) { return 0; }
