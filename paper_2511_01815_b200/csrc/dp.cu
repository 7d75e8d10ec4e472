// dp.cu — the DP bit allocation of P:L1541-1603 on the GPU (K7/K8).
#include "api_internal.h"
using namespace kvtc;

extern "C" kvtc_status kvtc_allocate_bits_from_coeffs(const float *, int64_t, int32_t, int32_t, const kvtc_dp_config *,
                                                      void *, kvtc_plan **) {
  set_error("allocate: not built yet");
  return KVTC_E_UNSUPPORTED;
}
extern "C" kvtc_status kvtc_allocate_bits(const kvtc_basis *, const kvtc_kv_view *, int32_t, const int64_t *, int64_t,
                                          const kvtc_dp_config *, void *, kvtc_plan **) {
  set_error("allocate: not built yet");
  return KVTC_E_UNSUPPORTED;
}
extern "C" kvtc_status kvtc_dp_best_table(const float *, int64_t, int32_t, int64_t, const kvtc_dp_config *, double *,
                                          void *) {
  set_error("allocate: not built yet");
  return KVTC_E_UNSUPPORTED;
}
