// Tensor-core LUT GEMM (int8 digit planes) — placeholder until the kernel lands.
#include "common.cuh"

namespace cq {
bool tc_path_ok(int64_t, int64_t, int64_t) { return false; }
cq_status lut_tc_grouped(const int8_t *, const float *, const int32_t *, int64_t, int64_t, int64_t,
                         const cq_expert_site *, const cq_expert_site *, int64_t, int64_t, float *,
                         cudaStream_t) {
    set_error("tensor-core path not built");
    return CQ_ERR_UNSUPPORTED;
}
}  // namespace cq

extern "C" cq_status cq_lut8_prepare(const uint8_t *, const float *, int64_t, int64_t, int64_t, uint8_t *,
                                     int8_t *, float *, void *) {
    cq::set_error("tensor-core path not built");
    return CQ_ERR_UNSUPPORTED;
}
extern "C" cq_status cq_lut_gemm_tc(const int8_t *, const float *, const uint8_t *, const int8_t *,
                                    const float *, int64_t, int64_t, int64_t, int64_t, float *, void *) {
    cq::set_error("tensor-core path not built");
    return CQ_ERR_UNSUPPORTED;
}
