// fp16 / bf16 tensor-core path (placeholder until the fused level kernels land).
#include "common.cuh"
#include "net.cuh"

namespace nsm {

bool f16_supported(const Plan&) { return false; }

size_t infer_f16_workspace(const Plan&, int, int, int) { return 0; }

nsm_status pack_f16(Plan&, std::vector<char>&, size_t&) { return NSM_OK; }

nsm_status forward_f16(const Plan&, const float*, int, int, int, float*, void*, size_t,
                       cudaStream_t) {
    return fail(NSM_ERR_UNSUPPORTED, "16-bit kernels not built");
}

nsm_status infer_f16(const Plan&, const nsm_gbuffer*, const float*, int64_t, const nsm_frame*, int,
                     int, int, void*, nsm_dtype, int64_t*, void*, size_t, cudaStream_t) {
    return fail(NSM_ERR_UNSUPPORTED, "16-bit kernels not built");
}

}  // namespace nsm
