// gemm_tc.cu — tcgen05 grouped GEMM engine (placeholder: not yet enabled).
#include "gemm.cuh"
namespace dmoe {
bool tc_rows_supported(const GemmRows&) { return false; }
bool tc_segk_supported(const GemmSegK&) { return false; }
dmoe_status tc_gemm_rows(const GemmRows&, cudaStream_t) { return DMOE_ERR_UNSUPPORTED; }
dmoe_status tc_gemm_segk(const GemmSegK&, cudaStream_t) { return DMOE_ERR_UNSUPPORTED; }
}  // namespace dmoe
