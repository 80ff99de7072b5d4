// attn_tc.cu — tensor-core (tcgen05 + TMA) block-sparse attention for sm_100a.
#include "attn.cuh"

namespace spion {

bool tc_supported(const AttnArgs &a, spion_dtype dt) { (void)a; (void)dt; return false; }
spion_status launch_fwd_tc(const AttnArgs &a, cudaStream_t s) { (void)a; (void)s; return SPION_ERR_UNSUPPORTED; }
spion_status launch_bwd_tc(const AttnArgs &a, cudaStream_t s) { (void)a; (void)s; return SPION_ERR_UNSUPPORTED; }

}  // namespace spion
