// Generated-operand forward GEMM instantiations: Hermite (table nodes, exact recurrence).
#include "ck_gemm_gen.cuh"

namespace ck {

int launch_gen_hermite(int exact, int d, const KArgs& k, const CUtensorMap& tb_hi, const CUtensorMap& tb_lo, int grid,
                      cudaStream_t s) {
  if (exact) return launch_gen_kind<kSrcExact, kHermite>(d, k, tb_hi, tb_lo, grid, s);
  return launch_gen_kind<kSrcNodes, kHermite>(d, k, tb_hi, tb_lo, grid, s);
}

}  // namespace ck
