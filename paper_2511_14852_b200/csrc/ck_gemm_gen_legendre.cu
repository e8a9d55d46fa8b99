// Generated-operand forward GEMM instantiations: Legendre (table nodes, exact recurrence).
#include "ck_gemm_gen.cuh"

namespace ck {

int launch_gen_legendre(int exact, int d, const KArgs& k, const CUtensorMap& tb_hi, const CUtensorMap& tb_lo, int grid,
                      cudaStream_t s) {
  if (exact) return launch_gen_kind<kSrcExact, kLegendre>(d, k, tb_hi, tb_lo, grid, s);
  return launch_gen_kind<kSrcNodes, kLegendre>(d, k, tb_hi, tb_lo, grid, s);
}

}  // namespace ck
