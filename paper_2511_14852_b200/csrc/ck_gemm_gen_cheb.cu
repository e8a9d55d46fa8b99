// Generated-operand forward GEMM instantiations: Chebyshev (table nodes, exact recurrence, exact cos(k acos t)).
#include "ck_gemm_gen.cuh"

namespace ck {

int launch_gen_cheb(int exact, int trig, int d, const KArgs& k, const CUtensorMap& tb_hi, const CUtensorMap& tb_lo,
                    int grid, cudaStream_t s) {
  if (trig) return launch_gen_kind<kSrcExact, kChebTrig>(d, k, tb_hi, tb_lo, grid, s);
  if (exact) return launch_gen_kind<kSrcExact, kCheb>(d, k, tb_hi, tb_lo, grid, s);
  return launch_gen_kind<kSrcNodes, kCheb>(d, k, tb_hi, tb_lo, grid, s);
}

}  // namespace ck
