// Generated-operand forward GEMM instantiations: Fourier (table nodes, exact recurrence).
#include "ck_gemm_gen.cuh"

namespace ck {

int launch_gen_fourier(int exact, int d, const KArgs& k, const CUtensorMap& tb_hi, const CUtensorMap& tb_lo, int grid,
                      cudaStream_t s) {
  if (exact) return launch_gen_kind<kSrcExact, kFourier>(d, k, tb_hi, tb_lo, grid, s);
  return launch_gen_kind<kSrcNodes, kFourier>(d, k, tb_hi, tb_lo, grid, s);
}

}  // namespace ck
