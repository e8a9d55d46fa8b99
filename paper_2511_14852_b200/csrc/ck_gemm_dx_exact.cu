// Fused input-gradient GEMM with the exact-mode epilogue: one instantiation
// per basis kind (analytic derivatives in registers, ck_basis.cuh).  Kept in
// its own translation unit so it compiles in parallel with ck_gemm.cu.
#include "ck_gemm_impl.cuh"

namespace ck {

int launch_dx_exact(const GemmProblem& p, cudaStream_t s) {
  switch (p.dx->lut.kind) {
    case kCheb:
      return launch<256, 64, 3, kEpiDx, 2, 0, 0, 1 + kCheb>(p, 1, nullptr, 0, 0, s);
    case kLegendre:
      return launch<256, 64, 3, kEpiDx, 2, 0, 0, 1 + kLegendre>(p, 1, nullptr, 0, 0, s);
    case kHermite:
      return launch<256, 64, 3, kEpiDx, 2, 0, 0, 1 + kHermite>(p, 1, nullptr, 0, 0, s);
    case kFourier:
      return launch<256, 64, 3, kEpiDx, 2, 0, 0, 1 + kFourier>(p, 1, nullptr, 0, 0, s);
    case kChebTrig:
      return launch<256, 64, 3, kEpiDx, 2, 0, 0, 1 + kChebTrig>(p, 1, nullptr, 0, 0, s);
    default:
      set_error("gemm: unsupported basis kind for the exact input gradient");
      return kUnsupported;
  }
}

}  // namespace ck
