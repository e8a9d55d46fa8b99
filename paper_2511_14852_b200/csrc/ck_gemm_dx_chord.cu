// Fused input-gradient GEMM, LUT mode, with the chord-slope epilogue
// (dx_epilogue_chord): one instantiation per three-term basis family.  Own
// translation unit so it compiles in parallel with ck_gemm.cu.
#include "ck_gemm_impl.cuh"

namespace ck {

int launch_dx_chord(const GemmProblem& p, cudaStream_t s) {
  switch (p.dx->lut.kind) {
    case kCheb:
      return launch<256, 64, 3, kEpiDx, 2, 0, 0, kDxmChord + kCheb>(p, 1, nullptr, 0, 0, s);
    case kLegendre:
      return launch<256, 64, 3, kEpiDx, 2, 0, 0, kDxmChord + kLegendre>(p, 1, nullptr, 0, 0, s);
    case kHermite:
      return launch<256, 64, 3, kEpiDx, 2, 0, 0, kDxmChord + kHermite>(p, 1, nullptr, 0, 0, s);
    default:
      set_error("gemm: no chord-slope epilogue for this basis kind");
      return kUnsupported;
  }
}

}  // namespace ck
