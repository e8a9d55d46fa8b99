// Fused input-gradient GEMM, LUT mode, with the chord-slope epilogue
// (dx_epilogue_chord): one instantiation per three-term basis family.  Own
// translation unit so it compiles in parallel with ck_gemm.cu.
#include "ck_gemm_impl.cuh"

namespace ck {

// epilogue warps of the chord-slope dX GEMM: 16 for d <= 8 (256^2 d3 dX
// 46 -> 42 us, d8 53 -> 48 us), 8 above (d15: 16 warps at 4 columns per
// block measured 5-7 % slower); CK_DX_EW=8 / 16 forces one
int dx_epi_warps(int d) {
  static int v = [] {
    const char* e = getenv("CK_DX_EW");
    return e ? atoi(e) : 0;
  }();
  if (v == 8 || v == 16) return v;
  return d <= 8 ? 16 : 8;
}

template <int KIND>
int launch_chord(const GemmProblem& p, cudaStream_t s) {
  if (dx_epi_warps(p.S) == 16) return launch<256, 64, 3, kEpiDx, 2, 0, 0, kDxmChord + KIND, 16>(p, 1, nullptr, 0, 0, s);
  return launch<256, 64, 3, kEpiDx, 2, 0, 0, kDxmChord + KIND, 8>(p, 1, nullptr, 0, 0, s);
}

int launch_dx_chord(const GemmProblem& p, cudaStream_t s) {
  switch (p.dx->lut.kind) {
    case kCheb:
      return launch_chord<kCheb>(p, s);
    case kLegendre:
      return launch_chord<kLegendre>(p, s);
    case kHermite:
      return launch_chord<kHermite>(p, s);
    default:
      set_error("gemm: no chord-slope epilogue for this basis kind");
      return kUnsupported;
  }
}

}  // namespace ck
