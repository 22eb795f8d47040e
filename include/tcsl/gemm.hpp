// Dense reference product — drop-in for proj/include/tcsl/gemm.hpp:7-18.
// Runs on the GPU with the reference's exact operation sequence: per output,
// one binary32 multiply and one binary32 add per k, k ascending, no FMA.
#pragma once

#include "tcsl/matrix.hpp"

namespace tcsl {

FloatMatrix dense_gemm_ref(const HalfMatrix& a, const HalfMatrix& b, const TileConfig& cfg = {});

}  // namespace tcsl
