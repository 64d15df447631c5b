// Blind OD²BP driver (proj/src/blind.cpp) -- placeholder until the blind
// kernels land.
#include "common.cuh"

namespace pdd {

void BlindConfig::validate(int64_t s, const double* mask) const {  // blind.cpp:30-44
  if (!(epsilon > 0.0 && epsilon < 1.0)) throw InvalidArgument("stagm: epsilon must lie in (0,1)");
  if (eta <= 0.0 || r <= 0.0 || mu <= 0.0 || gamma <= 0.0)
    throw InvalidArgument("BlindConfig: eta, r, mu, gamma must be > 0");
  if (max_iters < 1) throw InvalidArgument("BlindConfig: max_iters >= 1");
  if (tol_rf <= 0.0 || tol_re <= 0.0) throw InvalidArgument("BlindConfig: tolerances must be > 0");
  if (mask)
    for (int64_t i = 0; i < s * s; ++i)
      if (mask[i] != 0.0 && mask[i] != 1.0) throw InvalidArgument("BlindConfig: support mask entries must be 0 or 1");
}

std::unique_ptr<BlindGpu> make_blind(const Plan& plan, const DataSpec&, const BlindConfig& cfg, const double* mask,
                                     const double*, int, int, Comm*) {
  cfg.validate(plan.g.s, mask);
  throw RuntimeError("BlindSolver: CUDA path not built yet");
}

}  // namespace pdd
