// Result of the restarted MGS-GMRES (solver.cpp:169-300 semantics: relative residual
// history per iteration, restart re-entry with x0, Arnoldi breakdown -> ConvergenceFailure).
// The iteration itself runs on the device: Engine::gmres (cuda/engine.cu).
#pragma once

#include <vector>

#include "core.hpp"

namespace ifgfb200 {

struct GmresOutcome {
    std::vector<cplx> x;
    std::vector<double> history;
    int iterations = 0;
    bool converged = false;
};

}  // namespace ifgfb200
