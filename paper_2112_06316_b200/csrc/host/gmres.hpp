// Restarted MGS-GMRES with Givens rotations around a matrix-free apply, with the
// iteration semantics of /root/reference/proj/src/solver.cpp:169-300 (relative residual
// history per iteration, restart re-entry with x0, Arnoldi breakdown -> ConvergenceFailure).
#pragma once

#include <functional>
#include <vector>

#include "core.hpp"

namespace ifgfb200 {

struct GmresOutcome {
    std::vector<cplx> x;
    std::vector<double> history;
    int iterations = 0;
    bool converged = false;
};

using ApplyFn = std::function<void(const cplx* in, cplx* out)>;

GmresOutcome gmres(const ApplyFn& apply, const std::vector<cplx>& rhs, double tol, int max_iter,
                   int restart);

}  // namespace ifgfb200
