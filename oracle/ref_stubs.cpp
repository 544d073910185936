// Stubs for the reference symbols whose only definitions live in
// eigen_solvers.cpp (dense SVD / eigenvalue diagnostics, Eigen-only, out of
// scope per SURVEY.md §2 row 13). TEST INFRASTRUCTURE ONLY: they throw if a
// diagnostic path is ever reached while the oracle runs.
#include <stdexcept>
#include <utility>

#include "gadi/dense.hpp"
#include "gadi/errors.hpp"

namespace gadi {

std::pair<double, double> sigma_extremes(const SparseMatrix&) {
  throw std::logic_error("oracle/_ref: sigma_extremes is a diagnostic (eigen_solvers.cpp) not built here");
}

double spectral_radius(const DenseMatrix&) {
  throw std::logic_error("oracle/_ref: spectral_radius is a diagnostic (eigen_solvers.cpp) not built here");
}

}  // namespace gadi
