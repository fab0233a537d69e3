// fus drop-in: studies and diagnostics (reference: include/fus/analysis.hpp, src/analysis.cpp;
// shrink_domain_by_threshold from include/fus/grid.hpp:103). The off-grid evaluations, sources,
// transfers and field reductions run on the GPU; profile arithmetic is host code.
#pragma once
#include <string>
#include <vector>

#include "fus/cascade.hpp"
#include "fus/grid.hpp"

namespace fus {

struct OnAxisProfile {
  Eigen::VectorXd x;
  Eigen::VectorXcd p;
  int harmonic = 1;
};

struct ConvergenceRecord {
  int harmonic;
  std::string control;  // "n_w", "Q0" or "fraction"
  double value;
  double error_percent;
};

OnAxisProfile extract_on_axis(const HarmonicField& field);
double on_axis_error(const OnAxisProfile& p, const OnAxisProfile& p_ref, const OnAxisProfile& normalizer);
Eigen::VectorXd localisedness_map(const HarmonicField& f);
DomainBox shrink_domain_by_threshold(const HarmonicField& f, double q0);

struct QuadratureStudy {
  std::vector<ConvergenceRecord> records;
  double slope = 0.0;
};

QuadratureStudy quadrature_convergence_study(const BowlTransducer& transducer, const Medium& medium,
                                             const DomainBox& domain, const std::vector<int>& n_w_values,
                                             int n_w_ref);
MeshPlan plan_full_domain(const BowlTransducer& transducer, const Medium& medium, double d, int n_w,
                          int n_harmonics, double width_scale = 1.0);
std::vector<ConvergenceRecord> domain_shrink_study(const CascadeConfig& reference_config,
                                                   const CascadeResult& reference,
                                                   const std::vector<double>& levels, bool q0_mode);
double error_trend_diagnostic(const OnAxisProfile& p_i, const OnAxisProfile& p1, double q0);

}  // namespace fus
