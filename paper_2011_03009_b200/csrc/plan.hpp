// Per-axis FFT plan (host/device shared, no device code).
#pragma once
#include <vector_types.h>

namespace fusg {

constexpr int kMaxStages = 8;
constexpr int kMaxElems = 8;  // complex values a thread holds per stage (radix <= 8)

struct AxisPlan {
  int L;                     // transform length (padded size along this axis)
  int nst;                   // number of stages
  int radix[kMaxStages];
  int ns[kMaxStages];        // product of radices before stage s
  int tpl;                   // threads per line
  const double2* tw;         // device table exp(-2 pi i m / L), m in [0, L)
};

}  // namespace fusg
