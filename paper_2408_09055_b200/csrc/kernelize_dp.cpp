// kernelize_dp.cpp -- Alg. Kernelize placeholder:
// until the DP lands, fall back to OrderedKernelize (which Kernelize never
// does worse than, Thm. dp-optimal).
#include "internal.h"

namespace atlas {
KernelPlan dp_kernelize(const std::vector<KGate> &seq, const CostModel &cm,
                        const KernelizeOptions &o) {
  return ordered_kernelize(seq, cm, o);
}
}  // namespace atlas
