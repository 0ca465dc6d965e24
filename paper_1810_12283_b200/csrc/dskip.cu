// dskip.cu — placeholder until the D-SKIP device operator lands.
#include "gk_common.hpp"

namespace gk {
std::unique_ptr<Op> make_dskip(const gk_kernel&, const double*, i64, int, double, double, const gk_dskip_config&,
                               int) {
  fail(GK_ERR_UNSUPPORTED, "D-SKIP device operator not built yet");
}
int dskip_factor_count(const Op&) { fail(GK_ERR_UNSUPPORTED, "not a D-SKIP operator"); }
i64 dskip_factor_rank(const Op&, int) { fail(GK_ERR_UNSUPPORTED, "not a D-SKIP operator"); }
void dskip_factor_get(const Op&, int, double*, double*, double*) { fail(GK_ERR_UNSUPPORTED, "not a D-SKIP operator"); }
void dskip_dlogell(Op&, const double*, double*, int, cudaStream_t) { fail(GK_ERR_UNSUPPORTED, "not a D-SKIP operator"); }
}  // namespace gk
