// hcb_solve_inst.cu -- explicit solve_kernel instantiations, one group per
// object (make builds it with -DHC_INST_GROUP=0..11 in parallel).
#include "hcb_solve_dev.cuh"

#ifndef HC_INST_GROUP
#error "compile with -DHC_INST_GROUP=<0..11>"
#endif
#define HC_CAT2(a, b) a##b
#define HC_CAT(a, b) HC_CAT2(a, b)

namespace hcb {
namespace solve {
#define HC_DEF_INST(OffT, F, ST) template const void *kernel_ptr<OffT, F, ST>();
HC_CAT(HC_INST_G, HC_INST_GROUP)(HC_DEF_INST)
#undef HC_DEF_INST
}  // namespace solve
}  // namespace hcb
