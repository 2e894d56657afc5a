// spin_inst.cu — explicit instantiations of spin_persistent for one (MODE, SUP) pair,
// selected with -DINST_MODE=0|1 -DINST_SUP=0|1|2 (built six times by build.py; the
// adaptive SUP = 2 exists for BRUTE only).
#include "spin_persistent.cuh"

namespace spin {

#define SPIN_CAT2(a, b, c) a##b##_##c
#define SPIN_CAT(a, b, c) SPIN_CAT2(a, b, c)
const void* SPIN_CAT(kernel_ptr_, INST_MODE, INST_SUP)(int prune, int G, int nt) {
  constexpr int D = NT_DEFAULT;
  if (prune == 0) {
    if (nt == 512) return (const void*)spin_persistent<INST_MODE, 0, 32, INST_SUP, 512>;
    switch (G) {
      case 4: return (const void*)spin_persistent<INST_MODE, 0, 4, INST_SUP, D>;
      case 8: return (const void*)spin_persistent<INST_MODE, 0, 8, INST_SUP, D>;
      case 16: return (const void*)spin_persistent<INST_MODE, 0, 16, INST_SUP, D>;
      case 24: return (const void*)spin_persistent<INST_MODE, 0, 24, INST_SUP, D>;
      case 32: return (const void*)spin_persistent<INST_MODE, 0, 32, INST_SUP, D>;
      default: return (const void*)spin_persistent<INST_MODE, 0, 64, INST_SUP, D>;
    }
  }
#if INST_SUP == 2
  return nullptr;
#else
  switch (G) {
    case 4: return (const void*)spin_persistent<INST_MODE, 1, 4, INST_SUP, D>;
    case 8: return (const void*)spin_persistent<INST_MODE, 1, 8, INST_SUP, D>;
    case 16: return (const void*)spin_persistent<INST_MODE, 1, 16, INST_SUP, D>;
    case 32: return (const void*)spin_persistent<INST_MODE, 1, 32, INST_SUP, D>;
    default: return (const void*)spin_persistent<INST_MODE, 1, 64, INST_SUP, D>;
  }
#endif
}

}  // namespace spin
