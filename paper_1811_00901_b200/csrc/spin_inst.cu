// spin_inst.cu — explicit instantiations of spin_persistent for one (MODE, SUP, DEAL)
// triple, selected with -DINST_MODE=0|1 -DINST_SUP=0|1|2 -DINST_DEAL=0|1 (built twelve
// times by build.py; the adaptive SUP = 2 exists for BRUTE only; DEAL = 1 is the WF / AWF
// compare-and-swap dealer; the two-CTA cluster variant (cl = 2, G = 48 over the pair) for
// BRUTE NEAREST with the table dealer only).
#include "spin_persistent.cuh"

namespace spin {

#define SPIN_CAT2(a, b, c, d) a##b##_##c##_##d
#define SPIN_CAT(a, b, c, d) SPIN_CAT2(a, b, c, d)
const void* SPIN_CAT(kernel_ptr_, INST_MODE, INST_SUP, INST_DEAL)(int prune, int G, int nt, int cl) {
  constexpr int D = NT_DEFAULT;
  if (prune == 0) {
#if INST_DEAL == 0 && INST_MODE == 0
    if (cl == 2) return (const void*)spin_persistent<INST_MODE, 0, 48, INST_SUP, D, 0, 2>;
#endif
    if (cl != 1) return nullptr;
    if (nt == 512) return (const void*)spin_persistent<INST_MODE, 0, 32, INST_SUP, 512, INST_DEAL, 1>;
    switch (G) {
      case 4: return (const void*)spin_persistent<INST_MODE, 0, 4, INST_SUP, D, INST_DEAL, 1>;
      case 8: return (const void*)spin_persistent<INST_MODE, 0, 8, INST_SUP, D, INST_DEAL, 1>;
      case 16: return (const void*)spin_persistent<INST_MODE, 0, 16, INST_SUP, D, INST_DEAL, 1>;
      case 24: return (const void*)spin_persistent<INST_MODE, 0, 24, INST_SUP, D, INST_DEAL, 1>;
      case 32: return (const void*)spin_persistent<INST_MODE, 0, 32, INST_SUP, D, INST_DEAL, 1>;
      default: return (const void*)spin_persistent<INST_MODE, 0, 64, INST_SUP, D, INST_DEAL, 1>;
    }
  }
#if INST_SUP == 2
  return nullptr;
#else
  if (cl != 1) return nullptr;
  switch (G) {
    case 4: return (const void*)spin_persistent<INST_MODE, 1, 4, INST_SUP, D, INST_DEAL, 1>;
    case 8: return (const void*)spin_persistent<INST_MODE, 1, 8, INST_SUP, D, INST_DEAL, 1>;
    case 16: return (const void*)spin_persistent<INST_MODE, 1, 16, INST_SUP, D, INST_DEAL, 1>;
    case 32: return (const void*)spin_persistent<INST_MODE, 1, 32, INST_SUP, D, INST_DEAL, 1>;
    default: return (const void*)spin_persistent<INST_MODE, 1, 64, INST_SUP, D, INST_DEAL, 1>;
  }
#endif
}

}  // namespace spin
