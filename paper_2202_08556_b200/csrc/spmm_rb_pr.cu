// RB+PR launchers (K1 RB+RM+PR, K3 RB+CM+PR).
#include "launch_pr.cuh"
namespace daspmm {
DASPMM_PR_LAUNCHER(launch_rb_pr, k_rb_pr)
}  // namespace daspmm
