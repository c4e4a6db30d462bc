// EB+PR launchers (K5 EB+RM+PR, K7 EB+CM+PR).
#define DASPMM_PDL_EXPR (p.pdl)
#include "launch_pr.cuh"
namespace daspmm {
DASPMM_PR_LAUNCHER(launch_eb_pr, k_eb_pr)
}  // namespace daspmm
