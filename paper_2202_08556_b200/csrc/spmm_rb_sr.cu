// RB+SR launchers (K0 RB+RM+SR, K2 RB+CM+SR).
#include "launch_sr.cuh"
namespace daspmm {
DASPMM_SR_LAUNCHER(launch_rb_sr, k_rb_sr)
}  // namespace daspmm
