// k2_filter_tma10.cu — the TMA-ring K2 built with 10 compute warps per block
// (5 per scheduler at 2 blocks per SM; see k2_filter_tma.cu).  Selected with
// CUDAPRE_K2_WARPS=10.
#define K2_NW 10
#define K2_ENTRY launch_filter_tma10
#include "k2_filter_tma.cu"
