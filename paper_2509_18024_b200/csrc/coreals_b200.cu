// coreals_b200.cu -- unity translation unit for libcoreals_b200.so (sm_100a).
#include "sweep_small.cu"
#include "sweep_big.cu"
#include "sweep_tc.cu"
#include "sweep_solve.cu"
#include "sweep_refine.cu"
#include "misc.cu"
#include "abi.cu"
#include "index.cu"
