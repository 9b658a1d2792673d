// Register executor, 16 amplitudes per thread and state (K = 11 tile bits):
// forward programs (two to three blocks per SM) and, by default, adjoint sweeps.
#define VQB_RS_RB 4
#define VQB_RS_TB 7
#define VQB_RS_NS rs16
#ifndef VQB_RS16_FWD_BLOCKS
#define VQB_RS16_FWD_BLOCKS 3
#endif
#define VQB_RS_FWD_BLOCKS VQB_RS16_FWD_BLOCKS
#define VQB_RS_REV_BLOCKS 2
#include "regstage_impl.cuh"
