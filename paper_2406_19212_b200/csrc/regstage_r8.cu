// Register executor, 8 amplitudes per thread and state (K = 10 tile bits):
// half the data registers of rs16, so adjoint sweeps (two register states)
// run without spills at four blocks per SM.
#define VQB_RS_RB 3
#define VQB_RS_TB 7
#define VQB_RS_NS rs8
#define VQB_RS_FWD_BLOCKS 4
#define VQB_RS_REV_BLOCKS 3
#include "regstage_impl.cuh"
