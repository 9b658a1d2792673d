// Register executor, 16 amplitudes per thread and 256 threads per block
// (K = 12 tile bits): fewer, fuller forward stages (opt-in, VQB_REGS=16w).
#define VQB_RS_RB 4
#define VQB_RS_TB 8
#define VQB_RS_NS rs16w
#define VQB_RS_FWD_BLOCKS 2
#define VQB_RS_REV_BLOCKS 1
#include "regstage_impl.cuh"
