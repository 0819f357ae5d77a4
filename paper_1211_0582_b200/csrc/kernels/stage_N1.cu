// Stage kernels for order N=1 (all variants; see stage_inst.cuh).
#define DG_N 1
#include "stage_inst.cuh"
