// Stage kernels for order N=7 (all variants; see stage_inst.cuh).
#define DG_N 7
#include "stage_inst.cuh"
