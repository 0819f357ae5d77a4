// Stage kernels for order N=8 (all variants; see stage_inst.cuh).
#define DG_N 8
#include "stage_inst.cuh"
