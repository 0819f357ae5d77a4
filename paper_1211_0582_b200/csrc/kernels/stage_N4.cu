// Stage kernels for order N=4 (all variants; see stage_inst.cuh).
#define DG_N 4
#include "stage_inst.cuh"
