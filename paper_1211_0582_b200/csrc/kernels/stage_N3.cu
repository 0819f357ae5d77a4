// Stage kernels for order N=3 (all variants; see stage_inst.cuh).
#define DG_N 3
#include "stage_inst.cuh"
