// Stage kernels for order N=9 (all variants; see stage_inst.cuh).
#define DG_N 9
#include "stage_inst.cuh"
