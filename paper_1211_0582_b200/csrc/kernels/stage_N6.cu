// Stage kernels for order N=6 (all variants; see stage_inst.cuh).
#define DG_N 6
#include "stage_inst.cuh"
