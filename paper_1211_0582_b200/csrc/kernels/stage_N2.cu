// Stage kernels for order N=2 (all variants; see stage_inst.cuh).
#define DG_N 2
#include "stage_inst.cuh"
