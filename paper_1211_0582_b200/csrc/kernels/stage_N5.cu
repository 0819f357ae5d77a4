// Stage kernels for order N=5 (all variants; see stage_inst.cuh).
#define DG_N 5
#include "stage_inst.cuh"
