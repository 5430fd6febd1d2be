// 3D (tetrahedra) kernels and launchers for order k=4 (own constant-bank tables).
#define HDGC_ORDER3 4
#include "order3d_ops.cuh"

HDGC_INSTANTIATE_ORDER3(4)
