// 3D (tetrahedra) kernels and launchers for order k=4.
#include "order3d_ops.cuh"

HDGC_INSTANTIATE_ORDER3(4)
