// 3D (tetrahedra) kernels and launchers for order k=1.
#include "order3d_ops.cuh"

HDGC_INSTANTIATE_ORDER3(1)
