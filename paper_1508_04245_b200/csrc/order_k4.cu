// Kernels and launchers for order k=4 (own translation unit: parallel builds,
// and its own constant-bank tables).
#define HDGC_ORDER 4
#include "order_ops.cuh"

HDGC_INSTANTIATE_ORDER(4)
