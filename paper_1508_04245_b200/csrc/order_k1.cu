// Kernels and launchers for order k=1 (own translation unit: parallel builds,
// and its own constant-bank tables).
#define HDGC_ORDER 1
#include "order_ops.cuh"

HDGC_INSTANTIATE_ORDER(1)
