// Kernels and launchers for order k=7 (own translation unit: parallel builds,
// and its own constant-bank tables).
#define HDGC_ORDER 7
#include "order_ops.cuh"

HDGC_INSTANTIATE_ORDER(7)
