// Instantiation unit of the L = 6144 = 3 x 2048 torus (reference arm only, reading C16).
#include "holo_run.cuh"
HOLO_DEFINE_REF_OPS(6144)
