// Instantiation unit of the L = 128 torus (compiled in parallel with the other sizes).
#include "holo_run.cuh"
HOLO_DEFINE_OPS(128)
