#define EMF_T float
#define EMF_P 1
#include "inst.cuh"
