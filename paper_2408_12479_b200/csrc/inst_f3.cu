#define EMF_T float
#define EMF_P 3
#include "inst.cuh"
