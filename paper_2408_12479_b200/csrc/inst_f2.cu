#define EMF_T float
#define EMF_P 2
#include "inst.cuh"
