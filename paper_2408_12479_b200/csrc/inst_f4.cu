#define EMF_T float
#define EMF_P 4
#include "inst.cuh"
