#define EMF_T double
#define EMF_P 3
#include "inst.cuh"
