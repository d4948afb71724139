#define EMF_T double
#define EMF_P 2
#include "inst.cuh"
