#define EMF_T double
#define EMF_P 1
#include "inst.cuh"
