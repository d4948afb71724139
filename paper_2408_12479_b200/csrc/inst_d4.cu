#define EMF_T double
#define EMF_P 4
#include "inst.cuh"
