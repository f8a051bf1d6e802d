#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <stdint.h>
#include <omp.h>
#include <tgmath.h>
#define double float
#include "mpm_oracle_omp.c"
