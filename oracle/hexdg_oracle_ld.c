/* ORACLE, extended precision -- test infrastructure only. hexdg_oracle.c with every
 * double an x87 long double (64-bit significand) and <tgmath.h> routing sqrt / exp /
 * sin / cos / fabs to their long double forms: an accurate yardstick for the
 * floating-point error of the reference itself and of the FMA kernel set on
 * ill-conditioned (low-Mach) right-hand sides. The system headers are included
 * first, so the redefinition only reaches the oracle's own code. */
#include <math.h>
#include <omp.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <tgmath.h>
#define double long double
#include "hexdg_oracle.c"
