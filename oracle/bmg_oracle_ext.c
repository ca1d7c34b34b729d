/*
 * oracle/bmg_oracle_ext.c -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.
 *
 * The SAME oracle source (bmg_oracle.c, every step and its citation there)
 * evaluated in x86-64 extended precision: every `double` (storage, arithmetic,
 * the ABI's arrays) becomes `long double` (x87 80-bit, 64-bit significand, unit
 * roundoff 5.4e-20 against fp64's 1.1e-16), and <tgmath.h> routes sqrt/fabs/
 * fmin to their long double forms.  Used by tests/test_oracle_extended.py and
 * tests/test_gpu_parity.py only, to measure how far each fp64 implementation
 * (the fp64 oracle and the GPU path) sits from the iterate computed 2048x more
 * precisely -- the evidence behind the anisotropic tolerance of DESIGN.md §7.
 */
#include <math.h>
#include <tgmath.h>
#include <stdlib.h>
#include <string.h>
#undef I /* <complex.h> (pulled in by <tgmath.h>) defines I; the oracle uses it as an index */
#undef complex
#define double long double
#include "bmg_oracle.c"
