/* Exhaustive check that fma-refined multiplication by RN(1/f^2) reproduces the
 * correctly rounded quotient g / f^2 for every f in [2, 1024], g < f^2
 * (tests/test_adj_division.py; the device formula is adj_of() in ls_sortsub.cu). */
#include <math.h>
#include <stdio.h>
#include <stdint.h>
int main(void) {
    long bad = 0, tot = 0;
    for (int f = 2; f <= 1024; f++) {
        const double F2 = (double)f * (double)f, rcp = 1.0 / F2;
        const long gmax = (long)f * f;
        for (long g = 0; g < gmax; g++) {
            const double gd = (double)g;
            const double want = gd / F2;
            const double q0 = gd * rcp;
            const double r = fma(-q0, F2, gd);
            const double q = fma(r, rcp, q0);
            tot++;
            if (q != want) { if (bad < 5) printf("f=%d g=%ld %.17g %.17g\n", f, g, q, want); bad++; }
        }
    }
    printf("checked %ld bad %ld\n", tot, bad);
    return bad != 0;
}
