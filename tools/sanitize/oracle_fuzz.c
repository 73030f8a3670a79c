/* Host sanitizer driver (ASan + UBSan) for oracle/tt_oracle.c: every entry
 * point on seeded random small problems, checked against each other (the
 * odometer, the range form and the per-position decode must agree).
 *   gcc -fsanitize=address,undefined -g -O1 oracle_fuzz.c ../../oracle/tt_oracle.c */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

int oracle_permute(int, const int64_t*, const int*, int, const void*, void*);
int oracle_permute_range(int, const int64_t*, const int*, int, const void*, void*, int64_t, int64_t);
int oracle_permute_sample(int, const int64_t*, const int*, int, const void*, const int64_t*, int64_t, void*);
int oracle_permute_scaled(int, const int64_t*, const int*, int, const void*, void*, double, double);

static uint64_t s = 1705;
static uint64_t rnd(void) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; return s; }

int main(void) {
    int bad = 0;
    for (int it = 0; it < 4000; ++it) {
        int n = 1 + (int)(rnd() % 8), perm[8];
        int64_t d[8], vol = 1;
        for (int i = 0; i < n; ++i) { d[i] = 1 + (int64_t)(rnd() % 6); vol *= d[i]; perm[i] = i; }
        for (int i = n - 1; i > 0; --i) { int j = (int)(rnd() % (i + 1)), t = perm[i]; perm[i] = perm[j]; perm[j] = t; }
        const int E = (rnd() & 1) ? 4 : 8;
        unsigned char* in = malloc(vol * E), *a = malloc(vol * E), *b = malloc(vol * E), *c = malloc(vol * E);
        int64_t* pos = malloc(vol * sizeof(int64_t));
        for (int64_t i = 0; i < vol * E; ++i) in[i] = (unsigned char)rnd();
        for (int64_t i = 0; i < vol; ++i) pos[i] = i;
        bad |= oracle_permute(n, d, perm, E, in, a);
        const int64_t mid = vol / 3;
        bad |= oracle_permute_range(n, d, perm, E, in, b, 0, mid);
        bad |= oracle_permute_range(n, d, perm, E, in, b, mid, vol);
        bad |= oracle_permute_sample(n, d, perm, E, in, pos, vol, c);
        if (memcmp(a, b, vol * E) || memcmp(a, c, vol * E)) bad |= 2;
        /* scaled form on finite floats */
        for (int64_t i = 0; i < vol; ++i) {
            if (E == 4) { float f = (float)(rnd() % 1000) / 7.f; memcpy(in + 4 * i, &f, 4); memcpy(b + 4 * i, &f, 4); }
            else { double f = (double)(rnd() % 1000) / 7.; memcpy(in + 8 * i, &f, 8); memcpy(b + 8 * i, &f, 8); }
        }
        bad |= oracle_permute_scaled(n, d, perm, E, in, b, 1.5, 0.5);
        bad |= oracle_permute_scaled(n, d, perm, E, in, b, 2.0, 0.0);
        free(in); free(a); free(b); free(c); free(pos);
        if (bad) { printf("oracle fuzz: failure at iteration %d\n", it); return 1; }
    }
    /* rejected arguments */
    int64_t d2[2] = {2, 0};
    int p2[2] = {1, 0}, p3[2] = {0, 0};
    unsigned char x[64], y[64];
    if (oracle_permute(2, d2, p2, 4, x, y) == 0) return 1;
    d2[1] = 3;
    if (oracle_permute(2, d2, p3, 4, x, y) == 0 || oracle_permute(2, d2, p2, 2, x, y) == 0) return 1;
    printf("oracle fuzz: 4000 problems, every entry point agrees; bad arguments rejected\n");
    return 0;
}
