// tc_survivors.c -- offline count of the sets the threshold-count tier
// would keep: sets whose lower bound sum_e Q(min_c l[c][e]) <= tau, for a given threshold
// list t_1 < t_2 < ... (Q(x) = the largest t_j <= x, 0 below t_1).  Reads /tmp/l.bin
// (int32 E, int32 C, then C x E fp64 log-slowdowns, config-major), written by
// tools/tc_survivors_prep.py.  gcc -O3 -march=native -fopenmp -o /tmp/tc_surv tools/tc_survivors.c
//   /tmp/tc_surv <tau> <k: 2|3> <t_1> [<t_2> ...]
// count k=3 sets whose threshold lower bound <= s2, for several threshold sets
#include <stdio.h>
#include <stdlib.h>
#include <math.h>
#include <string.h>
#include <omp.h>
int main(int argc, char **argv) {
  FILE *f = fopen("/tmp/l.bin", "rb"); int E, C; fread(&E, 4, 1, f); fread(&C, 4, 1, f);
  double *l = malloc(sizeof(double) * E * C); fread(l, 8, (size_t)E * C, f); fclose(f); // [c][e]
  double s2 = atof(argv[1]); int k = atoi(argv[2]);
  int nt = argc - 3; double t[16]; for (int j = 0; j < nt; j++) t[j] = atof(argv[3 + j]);
  unsigned char *q = malloc((size_t)E * C);
  for (size_t i = 0; i < (size_t)E * C; i++) { int c = 0; while (c < nt && l[i] >= t[c]) c++; q[i] = c; }
  double w[17]; w[0] = 0; for (int j = 1; j <= nt; j++) w[j] = t[j - 1];  // Q(level j) = t_{j-1}
  long long surv = 0, tot = 0;
  if (k == 2) {
    for (int a = 0; a < C; a++) for (int b = a + 1; b < C; b++) { double s = 0; for (int e = 0; e < E; e++) { int m = q[a*E+e] < q[b*E+e] ? q[a*E+e] : q[b*E+e]; s += w[m]; } tot++; if (s <= s2) surv++; }
  } else {
    #pragma omp parallel for schedule(dynamic) reduction(+:surv,tot)
    for (int c2 = 2; c2 < C; c2++) { unsigned char A[1024]; for (int b = 0; b < c2; b++) { for (int e = 0; e < E; e++) A[e] = q[b*E+e] < q[c2*E+e] ? q[b*E+e] : q[c2*E+e];
      for (int a = 0; a < b; a++) { double s = 0; const unsigned char *qa = q + (size_t)a*E; for (int e = 0; e < E; e++) { int m = qa[e] < A[e] ? qa[e] : A[e]; s += w[m]; } tot++; if (s <= s2) surv++; } } }
  }
  printf("nt=%d surv=%lld of %lld\n", nt, surv, tot);
}
