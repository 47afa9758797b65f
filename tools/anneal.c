// Incremental-cost simulated annealing of the DMMA row groupings (gen/tiling.py states the
// problem): partition the output rows into groups of 8 and, per input partition, the input
// rows into groups of 4 (never mixing two classes) to minimise the number of nonzero 8x4
// tiles summed over the matrices that share the output.  Moves are pairwise swaps between
// groups; the block nonzero counts are updated along the swapped rows only.
//   anneal PROBLEM.txt MOVES SEED  ->  stdout: cost, og_of[nout], ig_of[part][nin]
// Problem file: nmats nout nin nparts / part_of[nmats] / cls_of_col[nin] / matrices (0/1).
// Build: gcc -O2 -o /tmp/anneal tools/anneal.c -lm   (driver: tools/reanneal.py)
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define MAXM 8
#define MAXR 128
static int nm, nout, nin, nparts, part_of[MAXM], cls[MAXR];
static unsigned char M[MAXM][MAXR][MAXR];
static int og_of[MAXR], ig_of[MAXM][MAXR];           // ig_of[part][col]
static int cnt[MAXM][MAXR / 4 + 1][MAXR / 4 + 1];      // cnt[mat][og][ig]
static long cost;
static unsigned long long s;
static inline unsigned rnd(void) { s = s * 6364136223846793005ULL + 1442695040888963407ULL; return (unsigned)(s >> 33); }
static inline double urand(void) { return rnd() / 2147483648.0; }

static inline void bump(int c, int a, int b, int d) {
  int v = cnt[c][a][b];
  if (d > 0) { if (v == 0) ++cost; } else { if (v == 1) --cost; }
  cnt[c][a][b] = v + d;
}
static void move_out(int r, int from, int to) {
  for (int c = 0; c < nm; ++c) { const int* ig = ig_of[part_of[c]];
    for (int j = 0; j < nin; ++j) if (M[c][r][j]) { bump(c, from, ig[j], -1); bump(c, to, ig[j], +1); } }
  og_of[r] = to;
}
static void move_in(int p, int j, int from, int to) {
  for (int c = 0; c < nm; ++c) if (part_of[c] == p)
    for (int r = 0; r < nout; ++r) if (M[c][r][j]) { bump(c, og_of[r], from, -1); bump(c, og_of[r], to, +1); }
  ig_of[p][j] = to;
}
static void recount(void) {
  memset(cnt, 0, sizeof cnt); cost = 0;
  for (int c = 0; c < nm; ++c) for (int r = 0; r < nout; ++r) for (int j = 0; j < nin; ++j)
    if (M[c][r][j]) bump(c, og_of[r], ig_of[part_of[c]][j], +1);
}

int main(int argc, char** argv) {
  FILE* f = fopen(argv[1], "r"); long moves = atol(argv[2]); s = strtoull(argv[3], 0, 10) * 2654435761ULL + 12345;
  if (!f || fscanf(f, "%d %d %d %d", &nm, &nout, &nin, &nparts) != 4) return 1;
  for (int c = 0; c < nm; ++c) if (fscanf(f, "%d", &part_of[c]) != 1) return 1;
  for (int j = 0; j < nin; ++j) if (fscanf(f, "%d", &cls[j]) != 1) return 1;
  for (int c = 0; c < nm; ++c) for (int r = 0; r < nout; ++r) for (int j = 0; j < nin; ++j) { int v; if (fscanf(f, "%d", &v) != 1) return 1; M[c][r][j] = (unsigned char)v; }
  // random start: shuffled rows chunked by 8; shuffled columns chunked by 4 within each class
  int perm[MAXR];
  for (int r = 0; r < nout; ++r) perm[r] = r;
  for (int r = nout - 1; r > 0; --r) { int k = rnd() % (r + 1), t = perm[r]; perm[r] = perm[k]; perm[k] = t; }
  for (int r = 0; r < nout; ++r) og_of[perm[r]] = r / 8;
  for (int p = 0; p < nparts; ++p) {
    int g = 0, ncls = 0;
    for (int j = 0; j < nin; ++j) if (cls[j] + 1 > ncls) ncls = cls[j] + 1;
    for (int cl = 0; cl < ncls; ++cl) {
      int n = 0;
      for (int j = 0; j < nin; ++j) if (cls[j] == cl) perm[n++] = j;
      for (int r = n - 1; r > 0; --r) { int k = rnd() % (r + 1), t = perm[r]; perm[r] = perm[k]; perm[k] = t; }
      for (int i = 0; i < n; ++i) ig_of[p][perm[i]] = g + i / 4;
      g += (n + 3) / 4;
    }
  }
  recount();
  long best = cost; int bog[MAXR], big[MAXM][MAXR];
  memcpy(bog, og_of, sizeof bog); memcpy(big, ig_of, sizeof big);
  double T = 1.5, decay = pow(0.03 / 1.5, 1.0 / (double)moves);
  for (long it = 0; it < moves; ++it, T *= decay) {
    int k = rnd() % (nparts + 1);
    long before = cost;
    if (k == nparts) {
      int r1 = rnd() % nout, r2 = rnd() % nout, a = og_of[r1], b = og_of[r2];
      if (a == b) continue;
      move_out(r1, a, b); move_out(r2, b, a);
      if (cost > before && urand() >= exp((before - cost) / T)) { move_out(r1, b, a); move_out(r2, a, b); }
    } else {
      int j1 = rnd() % nin, j2 = rnd() % nin, a = ig_of[k][j1], b = ig_of[k][j2];
      if (a == b || cls[j1] != cls[j2]) continue;
      move_in(k, j1, a, b); move_in(k, j2, b, a);
      if (cost > before && urand() >= exp((before - cost) / T)) { move_in(k, j1, b, a); move_in(k, j2, a, b); }
    }
    if (cost < best) { best = cost; memcpy(bog, og_of, sizeof bog); memcpy(big, ig_of, sizeof big); }
  }
  printf("%ld\n", best);
  for (int r = 0; r < nout; ++r) printf("%d ", bog[r]);
  printf("\n");
  for (int p = 0; p < nparts; ++p) { for (int j = 0; j < nin; ++j) printf("%d ", big[p][j]); printf("\n"); }
  return 0;
}
