/* pfsp_oracle CLI (TEST INFRASTRUCTURE ONLY): the C restatement as a command, for the
 * CPU-baseline legs of bench.py and for pinning LB2 golden counts.
 *
 *   pfsp_oracle solve <ta> <lb1|lb2> <ub|neh> <threads> <prefix_depth> <pinned 0|1> <time_limit_s>
 */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "pfsp_oracle.h"

int main(int argc, char** argv) {
  if (argc < 9 || strcmp(argv[1], "solve") != 0) {
    fprintf(stderr, "usage: pfsp_oracle solve <ta> <lb1|lb2> <ub|neh> <threads> <depth> <pinned> <limit>\n");
    return 2;
  }
  static int32_t p[512 * 64];
  int n = 0, m = 0;
  if (or_taillard_named(argv[2], &n, &m, p) != 0) {
    fprintf(stderr, "bad instance %s\n", argv[2]);
    return 2;
  }
  const int bound = strcmp(argv[3], "lb2") == 0 ? OR_LB2 : OR_LB1;
  int64_t ub;
  if (strcmp(argv[4], "neh") == 0) {
    int perm[512];
    ub = or_neh(n, m, p, perm);
  } else {
    ub = strtoll(argv[4], NULL, 10);
  }
  or_problem pr;
  if (or_problem_init(&pr, n, m, p, bound) != 0) return 2;
  static or_stats st;
  if (or_solve(&pr, ub, atoi(argv[5]), atoi(argv[6]), atoi(argv[7]), 0, atof(argv[8]), &st) != 0)
    return 1;
  printf("{\"mode\":\"solve\",\"instance\":\"%s\",\"bound\":\"%s\",\"initial_ub\":%lld,"
         "\"best_value\":%lld,\"improved\":%s,\"decomposed\":%llu,\"unique\":%llu,\"leaves\":%llu,"
         "\"improvements\":%llu,\"wall_s\":%.6f,\"completed\":%s,\"threads\":%d,\"hist\":{",
         argv[2], argv[3], (long long)ub, (long long)st.best, st.has_perm ? "true" : "false",
         (unsigned long long)st.decomposed, (unsigned long long)st.unique,
         (unsigned long long)st.leaves, (unsigned long long)st.improvements, st.wall_s,
         st.completed ? "true" : "false", atoi(argv[5]));
  int first = 1;
  for (int f = 0; f <= n; ++f) {
    if (!st.hist[f]) continue;
    printf("%s\"%d\":%llu", first ? "" : ",", f, (unsigned long long)st.hist[f]);
    first = 0;
  }
  printf("},\"best\":[");
  if (st.has_perm)
    for (int i = 0; i < n; ++i) printf("%s%d", i ? "," : "", st.best_perm[i]);
  printf("]}\n");
  or_problem_free(&pr);
  return 0;
}
