/* capi_example.c -- a plain C99 caller of the reshard C ABI (no Python, no
 * torch): plans a resize, prints its summary and verify verdict as JSON.
 *
 *   gcc -std=c99 -Iinclude tools/capi_example.c -Lpaper_2605_22014_b200 \
 *       -lreshard_b200 -Wl,-rpath,paper_2605_22014_b200 -o capi_example
 *   ./capi_example spec.txt  tp0 pp0 dp0  tp1 pp1 dp1
 */
#include <stdio.h>
#include <stdlib.h>

#include "rs_reshard.h"

static char* slurp(const char* path) {
  FILE* f = fopen(path, "rb");
  if (!f) return NULL;
  fseek(f, 0, SEEK_END);
  long n = ftell(f);
  fseek(f, 0, SEEK_SET);
  char* s = (char*)malloc((size_t)n + 1);
  if (fread(s, 1, (size_t)n, f) != (size_t)n) { fclose(f); free(s); return NULL; }
  s[n] = 0;
  fclose(f);
  return s;
}

static rs_config iota(uint64_t gen, int tp, int pp, int dp, int32_t* ranks) {
  rs_config c;
  int n = tp * pp * dp;
  for (int i = 0; i < n; ++i) ranks[i] = i;
  c.generation_id = gen;
  c.tp = tp; c.pp = pp; c.dp = dp;
  c.num_ranks = n;
  c.ranks = ranks;
  c.layer_stage = NULL;
  c.distributed_optimizer = 0;
  c.dist_opt_bucket_elems = 0;
  return c;
}

int main(int argc, char** argv) {
  if (argc != 8) {
    fprintf(stderr, "usage: %s spec tp0 pp0 dp0 tp1 pp1 dp1\n", argv[0]);
    return 2;
  }
  char* spec = slurp(argv[1]);
  if (!spec) { fprintf(stderr, "cannot read %s\n", argv[1]); return 3; }
  int32_t r0[4096], r1[4096];
  rs_config c_old = iota(1, atoi(argv[2]), atoi(argv[3]), atoi(argv[4]), r0);
  rs_config c_new = iota(2, atoi(argv[5]), atoi(argv[6]), atoi(argv[7]), r1);
  rs_plan* plan = NULL;
  int rc = rs_plan_compute(spec, &c_old, &c_new, NULL, &plan);
  if (rc != RS_OK) { printf("{\"rc\": %d, \"error\": \"%s\"}\n", rc, rs_last_error()); return 1; }
  rs_plan_summary_t s;
  rs_plan_summary(plan, &s);
  size_t need = 0;
  rs_plan_write(plan, NULL, 0, &need);
  int32_t nviol = -1;
  size_t vneed = 0;
  rs_plan_verify(plan, &c_old, &c_new, NULL, 0, &vneed, &nviol);
  printf("{\"rc\": 0, \"version\": \"%s\", \"total_bytes\": %lld, \"remote_bytes\": %lld, "
         "\"local_bytes\": %lld, \"carryover_bytes\": %lld, \"task_count\": %lld, "
         "\"plan_text_bytes\": %zu, \"violations\": %d}\n",
         rs_version(), (long long)s.total_bytes, (long long)s.remote_bytes, (long long)s.local_bytes,
         (long long)s.carryover_bytes, (long long)s.task_count, need, nviol);
  rs_plan_destroy(plan);
  free(spec);
  return 0;
}
