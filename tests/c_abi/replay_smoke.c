/* A plain C host of the drop-in boundary (include/peakmem_b200.h): two
 * traces replayed through pm_replay_host, no Python, no torch.  Prints one
 * line per trace: status peak_reserved peak_allocated final_reserved
 * final_allocated n_segments_peak stop_index.  tests/test_c_abi_gpu.py
 * builds it with gcc and compares the lines with the oracle. */
#include <stdio.h>
#include <stdint.h>

#include "peakmem_b200.h"

#define MIB (1ll << 20)

static pm_req_t A(int64_t size, int32_t h) {
  pm_req_t r = {size, h, PM_KIND_ALLOC};
  return r;
}
static pm_req_t F(int32_t h) {
  pm_req_t r = {0, h, PM_KIND_FREE};
  return r;
}

int main(void) {
  /* trace 0: split, coalesce and reuse; trace 1: a capacity that forces a
   * release and then an OOM */
  pm_req_t reqs[] = {
      A(1 * MIB, 0), A(3 * MIB, 1), A(700 * 1024, 2), F(0), A(512 * 1024, 3),
      F(2), F(3), A(25 * MIB, 4), F(1), A(2 * MIB, 5), F(4), F(5),
      A(10 * MIB, 0), A(10 * MIB, 1), F(0), A(30 * MIB, 2), A(40 * MIB, 3),
  };
  const int64_t offs[] = {0, 12, 17};
  pm_cfg_t cfg[2];
  for (int i = 0; i < 2; ++i) {
    cfg[i].k_small_size = 1 * MIB;
    cfg[i].k_small_buffer = 2 * MIB;
    cfg[i].k_min_large_alloc = 10 * MIB;
    cfg[i].k_large_buffer = 20 * MIB;
    cfg[i].k_round_large = 2 * MIB;
    cfg[i].alignment = 512;
    cfg[i].max_split_size = -1;
    cfg[i].device_capacity = -1;
  }
  cfg[1].device_capacity = 64 * MIB;
  const int32_t cfg_of[] = {0, 1};
  pm_result_t res[2];
  int rc = pm_replay_host(reqs, offs, 2, cfg, 2, cfg_of, res, NULL, NULL);
  if (rc != 0) {
    fprintf(stderr, "pm_replay_host failed: %d %s\n", rc, pm_last_error());
    return 1;
  }
  for (int t = 0; t < 2; ++t)
    printf("%d %lld %lld %lld %lld %d %lld\n", res[t].status,
           (long long)res[t].peak_reserved, (long long)res[t].peak_allocated,
           (long long)res[t].final_reserved, (long long)res[t].final_allocated,
           res[t].n_segments_peak, (long long)res[t].stop_index);
  return 0;
}
