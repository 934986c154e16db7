/* test_group.c — the multi-GPU C-ABI from plain C (gcc, no CUDA headers, no
 * torch): a C caller shards mapreduce and scan over a forge_group using only
 * include/forge.h.  Device memory comes from the Machine API (one Machine per
 * shard device).  Checked against host folds.  Built by
 * __graft_entry__.build() (Makefile target `cpptests`), run by
 * tests/test_gpu_cpp.py on a B200: G = 1 (NCCL clique) and G = 3 emulated. */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "forge.h"

static int fails = 0, passes = 0;
#define EXPECT(c, ...)                       \
  do {                                       \
    if (c) {                                 \
      ++passes;                              \
    } else {                                 \
      ++fails;                               \
      printf("FAIL line %d: ", __LINE__);    \
      printf(__VA_ARGS__);                   \
      printf(" (%s)\n", forge_last_error()); \
    }                                        \
  } while (0)

enum { MAXG = 4 };

/* every setup call must succeed; a failure aborts the case */
#define MUST(call)                                                        \
  do {                                                                    \
    int rc_ = (call);                                                     \
    if (rc_ != FORGE_OK) {                                                \
      ++fails;                                                            \
      printf("FAIL line %d: %s -> %d (%s)\n", __LINE__, #call, rc_, forge_last_error()); \
      return;                                                             \
    }                                                                     \
  } while (0)

static void run(const int32_t* devs, int G, uint64_t n) {
  forge_group* g = NULL;
  int rc = forge_group_create(devs, G, &g);
  EXPECT(rc == FORGE_OK, "group create G=%d rc=%d", G, rc);
  if (rc) return;
  forge_machine* m[MAXG];
  void *src[MAXG], *dst[MAXG], *ws[MAXG];
  uint64_t ns[MAXG], wsb[MAXG];
  forge_buffer_id bs[MAXG], bd[MAXG], bw[MAXG];
  int32_t* host = malloc(n * sizeof(int32_t)); /* (leaked on a failed setup: test program) */
  int32_t* back = malloc(n * sizeof(int32_t));
  for (uint64_t i = 0; i < n; ++i) host[i] = (int32_t)((i * 2654435761u) % 1000u) - 500;
  for (int r = 0; r < G; ++r) {
    uint64_t lo, hi, need_s, need_m;
    MUST(forge_shard_range(n, r, G, &lo, &hi));
    ns[r] = hi - lo;
    MUST(forge_machine_create(devs[r], &m[r]));
    MUST(forge_create_buffer(m[r], "u32", ns[r] ? ns[r] : 1, 4096, &bs[r]));
    MUST(forge_create_buffer(m[r], "u32", ns[r] ? ns[r] : 1, 4096, &bd[r]));
    MUST(forge_dev_workspace_bytes(FORGE_PRIM_SCAN, FORGE_OP_I32_SUM, ns[r], 0, &need_s));
    MUST(forge_dev_workspace_bytes(FORGE_PRIM_MAPREDUCE, FORGE_OP_I32_SUM, ns[r], 0, &need_m));
    wsb[r] = need_s > need_m ? need_s : need_m;
    MUST(forge_create_buffer(m[r], "u8", wsb[r], 4096, &bw[r])); /* zero-initialised, like the reference */
    MUST(forge_buffer_device_ptr(m[r], bs[r], &src[r]));
    MUST(forge_buffer_device_ptr(m[r], bd[r], &dst[r]));
    MUST(forge_buffer_device_ptr(m[r], bw[r], &ws[r]));
    if (ns[r]) MUST(forge_write_bytes(m[r], bs[r], 0, host + lo, ns[r] * sizeof(int32_t)));
    MUST(forge_machine_synchronize(m[r]));
  }
  /* mapreduce: wrapping i32 sum */
  int32_t got = 0;
  uint32_t want = 0;
  for (uint64_t i = 0; i < n; ++i) want += (uint32_t)host[i];
  rc = forge_sharded_mapreduce(g, FORGE_OP_I32_SUM, (const void* const*)src, ns, ws, wsb, &got);
  EXPECT(rc == FORGE_OK && (uint32_t)got == want, "sharded mapreduce G=%d n=%llu: %d vs %d", G,
         (unsigned long long)n, got, (int32_t)want);
  /* inclusive scan over the concatenation of the shards */
  rc = forge_sharded_scan(g, FORGE_OP_I32_SUM, 1, (const void* const*)src, dst, ns, ws, wsb);
  EXPECT(rc == FORGE_OK, "sharded scan rc=%d", rc);
  forge_group_synchronize(g);
  uint64_t off = 0;
  for (int r = 0; r < G; ++r) {
    if (ns[r]) forge_read_bytes(m[r], bd[r], 0, back + off, ns[r] * sizeof(int32_t));
    off += ns[r];
  }
  uint32_t acc = 0;
  uint64_t bad = 0;
  for (uint64_t i = 0; i < n; ++i) {
    acc += (uint32_t)host[i];
    bad += (uint32_t)back[i] != acc;
  }
  EXPECT(bad == 0, "sharded scan G=%d n=%llu: %llu mismatches", G, (unsigned long long)n,
         (unsigned long long)bad);
  for (int r = 0; r < G; ++r) forge_machine_destroy(m[r]);
  forge_group_destroy(g);
  free(host);
  free(back);
}

int main(void) {
  int count = 0;
  if (forge_device_count(&count) != FORGE_OK || count == 0) {
    printf("no CUDA device\n");
    return 2;
  }
  const int32_t one[1] = {0};
  const int32_t emu[3] = {0, 0, 0};
  for (int k = 0; k < 2; ++k) {
    const uint64_t n = k == 0 ? 2 : 3000017; /* 2 elements over 3 shards: one empty shard */
    run(one, 1, n);
    run(emu, 3, n);
  }
  /* errors */
  forge_group* g = NULL;
  const int32_t mixed[3] = {0, 0, 1};
  EXPECT(forge_group_create(mixed, 3, &g) == FORGE_ERR_INVALID_ARGUMENT, "mixed device list rejected");
  uint64_t lo, hi;
  EXPECT(forge_shard_range(10, 3, 3, &lo, &hi) == FORGE_ERR_INVALID_ARGUMENT, "rank out of range");
  printf("%s: %d passed, %d failed\n", fails ? "FAIL" : "PASS", passes, fails);
  return fails ? 1 : 0;
}
