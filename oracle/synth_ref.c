/*
 * TEST / BENCH INFRASTRUCTURE ONLY — the CPU generator of the seeded
 * synthetic config volumes (the bench's reference arm and cpu_baseline leg,
 * tests). It runs the same per-voxel construction as the device generator
 * (paper_1806_08741_b200/csrc/synth_gen.h, IEEE-exact single precision,
 * compiled here with -ffp-contract=off), so it produces the device's bytes
 * without loading the product library. Multi-threaded over planes.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>

#include "../paper_1806_08741_b200/csrc/synth_gen.h"

typedef struct {
  const SynthSpec* s;
  const SynthSeed* table;
  void* out;
  int64_t lo, hi;
} Job;

static void* run(void* arg) {
  const Job* j = (const Job*)arg;
  for (int64_t li = j->lo; li < j->hi; ++li) syn_voxel(j->s, j->table, li, j->out);
  return NULL;
}

/* Planes [z_begin, z_end) of config `config` into out (host, native dtype).
 * Returns 0, or -1 for a shape the config does not define. */
int orc_synth_generate(int config, int rank, const int64_t* dims, int channels, uint64_t seed,
                       int64_t z_begin, int64_t z_end, void* out, int threads) {
  SynthSpec s;
  if (syn_spec(&s, config, rank, dims, channels, seed, z_begin, z_end) != 0) return -1;
  const int64_t nb = syn_bin_count(&s);
  SynthSeed* table = (SynthSeed*)malloc((size_t)nb * sizeof(SynthSeed));
  if (!table) return -2;
  for (int64_t i = 0; i < nb; ++i) table[i] = syn_seed(&s, i);
  const int64_t n = s.dims[0] * s.dims[1] * (s.z_end - s.z_begin);
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  pthread_t tid[256];
  Job jobs[256];
  for (int t = 0; t < threads; ++t) {
    jobs[t].s = &s;
    jobs[t].table = table;
    jobs[t].out = out;
    jobs[t].lo = n * t / threads;
    jobs[t].hi = n * (t + 1) / threads;
    pthread_create(&tid[t], NULL, run, &jobs[t]);
  }
  for (int t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
  free(table);
  return 0;
}
