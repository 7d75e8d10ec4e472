// profile.cu — stage timing and launch counting (kvtc_profile_*, kvtc_launch_count).
#include <atomic>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "internal.h"

namespace kvtc {

static std::atomic<int64_t> g_launches{0};
static std::mutex g_mu;
static bool g_on = false;
struct Rec {
  std::string name;
  cudaEvent_t a, b;
};
static std::vector<Rec> g_recs;
static size_t g_used = 0;

void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

ProfScope::ProfScope(const char *name, cudaStream_t s) : st(s) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g_on) return;
  if (g_used == g_recs.size()) {
    Rec r;
    r.name = name;
    if (cudaEventCreate(&r.a) != cudaSuccess || cudaEventCreate(&r.b) != cudaSuccess) return;
    g_recs.push_back(r);
  }
  slot = int(g_used++);
  g_recs[slot].name = name;
  cudaEventRecord(g_recs[slot].a, st);
}
ProfScope::~ProfScope() {
  if (slot < 0) return;
  std::lock_guard<std::mutex> lk(g_mu);
  cudaEventRecord(g_recs[slot].b, st);
}

}  // namespace kvtc

using namespace kvtc;

extern "C" void kvtc_profile_enable(int32_t on) {
  std::lock_guard<std::mutex> lk(g_mu);
  g_on = on != 0;
  g_used = 0;
}

extern "C" int32_t kvtc_profile_read(char *names, size_t names_cap, double *ms, int32_t *calls, int32_t cap) {
  std::lock_guard<std::mutex> lk(g_mu);
  std::vector<std::string> keys;
  std::vector<double> tot;
  std::vector<int32_t> cnt;
  for (size_t i = 0; i < g_used; ++i) {
    cudaEventSynchronize(g_recs[i].b);
    float t = 0.f;
    if (cudaEventElapsedTime(&t, g_recs[i].a, g_recs[i].b) != cudaSuccess) continue;
    size_t k = 0;
    while (k < keys.size() && keys[k] != g_recs[i].name) ++k;
    if (k == keys.size()) {
      keys.push_back(g_recs[i].name);
      tot.push_back(0);
      cnt.push_back(0);
    }
    tot[k] += t;
    cnt[k] += 1;
  }
  size_t off = 0;
  int32_t n = 0;
  for (size_t k = 0; k < keys.size() && n < cap; ++k, ++n) {
    if (names && off + keys[k].size() + 1 <= names_cap) {
      memcpy(names + off, keys[k].c_str(), keys[k].size() + 1);
      off += keys[k].size() + 1;
    }
    if (ms) ms[n] = tot[k];
    if (calls) calls[n] = cnt[k];
  }
  return n;
}

extern "C" int64_t kvtc_launch_count(void) { return g_launches.load(); }
extern "C" void kvtc_launch_count_reset(void) { g_launches.store(0); }
