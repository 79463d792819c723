// ThreadPool contract (include/trismooth/parallel.hpp; reference proj/tests/test_parallel.cpp
// checks the same): every index of a run() is called exactly once, run() returns only after
// all calls finished, the caller participates, back-to-back runs of different sizes never
// mix, a 1-worker pool runs inline, and worker_chunk splits like the reference.
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <thread>
#include <vector>

#include "trismooth/parallel.hpp"

#define CHECK(c)                                                   \
  do {                                                             \
    if (!(c)) {                                                    \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #c); \
      std::exit(1);                                                \
    }                                                              \
  } while (0)

int main() {
  using trismooth::ThreadPool;
  using trismooth::worker_chunk;
  // worker_chunk: ceil-division chunks, trailing ones short or empty
  CHECK(worker_chunk(10, 3, 0).begin == 0 && worker_chunk(10, 3, 0).end == 4);
  CHECK(worker_chunk(10, 3, 2).begin == 8 && worker_chunk(10, 3, 2).end == 10);
  CHECK(worker_chunk(4, 8, 5).begin == 4 && worker_chunk(4, 8, 5).end == 4);
  for (int workers : {1, 2, 5, 16}) {
    ThreadPool pool(workers);
    CHECK(pool.workers() == workers);
    for (int rep = 0; rep < 2000; ++rep) {
      const int count = (rep * 7919) % 97;  // includes 0 and sizes below / above workers
      std::vector<std::atomic<int>> hits(count);
      std::atomic<int> done{0};
      pool.run(count, [&](int i) {
        hits[i].fetch_add(1);
        done.fetch_add(1);
      });
      CHECK(done.load() == count);
      for (int i = 0; i < count; ++i) CHECK(hits[i].load() == 1);
    }
    // the caller thread participates
    const auto me = std::this_thread::get_id();
    std::atomic<int> on_caller{0};
    for (int rep = 0; rep < 200 && on_caller.load() == 0; ++rep)
      pool.run(64, [&](int) {
        if (std::this_thread::get_id() == me) on_caller.fetch_add(1);
      });
    CHECK(on_caller.load() > 0);
  }
  std::puts("ok");
  return 0;
}
