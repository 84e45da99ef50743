// A small persistent worker pool for independent host loops (the per-PE
// sample streams of one level).  Workers are started on first use and park
// on a condition variable; parallel_for hands out indices through an atomic
// counter and the calling thread works too.
#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "../ams_host.h"

namespace ams {
namespace {

struct Pool {
  std::mutex mu;
  std::condition_variable cv, done_cv;
  const std::function<void(int)>* fn = nullptr;
  int n = 0;
  std::atomic<int> next{0};
  int active = 0;
  uint64_t epoch = 0;
  int nworkers = 0;

  Pool() {
    const unsigned hw = std::thread::hardware_concurrency();
    nworkers = (int)std::min<unsigned>(hw > 1 ? hw - 1 : 0, 15);
    for (int i = 0; i < nworkers; ++i) std::thread([this] { loop(); }).detach();
  }

  void drain() {
    for (int i = next.fetch_add(1); i < n; i = next.fetch_add(1)) (*fn)(i);
  }

  void loop() {
    uint64_t seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> lk(mu);
        cv.wait(lk, [&] { return epoch != seen; });
        seen = epoch;
        ++active;
      }
      drain();
      {
        std::lock_guard<std::mutex> lk(mu);
        if (--active == 0) done_cv.notify_all();
      }
    }
  }

  void run(int count, const std::function<void(int)>& f) {
    std::lock_guard<std::mutex> serial(run_mu);  // one parallel_for at a time
    {
      std::lock_guard<std::mutex> lk(mu);
      fn = &f;
      n = count;
      next.store(0);
      ++epoch;
    }
    cv.notify_all();
    drain();
    std::unique_lock<std::mutex> lk(mu);
    done_cv.wait(lk, [&] { return active == 0 && next.load() >= n; });
    fn = nullptr;
  }
  std::mutex run_mu;
};

}  // namespace

void parallel_for(int count, const std::function<void(int)>& f) {
  if (count <= 0) return;
  static Pool* pool = new Pool();  // never destroyed: workers outlive main's statics
  if (count == 1 || pool->nworkers == 0) {
    for (int i = 0; i < count; ++i) f(i);
    return;
  }
  pool->run(count, f);
}

}  // namespace ams
