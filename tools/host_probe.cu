// Host-memory probe for the host-buffer executor's design (csrc/host_exec.cu):
// how fast fresh pageable memory can be first-touched, how fast pinned ->
// pageable memcpy runs with T threads, what direct pageable cudaMemcpy
// achieves, and what cudaHostRegister costs.  Prints one JSON object.
// Build: nvcc -O2 -std=c++17 -o tools/host_probe tools/host_probe.cu -lpthread
#include <sys/mman.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

static double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

static const size_t kBytes = 1ull << 30;

static void par(int threads, size_t bytes, void (*fn)(char*, const char*, size_t), char* dst,
                const char* src) {
  std::vector<std::thread> ts;
  size_t per = (bytes / threads + 4095) & ~size_t(4095);
  for (int t = 0; t < threads; t++) {
    size_t o = t * per;
    if (o >= bytes) break;
    size_t n = o + per > bytes ? bytes - o : per;
    ts.emplace_back(fn, dst + o, src ? src + o : nullptr, n);
  }
  for (auto& t : ts) t.join();
}

static void touch(char* d, const char*, size_t n) {
  for (size_t i = 0; i < n; i += 4096) d[i] = 1;
}
static void copy(char* d, const char* s, size_t n) { memcpy(d, s, n); }

static char* fresh(bool huge) {
  void* p = mmap(nullptr, kBytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
  if (p == MAP_FAILED) exit(2);
  if (huge) madvise(p, kBytes, MADV_HUGEPAGE);
  return static_cast<char*>(p);
}

int main() {
  std::string out = "{";
  auto add = [&](const std::string& k, double v) {
    char buf[128];
    snprintf(buf, sizeof buf, "%s\"%s\": %.2f", out.size() > 1 ? ", " : "", k.c_str(), v);
    out += buf;
  };
  add("hw_threads", std::thread::hardware_concurrency());
  // first touch of fresh anonymous memory
  for (int huge = 0; huge < 2; huge++)
    for (int t : {1, 4, 8, 16, 32}) {
      char* p = fresh(huge);
      double t0 = now();
      par(t, kBytes, touch, p, nullptr);
      double dt = now() - t0;
      munmap(p, kBytes);
      add(std::string("first_touch_") + (huge ? "thp_" : "") + std::to_string(t) + "t_GBs",
          kBytes / dt / 1e9);
    }
  // memcpy pinned -> prefaulted pageable, and pinned -> fresh pageable
  char* pin = nullptr;
  CK(cudaHostAlloc((void**)&pin, kBytes, cudaHostAllocDefault));
  memset(pin, 3, kBytes);
  char* pg = fresh(true);
  memset(pg, 1, kBytes);
  for (int t : {1, 4, 8, 16, 32}) {
    double best = 1e9;
    for (int r = 0; r < 3; r++) {
      double t0 = now();
      par(t, kBytes, copy, pg, pin);
      best = std::min(best, now() - t0);
    }
    add("memcpy_pin_to_pageable_" + std::to_string(t) + "t_GBs", kBytes / best / 1e9);
  }
  for (int t : {8, 16, 32}) {
    char* f = fresh(true);
    double t0 = now();
    par(t, kBytes, copy, f, pin);
    double dt = now() - t0;
    munmap(f, kBytes);
    add("memcpy_pin_to_fresh_thp_" + std::to_string(t) + "t_GBs", kBytes / dt / 1e9);
  }
  // device copies
  char* dev = nullptr;
  CK(cudaMalloc((void**)&dev, kBytes));
  CK(cudaMemset(dev, 0, kBytes));
  auto timed = [&](const char* name, void* dst, const void* src, cudaMemcpyKind kind) {
    double best = 1e9;
    for (int r = 0; r < 3; r++) {
      CK(cudaDeviceSynchronize());
      double t0 = now();
      CK(cudaMemcpy(dst, src, kBytes, kind));
      best = std::min(best, now() - t0);
    }
    add(name, kBytes / best / 1e9);
  };
  timed("d2h_pinned_GBs", pin, dev, cudaMemcpyDeviceToHost);
  timed("h2d_pinned_GBs", dev, pin, cudaMemcpyHostToDevice);
  timed("d2h_pageable_GBs", pg, dev, cudaMemcpyDeviceToHost);
  timed("h2d_pageable_GBs", dev, pg, cudaMemcpyHostToDevice);
  {
    char* f = fresh(true);
    double t0 = now();
    CK(cudaMemcpy(f, dev, kBytes, cudaMemcpyDeviceToHost));
    add("d2h_pageable_fresh_GBs", kBytes / (now() - t0) / 1e9);
    munmap(f, kBytes);
  }
  // host registration of prefaulted pageable memory
  {
    double t0 = now();
    CK(cudaHostRegister(pg, kBytes, cudaHostRegisterDefault));
    double reg = now() - t0;
    timed("d2h_registered_GBs", pg, dev, cudaMemcpyDeviceToHost);
    t0 = now();
    CK(cudaHostUnregister(pg));
    add("host_register_1GiB_ms", reg * 1e3);
    add("host_unregister_1GiB_ms", (now() - t0) * 1e3);
  }
  {
    char* f = fresh(true);
    double t0 = now();
    CK(cudaHostRegister(f, kBytes, cudaHostRegisterDefault));
    add("host_register_fresh_1GiB_ms", (now() - t0) * 1e3);
    CK(cudaHostUnregister(f));
    munmap(f, kBytes);
  }
  {
    double t0 = now();
    char* p2 = nullptr;
    CK(cudaHostAlloc((void**)&p2, kBytes, cudaHostAllocDefault));
    add("cuda_host_alloc_1GiB_ms", (now() - t0) * 1e3);
    t0 = now();
    CK(cudaFreeHost(p2));
    add("cuda_free_host_1GiB_ms", (now() - t0) * 1e3);
  }
  out += "}";
  printf("%s\n", out.c_str());
  return 0;
}
