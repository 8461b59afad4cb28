// Host-memory probe for the host-buffer executor's design (csrc/host_exec.cu):
// how fast fresh pageable memory can be first-touched, how fast pinned ->
// pageable memcpy runs with T threads, what direct pageable cudaMemcpy
// achieves, and what cudaHostRegister costs.  Prints one JSON object.
// Build: nvcc -O2 -std=c++17 -o tools/host_probe tools/host_probe.cu -lpthread
#include <emmintrin.h>
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
static void copy_nt(char* d, const char* s, size_t n) {  // d 16-byte aligned, n % 16 == 0
  for (size_t i = 0; i < n; i += 16)
    _mm_stream_si128(reinterpret_cast<__m128i*>(d + i),
                     _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i)));
  _mm_sfence();
}

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
  // staging pack: prefaulted 4 KiB-page source (like a numpy array) into a
  // ring of page-locked slots, T threads per slot
  {
    const size_t src_bytes = 2ull << 30;
    char* src = static_cast<char*>(mmap(nullptr, src_bytes, PROT_READ | PROT_WRITE,
                                        MAP_PRIVATE | MAP_ANONYMOUS, -1, 0));
    madvise(src, src_bytes, MADV_NOHUGEPAGE);
    par(16, src_bytes, touch, src, nullptr);
    for (size_t slot_mb : {4, 16, 64}) {
      const size_t slot = slot_mb << 20;
      char* ring = nullptr;
      CK(cudaHostAlloc((void**)&ring, 4 * slot, cudaHostAllocPortable));
      for (int t : {4, 8, 16}) {
        double t0 = now();
        for (size_t off = 0, i = 0; off < src_bytes; off += slot, i++)
          par(t, slot, copy, ring + (i % 4) * slot, src + off);
        add("pack_4k_src_slot" + std::to_string(slot_mb) + "M_" + std::to_string(t) + "t_GBs",
            src_bytes / (now() - t0) / 1e9);
      }
      CK(cudaFreeHost(ring));
    }
    // the same source advised for huge pages after the fact
    madvise(src, src_bytes, MADV_HUGEPAGE);
    munmap(src, src_bytes);
  }
  // DMA right after a CPU pack vs from a slot written long before: does the
  // copy engine slow down on freshly written (cache-dirty) pinned lines?
  {
    const size_t slot = 16ull << 20;
    char* ring = nullptr;
    CK(cudaHostAlloc((void**)&ring, 4 * slot, cudaHostAllocPortable));
    char* src = static_cast<char*>(malloc(256ull << 20));
    memset(src, 5, 256ull << 20);
    cudaStream_t st;
    CK(cudaStreamCreate(&st));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    auto dma = [&](char* from) {
      CK(cudaEventRecord(e0, st));
      CK(cudaMemcpyAsync(dev, from, slot, cudaMemcpyHostToDevice, st));
      CK(cudaEventRecord(e1, st));
      CK(cudaEventSynchronize(e1));
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      return ms;
    };
    memset(ring, 1, 4 * slot);
    float cold = 0, hot_contig = 0, hot_gather = 0;
    for (int r = 0; r < 8; r++) cold += dma(ring + (r % 4) * slot);
    for (int r = 0; r < 8; r++) {
      char* sl = ring + (r % 4) * slot;
      par(16, slot, copy, sl, src + r * slot);
      hot_contig += dma(sl);
    }
    for (int r = 0; r < 8; r++) {  // 16 KiB pieces gathered from a 128 KiB pitch
      char* sl = ring + (r % 4) * slot;
      const size_t rows = slot / 16384;
      for (size_t i = 0; i < rows; i++) memcpy(sl + i * 16384, src + (i * 131072) % (256ull << 20), 16384);
      hot_gather += dma(sl);
    }
    float hot_nt = 0;
    for (int r = 0; r < 8; r++) {  // the same contiguous pack with streaming stores
      char* sl = ring + (r % 4) * slot;
      par(16, slot, copy_nt, sl, src + r * slot);
      hot_nt += dma(sl);
    }
    add("dma16M_after_contig_pack_nt_GBs", slot * 8 / (hot_nt * 1e-3) / 1e9);
    add("dma16M_cold_slot_GBs", slot * 8 / (cold * 1e-3) / 1e9);
    add("dma16M_after_contig_pack_GBs", slot * 8 / (hot_contig * 1e-3) / 1e9);
    add("dma16M_after_gather_pack_GBs", slot * 8 / (hot_gather * 1e-3) / 1e9);
    CK(cudaFreeHost(ring));
    free(src);
  }
  out += "}";
  printf("%s\n", out.c_str());
  return 0;
}
