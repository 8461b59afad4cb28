// Host-side resources of the host-buffer executor; see host_runtime.h.
#include "host_runtime.h"

#include <algorithm>
#include <atomic>
#include <cerrno>
#include <chrono>
#include <cstdio>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <mutex>
#include <thread>
#include <unordered_map>

#include <emmintrin.h>
#include <sys/mman.h>

#include "../../include/moa_b200.h"

namespace moa::host {
namespace {

// ------------------------------------------------------------- copy threads
class Workers {
 public:
  explicit Workers(int n) {
    for (int i = 0; i < n; i++) threads_.emplace_back([this] { loop(); });
  }
  int size() const { return (int)threads_.size(); }

  void run(int n, const std::function<void(int)>& fn) {
    if (n <= 0) return;
    if (n == 1 || threads_.empty()) {
      for (int i = 0; i < n; i++) fn(i);
      return;
    }
    Job job{&fn, n};
    {
      std::lock_guard<std::mutex> lk(mu_);
      jobs_.push_back(&job);
    }
    cv_.notify_all();
    for (;;) {  // the caller works too
      int i;
      {
        std::lock_guard<std::mutex> lk(mu_);
        i = job.next++;
      }
      if (i >= n) break;
      fn(i);
      job.finished.fetch_add(1, std::memory_order_acq_rel);
    }
    std::unique_lock<std::mutex> lk(mu_);
    auto it = std::find(jobs_.begin(), jobs_.end(), &job);
    if (it != jobs_.end()) jobs_.erase(it);
    done_.wait(lk, [&] { return job.finished.load(std::memory_order_acquire) == n; });
  }

 private:
  struct Job {
    const std::function<void(int)>* fn;
    int n;
    int next = 0;  // guarded by mu_
    std::atomic<int> finished{0};
  };

  void loop() {
    std::unique_lock<std::mutex> lk(mu_);
    for (;;) {
      cv_.wait(lk, [&] { return !jobs_.empty(); });
      Job* job = jobs_.front();
      const int i = job->next++;
      if (i >= job->n) {  // exhausted: drop it so the next job is seen
        jobs_.pop_front();
        continue;
      }
      lk.unlock();
      (*job->fn)(i);
      const int f = job->finished.fetch_add(1, std::memory_order_acq_rel) + 1;
      const bool last = f == job->n;  // job may be gone once finished == n
      lk.lock();
      if (last) done_.notify_all();
    }
  }

  std::mutex mu_;
  std::condition_variable cv_, done_;
  std::deque<Job*> jobs_;
  std::vector<std::thread> threads_;
};

Workers& workers() {
  static Workers* w = [] {
    int n = (int)std::thread::hardware_concurrency();
    if (const char* e = std::getenv("MOA_HOST_COPY_THREADS")) n = std::atoi(e) + 1;
    n = std::max(1, std::min(n, 16)) - 1;  // + the calling thread
    return new Workers(n);                 // lives for the process
  }();
  return *w;
}

// -------------------------------------------------------------- per device
// staging geometry: slot size and slots per transfer ($MOA_HOST_SLOT_MB,
// $MOA_HOST_SLOTS override them); at most 256 MiB of slots per GPU
size_t env_or(const char* name, size_t dflt) {
  const char* e = std::getenv(name);
  return e ? (size_t)std::strtoull(e, nullptr, 10) : dflt;
}
const size_t kSlotBytes = env_or("MOA_HOST_SLOT_MB", 16) << 20;
const int kSlotsPerTransfer = (int)env_or("MOA_HOST_SLOTS", 4);
const int kMaxSlots = (int)std::max<size_t>(kSlotsPerTransfer, (256ull << 20) / kSlotBytes);
constexpr size_t kDirectBytes = 256ull << 10;
constexpr size_t kPrefaultBytes = 32ull << 20;  // pageable destinations this large are prefaulted
constexpr size_t kCacheLimit = 16ull << 20;  // per cached device buffer

struct Slot {
  char* ptr;
  cudaEvent_t ev;  // recorded after the slot's last device copy
};

struct DeviceState {
  std::mutex mu;
  std::condition_variable slot_cv;
  std::vector<Queues*> free_queues;
  std::vector<Slot> free_slots;
  int slots_total = 0;
  cudaMemPool_t pool = nullptr;
};

DeviceState& state(int device) {
  static DeviceState states[64];
  return states[device & 63];
}

// slots for one transfer: at least one (waiting if every slot is busy), at
// most `want`; each is free of pending device copies on return
std::vector<Slot> acquire(int device, int want, cudaError_t& err) {
  DeviceState& ds = state(device);
  std::vector<Slot> got;
  std::unique_lock<std::mutex> lk(ds.mu);
  ds.slot_cv.wait(lk, [&] { return !ds.free_slots.empty() || ds.slots_total < kMaxSlots; });
  while ((int)got.size() < want) {
    if (!ds.free_slots.empty()) {
      got.push_back(ds.free_slots.back());
      ds.free_slots.pop_back();
    } else if (ds.slots_total < kMaxSlots) {
      Slot s{nullptr, nullptr};
      cudaError_t e = cudaHostAlloc(reinterpret_cast<void**>(&s.ptr), kSlotBytes,
                                    cudaHostAllocPortable);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&s.ev, cudaEventDisableTiming);
      if (e != cudaSuccess) {
        if (s.ptr) cudaFreeHost(s.ptr);
        if (got.empty()) err = e;
        break;
      }
      ds.slots_total++;
      got.push_back(s);
    } else {
      break;
    }
  }
  lk.unlock();
  for (const Slot& s : got) {
    const cudaError_t e = cudaEventSynchronize(s.ev);
    if (e != cudaSuccess && err == cudaSuccess) err = e;
  }
  return got;
}

void release(int device, std::vector<Slot>& slots) {
  DeviceState& ds = state(device);
  {
    std::lock_guard<std::mutex> lk(ds.mu);
    for (const Slot& s : slots) ds.free_slots.push_back(s);
  }
  ds.slot_cv.notify_all();
  slots.clear();
}

// One chunk of a 2-D transfer that fits a slot: rows [r0, r0+nr) and bytes
// [c0, c0+cw) of each row (cw == width unless one row exceeds a slot).
struct Chunk {
  size_t r0, nr, c0, cw;
};

std::vector<Chunk> chunks_of(size_t width, size_t rows) {
  std::vector<Chunk> out;
  if (width == 0 || rows == 0) return out;
  if (width <= kSlotBytes) {
    const size_t per = kSlotBytes / width;
    for (size_t r = 0; r < rows; r += per) out.push_back({r, std::min(per, rows - r), 0, width});
  } else {
    for (size_t r = 0; r < rows; r++)
      for (size_t c = 0; c < width; c += kSlotBytes)
        out.push_back({r, 1, c, std::min(kSlotBytes, width - c)});
  }
  return out;
}

// Copy into a staging slot with non-temporal (streaming) stores.  The copy
// engine reads the slot right after the threads write it; lines left dirty in
// the 16 cores' private caches make those DMA reads snoop-bound — 7 GB/s
// instead of 54 GB/s for a 16 MiB slot packed by 16 threads
// (tools/host_probe.cu, profiles/r02_host_probe.json) — so the packed data
// goes straight to memory instead.
void stream_copy(char* dst, const char* src, size_t n) {
  size_t head = (16 - reinterpret_cast<uintptr_t>(dst) % 16) % 16;
  if (head > n) head = n;
  std::memcpy(dst, src, head);
  dst += head;
  src += head;
  n -= head;
  const size_t body = n / 64 * 64;
  for (size_t i = 0; i < body; i += 64) {
    const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i));
    const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 16));
    const __m128i c = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 32));
    const __m128i d = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 48));
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i), a);
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 16), b);
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 32), c);
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 48), d);
  }
  std::memcpy(dst + body, src + body, n - body);
}

// copy a chunk between the slot (dense, pitch cw) and host rows (pitch hp),
// split over the copy threads in >= 1 MiB pieces
void pack(char* slot, const char* host, size_t hp, const Chunk& ch, bool to_slot) {
  const size_t total = ch.nr * ch.cw;
  const int pieces = (int)std::min<size_t>(
      (size_t)workers().size() + 1, std::max<size_t>(1, total / (1ull << 20)));
  const size_t per = (total + pieces - 1) / pieces;
  parallel_for(pieces, [&](int p) {
    size_t b = (size_t)p * per;
    const size_t e = std::min(total, b + per);
    while (b < e) {
      const size_t r = b / ch.cw, c = b % ch.cw;
      const size_t n = std::min(ch.cw - c, e - b);
      char* s = slot + b;
      char* h = const_cast<char*>(host) + (ch.r0 + r) * hp + ch.c0 + c;
      // streaming stores into a slot (see stream_copy); plain stores into the
      // caller's rows (streaming them measured no faster)
      if (to_slot)
        stream_copy(s, h, n);
      else
        std::memcpy(h, s, n);
      b += n;
    }
    if (to_slot) _mm_sfence();  // streaming stores visible before the copy is issued
  });
}

#ifndef MADV_POPULATE_WRITE
#define MADV_POPULATE_WRITE 23  // Linux 5.14
#endif

// A large pageable destination (a freshly allocated numpy result: untouched
// 4 KiB pages) is faulted in before the copy-back reaches it: huge pages
// advised over its 2 MiB-aligned interior, then populated writable by the
// copy threads in parallel (MADV_POPULATE_WRITE keeps the contents, so rows
// of other callers inside the span are safe).  Without it the copy-back into
// fresh memory ran at ~5 GB/s, page faults serialising the copy threads
// (profiles/r02_host_probe.json d2h_pageable_fresh_GBs).  On kernels without
// MADV_POPULATE_WRITE only the advice is given.
void prefault_destination(char* lo, char* hi) {
  constexpr uintptr_t kHuge = 2ull << 20, kPage = 4096;
  const uintptr_t a = (reinterpret_cast<uintptr_t>(lo) + kHuge - 1) & ~(kHuge - 1);
  const uintptr_t b = reinterpret_cast<uintptr_t>(hi) & ~(kHuge - 1);
  if (b > a) (void)madvise(reinterpret_cast<void*>(a), b - a, MADV_HUGEPAGE);
  const uintptr_t p0 = reinterpret_cast<uintptr_t>(lo) & ~(kPage - 1);
  const uintptr_t p1 = (reinterpret_cast<uintptr_t>(hi) + kPage - 1) & ~(kPage - 1);
  if (p1 <= p0) return;
  static std::atomic<bool> unsupported{false};
  if (unsupported.load(std::memory_order_relaxed)) return;
  const int parts = std::max(1, copy_threads());
  const uintptr_t per = ((p1 - p0) / parts + kHuge - 1) & ~(kHuge - 1);
  parallel_for(parts, [&](int i) {
    const uintptr_t s0 = p0 + (uintptr_t)i * per;
    if (s0 >= p1 || unsupported.load(std::memory_order_relaxed)) return;
    const uintptr_t s1 = std::min(p1, s0 + per);
    if (madvise(reinterpret_cast<void*>(s0), s1 - s0, MADV_POPULATE_WRITE) != 0 && errno == EINVAL)
      unsupported.store(true, std::memory_order_relaxed);
  });
}

// $MOA_HOST_TRACE: per staged transfer, time packing vs waiting for slots
struct StageTrace {
  const bool on = std::getenv("MOA_HOST_TRACE") != nullptr;
  double pack_ms = 0, wait_ms = 0, prefault_ms = 0;
  size_t bytes = 0;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  const char* dir;
  explicit StageTrace(const char* d) : dir(d) {}
  static double since(std::chrono::steady_clock::time_point t) {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t).count();
  }
  ~StageTrace() {
    if (on && bytes)
      fprintf(stderr, "[moa_stage] %s %.1f MiB total=%.2f ms pack=%.2f wait=%.2f prefault=%.2f -> %.1f GB/s\n",
              dir, bytes / 1048576.0, since(t0), pack_ms, wait_ms, prefault_ms, bytes / since(t0) / 1e6);
  }
};

}  // namespace

void parallel_for(int n, const std::function<void(int)>& fn) { workers().run(n, fn); }
int copy_threads() { return workers().size() + 1; }

// ------------------------------------------------------------------ queues
cudaEvent_t Queues::event(cudaError_t& err) {
  if (events_used == events.size()) {
    cudaEvent_t e = nullptr;
    const cudaError_t r = cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    if (r != cudaSuccess) {
      if (err == cudaSuccess) err = r;
      return nullptr;
    }
    events.push_back(e);
  }
  return events[events_used++];
}

void* Queues::cached_buffer(int i, size_t bytes, cudaMemPool_t pool, cudaStream_t st,
                            cudaError_t& err) {
  if (bytes == 0) bytes = 16;
  if (i < 0 || i >= kCached || bytes > kCacheLimit) return nullptr;
  if (cached_bytes[i] < bytes) {
    // stream-ordered: the old buffer's last use precedes this point on the
    // queue set, and the new one is ready on `st` before anything it orders
    if (cached[i]) cudaFreeAsync(cached[i], st);
    cached[i] = nullptr;
    cached_bytes[i] = 0;
    const size_t cap = std::max<size_t>(bytes, 1ull << 20);
    const cudaError_t r = cudaMallocFromPoolAsync(&cached[i], cap, pool, st);
    if (r != cudaSuccess) {
      if (err == cudaSuccess) err = r;
      return nullptr;
    }
    cached_bytes[i] = cap;
  }
  return cached[i];
}

Queues* checkout(int device, cudaError_t& err) {
  DeviceState& ds = state(device);
  {
    std::lock_guard<std::mutex> lk(ds.mu);
    if (!ds.free_queues.empty()) {
      Queues* q = ds.free_queues.back();
      ds.free_queues.pop_back();
      q->events_used = 0;
      return q;
    }
  }
  Queues* q = new Queues();
  q->device = device;
  cudaStream_t* all[6] = {&q->s_in, &q->s_comp, &q->s_out, &q->s_aux[0], &q->s_aux[1],
                          &q->s_aux[2]};
  for (cudaStream_t* s : all) {
    err = cudaStreamCreateWithFlags(s, cudaStreamNonBlocking);
    if (err != cudaSuccess) {
      for (cudaStream_t* t : all)
        if (*t) cudaStreamDestroy(*t);
      delete q;
      return nullptr;
    }
  }
  return q;
}

void checkin(Queues* q) {
  if (q == nullptr) return;
  DeviceState& ds = state(q->device);
  std::lock_guard<std::mutex> lk(ds.mu);
  ds.free_queues.push_back(q);
}

cudaMemPool_t device_pool(int device, cudaError_t& err) {
  DeviceState& ds = state(device);
  std::lock_guard<std::mutex> lk(ds.mu);
  if (ds.pool == nullptr) {
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.handleTypes = cudaMemHandleTypeNone;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = device;
    cudaMemPool_t pool = nullptr;
    err = cudaMemPoolCreate(&pool, &props);
    if (err != cudaSuccess) return nullptr;
    // keep up to 16 GiB mapped between calls (9% of a B200): the streamed
    // schedule of a 16384^3 float64 product alone holds 4 GiB of block
    // buffers, and a threshold at its working set made every call unmap at
    // its final synchronize and map again in the next (+15-45 ms per c4 call)
    uint64_t keep = 16ull << 30;
    if (const char* e = std::getenv("MOA_HOST_POOL_KEEP_BYTES")) keep = std::strtoull(e, nullptr, 10);
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    ds.pool = pool;
  }
  return ds.pool;
}

bool is_pinned(const void* p) {
  if (p == nullptr) return false;
  cudaPointerAttributes attr;
  if (cudaPointerGetAttributes(&attr, p) != cudaSuccess) {
    (void)cudaGetLastError();
    return false;
  }
  return attr.type == cudaMemoryTypeHost;
}

void* device_view(void* p) {
  if (p == nullptr) return nullptr;
  cudaPointerAttributes attr;
  if (cudaPointerGetAttributes(&attr, p) != cudaSuccess) {
    (void)cudaGetLastError();
    return nullptr;
  }
  return attr.type == cudaMemoryTypeHost ? attr.devicePointer : nullptr;
}

// ---------------------------------------------------------------- transfers
cudaError_t h2d(int device, void* dst, size_t dpitch, const void* src, size_t hpitch,
                size_t width, size_t rows, bool pinned, cudaStream_t st) {
  if (width == 0 || rows == 0) return cudaSuccess;
  if (pinned || width * rows <= kDirectBytes)
    return cudaMemcpy2DAsync(dst, dpitch, src, hpitch, width, rows, cudaMemcpyHostToDevice, st);
  const std::vector<Chunk> chunks = chunks_of(width, rows);
  cudaError_t err = cudaSuccess;
  std::vector<Slot> slots =
      acquire(device, (int)std::min<size_t>(kSlotsPerTransfer, chunks.size()), err);
  if (slots.empty()) return err != cudaSuccess ? err : cudaErrorMemoryAllocation;
  const size_t d = slots.size();
  StageTrace tr("h2d");
  tr.bytes = width * rows;
  for (size_t c = 0; c < chunks.size() && err == cudaSuccess; c++) {
    Slot& s = slots[c % d];
    auto t = std::chrono::steady_clock::now();
    if (c >= d) err = cudaEventSynchronize(s.ev);  // its previous chunk has left
    tr.wait_ms += StageTrace::since(t);
    if (err != cudaSuccess) break;
    const Chunk& ch = chunks[c];
    t = std::chrono::steady_clock::now();
    pack(s.ptr, static_cast<const char*>(src), hpitch, ch, true);
    tr.pack_ms += StageTrace::since(t);
    char* d = static_cast<char*>(dst) + ch.r0 * dpitch + ch.c0;
    err = dpitch == ch.cw
              ? cudaMemcpyAsync(d, s.ptr, ch.cw * ch.nr, cudaMemcpyHostToDevice, st)
              : cudaMemcpy2DAsync(d, dpitch, s.ptr, ch.cw, ch.cw, ch.nr, cudaMemcpyHostToDevice, st);
    if (err == cudaSuccess) err = cudaEventRecord(s.ev, st);
  }
  release(device, slots);  // the next user of a slot waits for its event
  return err;
}

cudaError_t d2h(int device, void* dst, size_t hpitch, const void* src, size_t dpitch,
                size_t width, size_t rows, bool pinned, cudaStream_t st) {
  if (width == 0 || rows == 0) return cudaSuccess;
  if (pinned)
    return cudaMemcpy2DAsync(dst, hpitch, src, dpitch, width, rows, cudaMemcpyDeviceToHost, st);
  if (width * rows <= kDirectBytes) {
    cudaError_t e =
        cudaMemcpy2DAsync(dst, hpitch, src, dpitch, width, rows, cudaMemcpyDeviceToHost, st);
    return e == cudaSuccess ? cudaStreamSynchronize(st) : e;
  }
  const std::vector<Chunk> chunks = chunks_of(width, rows);
  cudaError_t err = cudaSuccess;
  std::vector<Slot> slots =
      acquire(device, (int)std::min<size_t>(kSlotsPerTransfer, chunks.size()), err);
  if (slots.empty()) return err != cudaSuccess ? err : cudaErrorMemoryAllocation;
  const size_t d = slots.size();
  auto issue = [&](size_t c) {
    const Chunk& ch = chunks[c];
    Slot& s = slots[c % d];
    const char* d = static_cast<const char*>(src) + ch.r0 * dpitch + ch.c0;
    cudaError_t e = dpitch == ch.cw
                        ? cudaMemcpyAsync(s.ptr, d, ch.cw * ch.nr, cudaMemcpyDeviceToHost, st)
                        : cudaMemcpy2DAsync(s.ptr, ch.cw, d, dpitch, ch.cw, ch.nr,
                                            cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaEventRecord(s.ev, st);
    if (e != cudaSuccess && err == cudaSuccess) err = e;
  };
  for (size_t c = 0; c < d && c < chunks.size(); c++) issue(c);
  StageTrace tr("d2h");
  tr.bytes = width * rows;
  static const bool prefault_on = [] {  // $MOA_HOST_PREFAULT=0: off, for comparisons
    const char* e = std::getenv("MOA_HOST_PREFAULT");
    return e == nullptr || std::atoi(e) != 0;
  }();
  if (prefault_on && width * rows >= kPrefaultBytes) {  // while the first chunks are on the link
    auto t = std::chrono::steady_clock::now();
    char* lo = static_cast<char*>(dst);
    prefault_destination(lo, lo + (rows - 1) * hpitch + width);
    tr.prefault_ms = StageTrace::since(t);
  }
  for (size_t c = 0; c < chunks.size() && err == cudaSuccess; c++) {
    Slot& s = slots[c % d];
    auto t = std::chrono::steady_clock::now();
    err = cudaEventSynchronize(s.ev);
    tr.wait_ms += StageTrace::since(t);
    if (err != cudaSuccess) break;
    t = std::chrono::steady_clock::now();
    pack(s.ptr, static_cast<const char*>(dst), hpitch, chunks[c], false);
    tr.pack_ms += StageTrace::since(t);
    if (c + d < chunks.size()) issue(c + d);
  }
  if (err != cudaSuccess) cudaStreamSynchronize(st);  // no copy may still target a slot
  release(device, slots);
  return err;
}

}  // namespace moa::host

// ------------------------------------------------------- host result blocks
namespace moa::host {
namespace {

constexpr size_t kHugePage = 2ull << 20;

struct HostBlock {
  char* map = nullptr;  // the mapping (one huge page longer, for alignment)
  size_t map_bytes = 0;
  char* ptr = nullptr;  // 2 MiB aligned
  size_t bytes = 0;
  bool registered = false;
};

struct HostCache {
  std::mutex mu;
  std::unordered_map<void*, HostBlock> live;
  std::deque<HostBlock> idle;  // oldest first
  size_t idle_bytes = 0;
};

HostCache& host_cache() {
  static HostCache* c = new HostCache();
  return *c;
}

size_t host_cache_cap() {
  static const size_t cap = [] {
    if (const char* e = std::getenv("MOA_HOST_CACHE_BYTES")) return (size_t)std::strtoull(e, nullptr, 10);
    return (size_t)(4ull << 30);
  }();
  return cap;
}

void destroy(HostBlock& b) {
  if (b.registered) {
    cudaHostUnregister(b.ptr);
    (void)cudaGetLastError();
  }
  munmap(b.map, b.map_bytes);
}

}  // namespace
}  // namespace moa::host

extern "C" void* moa_host_alloc(size_t bytes) {
  using namespace moa::host;
  if (bytes == 0) bytes = 1;
  const size_t size = (bytes + kHugePage - 1) / kHugePage * kHugePage;
  HostCache& hc = host_cache();
  {
    // reuse the smallest idle block that fits without wasting over a quarter
    std::lock_guard<std::mutex> lk(hc.mu);
    auto best = hc.idle.end();
    for (auto it = hc.idle.begin(); it != hc.idle.end(); ++it)
      if (it->bytes >= size && it->bytes <= size + size / 4 &&
          (best == hc.idle.end() || it->bytes < best->bytes))
        best = it;
    if (best != hc.idle.end()) {
      HostBlock b = *best;
      hc.idle.erase(best);
      hc.idle_bytes -= b.bytes;
      hc.live[b.ptr] = b;
      return b.ptr;
    }
  }
  HostBlock b;
  b.map_bytes = size + kHugePage;
  void* m = mmap(nullptr, b.map_bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
  if (m == MAP_FAILED) return nullptr;
  b.map = static_cast<char*>(m);
  b.ptr = b.map + ((kHugePage - reinterpret_cast<uintptr_t>(b.map) % kHugePage) % kHugePage);
  b.bytes = size;
  madvise(b.ptr, size, MADV_HUGEPAGE);
  // first touch by the copy threads, each a contiguous run of huge pages
  // (~60 GB/s on a 16-core B200 host vs ~10 GB/s from one thread)
  const size_t pages = size / kHugePage;
  const int parts = (int)std::min<size_t>(pages, (size_t)copy_threads());
  parallel_for(parts, [&](int p) {
    const size_t p0 = pages * p / parts, p1 = pages * (p + 1) / parts;
    for (size_t i = p0 * kHugePage; i < p1 * kHugePage; i += 4096) b.ptr[i] = 0;
  });
  // page-lock it once; from then on device copies into it run at link speed
  // with no staging (cudaHostRegister of faulted memory: ~18 ms per GiB, vs
  // ~390 ms per GiB for cudaHostAlloc)
  b.registered = cudaHostRegister(b.ptr, size, cudaHostRegisterPortable) == cudaSuccess;
  if (!b.registered) (void)cudaGetLastError();  // stays usable, staged
  std::lock_guard<std::mutex> lk(hc.mu);
  hc.live[b.ptr] = b;
  return b.ptr;
}

extern "C" void moa_host_free(void* p) {
  using namespace moa::host;
  if (p == nullptr) return;
  HostCache& hc = host_cache();
  std::vector<HostBlock> evict;
  {
    std::lock_guard<std::mutex> lk(hc.mu);
    auto it = hc.live.find(p);
    if (it == hc.live.end()) return;
    hc.idle.push_back(it->second);
    hc.idle_bytes += it->second.bytes;
    hc.live.erase(it);
    while (hc.idle_bytes > host_cache_cap() && !hc.idle.empty()) {
      evict.push_back(hc.idle.front());
      hc.idle_bytes -= hc.idle.front().bytes;
      hc.idle.pop_front();
    }
  }
  for (HostBlock& b : evict) destroy(b);
}
