// Host-side resources of the host-buffer executor; see host_runtime.h.
#include "host_runtime.h"

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <mutex>
#include <thread>

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
constexpr size_t kSlotBytes = 8ull << 20;
constexpr int kMaxSlots = 32;         // <= 256 MiB of page-locked staging per GPU
constexpr int kSlotsPerTransfer = 6;  // 48 MiB in flight per copy
constexpr size_t kDirectBytes = 256ull << 10;
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

// copy a chunk between the slot (dense, pitch cw) and host rows (pitch hp),
// split over the copy threads in ~512 KiB pieces
void pack(char* slot, const char* host, size_t hp, const Chunk& ch, bool to_slot) {
  const size_t total = ch.nr * ch.cw;
  const int pieces = (int)std::min<size_t>(
      (size_t)workers().size() + 1, std::max<size_t>(1, total / (512ull << 10)));
  const size_t per = (total + pieces - 1) / pieces;
  parallel_for(pieces, [&](int p) {
    size_t b = (size_t)p * per;
    const size_t e = std::min(total, b + per);
    while (b < e) {
      const size_t r = b / ch.cw, c = b % ch.cw;
      const size_t n = std::min(ch.cw - c, e - b);
      char* s = slot + b;
      char* h = const_cast<char*>(host) + (ch.r0 + r) * hp + ch.c0 + c;
      if (to_slot)
        std::memcpy(s, h, n);
      else
        std::memcpy(h, s, n);
      b += n;
    }
  });
}

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
    uint64_t keep = 4ull << 30;
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
  for (size_t c = 0; c < chunks.size() && err == cudaSuccess; c++) {
    Slot& s = slots[c % d];
    if (c >= d) err = cudaEventSynchronize(s.ev);  // its previous chunk has left
    if (err != cudaSuccess) break;
    const Chunk& ch = chunks[c];
    pack(s.ptr, static_cast<const char*>(src), hpitch, ch, true);
    err = cudaMemcpy2DAsync(static_cast<char*>(dst) + ch.r0 * dpitch + ch.c0, dpitch, s.ptr,
                            ch.cw, ch.cw, ch.nr, cudaMemcpyHostToDevice, st);
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
    cudaError_t e = cudaMemcpy2DAsync(s.ptr, ch.cw, static_cast<const char*>(src) + ch.r0 * dpitch + ch.c0,
                                      dpitch, ch.cw, ch.nr, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaEventRecord(s.ev, st);
    if (e != cudaSuccess && err == cudaSuccess) err = e;
  };
  for (size_t c = 0; c < d && c < chunks.size(); c++) issue(c);
  for (size_t c = 0; c < chunks.size() && err == cudaSuccess; c++) {
    Slot& s = slots[c % d];
    err = cudaEventSynchronize(s.ev);
    if (err != cudaSuccess) break;
    pack(s.ptr, static_cast<const char*>(dst), hpitch, chunks[c], false);
    if (c + d < chunks.size()) issue(c + d);
  }
  if (err != cudaSuccess) cudaStreamSynchronize(st);  // no copy may still target a slot
  release(device, slots);
  return err;
}

}  // namespace moa::host
