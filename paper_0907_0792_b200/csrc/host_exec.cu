// Host-buffer entry point: the exact drop-in for the reference's compiled loop
// _ckernel.product_rows (_ckernel.pyx:75-88), whose res/a/b are host numpy
// buffers.  moa_product_rows_host takes the same thirteen arguments with HOST
// pointers and does the whole round trip natively: the row set start::step of
// A and of res (and B) moves to the device with 2-D copies (cudaMemcpy2DAsync
// packs a strided row set densely, so no host-side gather), the product runs
// through moa_product_rows, and exactly the caller's result rows are copied
// back — so concurrent callers on disjoint row sets of one res (the
// reference's execute_parallel, parallel.py:26-43) never touch each other's
// rows.
//
// Products with one block of result (< 1 GiB) run in order on one queue, with
// two refinements for page-locked res: a write-only result of <= 1 MiB is
// stored by the kernel straight into res (no copy after the kernel), and one
// of >= 64 MiB runs as four row parts whose copy-out overlaps the next part.
// Large products are streamed (the public Python API's host path runs through
// here too, kernel.execute_host): row blocks with a 4/16 first block, three middle
// blocks and a 1/16 last block; A rows of the next block copy in on one
// stream while the current block computes on another and the previous block's
// rows copy out on a third, double-buffered.  Every row needs all of B, so B
// arrives in k-slab-aligned chunks (a ramp from ~K/32 up for K >= 1024, eight
// equal ones below) behind the first block's A rows and the
// first block is computed chunk by chunk as they land (MOA_FLAG_ACCUMULATE),
// wherever the fold replays exactly under chunked accumulation (everything but
// float32 data folded in float64).  Page-locked host buffers move with
// asynchronous copies; pageable ones (plain numpy arrays) are staged through
// page-locked slots by a small pool of host copy threads (host_runtime.cu), at
// link speed instead of the driver's 11-22 GB/s pageable path.  Streams,
// events and small device buffers come from a per-device pool of queue sets
// (one per concurrent caller), large block buffers from a private device
// memory pool, so a call costs a few API calls beyond its copies and kernels.
#include <algorithm>
#include <cstdint>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "host_runtime.h"
#include "moa_common.cuh"
#include "moa_kernels.h"
#include "../../include/moa_b200.h"

namespace moa {
void set_last_error(const std::string& msg);  // capi.cu
}

namespace {

constexpr int64_t kStreamMinOutBytes = 128ll << 20;  // stream results of >= 1 GiB (8 x this)
constexpr int64_t kRowAlign = 128;

struct Block {
  int64_t r0, r1;  // rows of the row set (0-based, in units of the set)
};

// A rows + C rows of one block: 4 GiB ($MOA_HOST_BLOCK_BYTES overrides it, so
// tests can exercise the multi-block schedules at small sizes)
int64_t max_block_bytes() {
  if (const char* e = std::getenv("MOA_HOST_BLOCK_BYTES")) {
    const long long v = std::atoll(e);
    if (v > 0) return v;
  }
  return 4ll << 30;
}

// Row blocks of the set: one block below 1 GiB of result; outer products (and
// K = 0) in equal blocks of at most max_block_bytes(), whose copy-out overlaps
// the next block's kernel; inner products as a 4/16 first block (computed per
// k-chunk of B), middle blocks, a 1/16 last block, every block within
// max_block_bytes() so device memory stays bounded (two slots of each buffer).
std::vector<Block> plan_blocks(int64_t rows, int64_t out_bytes, int64_t K, int64_t row_bytes) {
  const int64_t cap_bytes = max_block_bytes();
  if (out_bytes < 8 * kStreamMinOutBytes && out_bytes <= cap_bytes) return {{0, rows}};
  const int64_t cap_rows = cap_bytes / (row_bytes > 0 ? row_bytes : 1);
  if (K < 2) {
    if (rows <= cap_rows || cap_rows < 1) return {{0, rows}};
    const int64_t nb = (rows + cap_rows - 1) / cap_rows, size = (rows + nb - 1) / nb;
    std::vector<Block> out;
    for (int64_t r = 0; r < rows; r += size) out.push_back({r, r + size < rows ? r + size : rows});
    return out;
  }
  // first block: 4/16 of the rows (c4 through the C ABI 257.7 ms with 3/16,
  // 254.0 with 4/16, 255.0 with 5/16; c5 215.4 / 215.5 / 217.2 ms,
  // profiles/r02_e2e_first_block.log): long enough that B and the next
  // block's A rows are in before it ends; $MOA_HOST_FIRST_16THS overrides it
  int64_t first_16ths = 4;
  if (const char* e = std::getenv("MOA_HOST_FIRST_16THS"))
    first_16ths = std::min<int64_t>(12, std::max<int64_t>(1, std::atoll(e)));  // leaves room for the rest
  int64_t first = rows * first_16ths / 16, last = rows / 16;
  if (cap_rows >= kRowAlign) {
    first = first < cap_rows ? first : cap_rows;
    last = last < cap_rows ? last : cap_rows;
  }
  first -= first % kRowAlign;
  last -= last % kRowAlign;
  if (first <= 0 || last <= 0) return {{0, rows}};
  const int64_t mid = rows - first - last;
  if (mid <= 0) return {{0, rows}};
  int64_t nmid = 3;
  if (const char* e = std::getenv("MOA_HOST_MID_BLOCKS"))
    nmid = std::min<int64_t>(64, std::max<int64_t>(1, std::atoll(e)));
  const int64_t cap_aligned = cap_rows - cap_rows % kRowAlign;  // whole tiles per block
  if (cap_aligned >= kRowAlign && (mid + nmid - 1) / nmid > cap_aligned)
    nmid = (mid + cap_aligned - 1) / cap_aligned;
  int64_t size = (mid + nmid - 1) / nmid;
  size += (kRowAlign - size % kRowAlign) % kRowAlign;
  if (cap_aligned >= kRowAlign && size > cap_aligned) size = cap_aligned;
  std::vector<Block> out{{0, first}};
  for (int64_t r = first; r < rows - last; r += size)
    out.push_back({r, r + size < rows - last ? r + size : rows - last});
  out.push_back({rows - last, rows});
  return out;
}

// [0, K) in up to `chunks` ranges with inner boundaries on multiples of
// `align`; a tail shorter than `align` joins the previous range, so every
// chunk keeps the route (and fold) of the whole product (capi.cu route())
std::vector<std::pair<int64_t, int64_t>> k_chunks(int64_t K, int chunks, int64_t align) {
  if (chunks <= 1 || K <= align) return {{0, K}};
  int64_t step = (K + chunks - 1) / chunks;
  step = (step + align - 1) / align * align;
  std::vector<std::pair<int64_t, int64_t>> out;
  for (int64_t k0 = 0; k0 < K; k0 += step) out.push_back({k0, k0 + step < K ? k0 + step : K});
  if (out.size() > 1 && out.back().second - out.back().first < align) {
    out[out.size() - 2].second = K;
    out.pop_back();
  }
  return out;
}

// [0, K) as a ramp for the first block: a first chunk of ~K/32 (so its
// kernel starts after a short copy), each next one 1.25x the last (B's chunk
// plus the block's A columns copy in at >= 0.8x the speed the block computes
// them even at c4, the most copy-heavy case: 48.8 ms of copies per 61 ms of
// compute), inner boundaries on multiples of `align` and no chunk shorter
// than `align` (each keeps the whole product's route).
std::vector<std::pair<int64_t, int64_t>> ramp_chunks(int64_t K, int64_t align) {
  if (K <= 2 * align) return {{0, K}};
  const auto up = [&](double x) {
    const int64_t v = (int64_t)x;
    return std::max<int64_t>(align, (v + align - 1) / align * align);
  };
  std::vector<std::pair<int64_t, int64_t>> out;
  double size = (double)K / 32;
  for (int64_t k0 = 0; k0 < K; size *= 1.25) {
    const int64_t s = up(size);
    out.push_back({k0, k0 + s < K ? k0 + s : K});
    k0 += s;
  }
  if (out.size() > 1 && out.back().second - out.back().first < align) {
    out[out.size() - 2].second = K;
    out.pop_back();
  }
  return out;
}

bool chunk_ramp_enabled() {  // $MOA_HOST_CHUNK_RAMP=0: eight equal chunks (round 1)
  static const bool v = [] {
    const char* e = std::getenv("MOA_HOST_CHUNK_RAMP");
    return e == nullptr || std::atoi(e) != 0;
  }();
  return v;
}

// Write-only single-block products with a page-locked res up to this many
// result bytes ($MOA_HOST_DIRECT_OUT_BYTES overrides it; 0 disables) store
// their rows straight into res through its device mapping: no device result
// buffer and no D2H copy after the kernel, whose start trails the kernel by
// ~8 us.  The kernels' stores reach ~28 GB/s over PCIe against the copy
// engine's ~55, so this pays only for small results: c1 (512 KiB) 62.4 vs
// 65.7 us per call, 1024^3 f64 (8 MiB) 756 vs 560 us
// (profiles/r02_c1_e2e_probe.log).
size_t direct_out_bytes() {
  static const size_t v = [] {
    if (const char* e = std::getenv("MOA_HOST_DIRECT_OUT_BYTES")) return (size_t)std::strtoull(e, nullptr, 10);
    return (size_t)1 << 20;
  }();
  return v;
}

// Accumulating into a result that holds nothing but the reduce identity (the
// reference's _Runner prefills res with it, kernel.py:149) is the write-only
// product bit for bit (every kernel folds from the identity in registers), so
// for results of >= 32 MiB the executor checks the row set's rows first — in
// parallel, ~10 ms per GiB, stopping at the first other value — and skips
// sending res to the GPU when the check passes.
constexpr size_t kIdentityCheckBytes = 32ull << 20;

uint64_t identity_bits(int dtype, int reduce) {
  switch (dtype) {
    case MOA_DTYPE_F64: {
      const double v = reduce == moa::R_ADD ? 0.0 : reduce == moa::R_MUL ? 1.0
                       : reduce == moa::R_MIN ? __builtin_huge_val() : -__builtin_huge_val();
      uint64_t u;
      std::memcpy(&u, &v, 8);
      return u;
    }
    case MOA_DTYPE_F32: {
      const float v = reduce == moa::R_ADD ? 0.0f : reduce == moa::R_MUL ? 1.0f
                      : reduce == moa::R_MIN ? __builtin_huge_valf() : -__builtin_huge_valf();
      uint32_t u;
      std::memcpy(&u, &v, 4);
      return u;
    }
    case MOA_DTYPE_I32:
      return (uint32_t)(reduce == moa::R_ADD ? 0 : reduce == moa::R_MUL ? 1
                        : reduce == moa::R_MIN ? INT32_MAX : INT32_MIN);
    default:
      return (uint64_t)(reduce == moa::R_ADD ? int64_t(0) : reduce == moa::R_MUL ? int64_t(1)
                        : reduce == moa::R_MIN ? INT64_MAX : INT64_MIN);
  }
}

template <typename W>
bool rows_hold(const char* c_rows, size_t c_pitch, int64_t rows, int64_t n, W pat) {
  std::atomic<bool> other{false};
  const int parts = (int)std::min<int64_t>(rows, std::max(1, moa::host::copy_threads()));
  const int64_t per = (rows + parts - 1) / parts;
  moa::host::parallel_for(parts, [&](int p) {
    const int64_t r0 = p * per, r1 = std::min(rows, r0 + per);
    for (int64_t r = r0; r < r1 && !other.load(std::memory_order_relaxed); r++) {
      const W* row = reinterpret_cast<const W*>(c_rows + (size_t)r * c_pitch);
      W diff = 0;
      for (int64_t j = 0; j < n; j++) diff |= row[j] ^ pat;  // vectorises; no early exit per row
      if (diff) other.store(true, std::memory_order_relaxed);
    }
  });
  return !other.load();
}

// $MOA_HOST_ROW_PARTS=0 turns the row-part pipeline of large single-block
// results off (one kernel, then the copy-out), for comparisons
bool row_parts_enabled() {
  static const bool v = [] {
    const char* e = std::getenv("MOA_HOST_ROW_PARTS");
    return e == nullptr || std::atoi(e) != 0;
  }();
  return v;
}

// $MOA_HOST_TRACE=1: one stderr line per call with the host-side phase times
struct Trace {
  const bool on = std::getenv("MOA_HOST_TRACE") != nullptr;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  std::string line;
  void mark(const char* what) {
    if (!on) return;
    const double ms = std::chrono::duration<double, std::milli>(
                          std::chrono::steady_clock::now() - t0).count();
    char buf[64];
    snprintf(buf, sizeof buf, " %s=%.3f", what, ms);
    line += buf;
  }
  ~Trace() {
    if (on) fprintf(stderr, "[moa_host]%s\n", line.c_str());
  }
};

// one call's resources: a pooled queue set (returned at the end) and the
// block buffers drawn from the device's private pool
struct Session {
  int prev_device = -1;
  int device = -1;
  moa::host::Queues* q = nullptr;
  cudaMemPool_t pool = nullptr;
  std::vector<void*> pooled;  // freed (stream-ordered) at the end
  cudaError_t err = cudaSuccess;

  cudaEvent_t event() { return q->event(err); }
  // small buffers come from the queue set's cache; large ones from the pool
  void* alloc(int slot, size_t bytes, cudaStream_t st) {
    if (err != cudaSuccess) return nullptr;
    if (void* p = q->cached_buffer(slot, bytes, pool, st, err)) return p;
    if (err != cudaSuccess) return nullptr;
    void* p = nullptr;
    err = cudaMallocFromPoolAsync(&p, bytes ? bytes : 16, pool, st);
    if (p) pooled.push_back(p);
    return p;
  }
  void check(cudaError_t e) {
    if (err == cudaSuccess && e != cudaSuccess) err = e;
  }
  ~Session() {
    const auto t0 = std::chrono::steady_clock::now();
    if (q) {
      if (err != cudaSuccess || !pooled.empty()) {
        // drain every queue before buffers or the queue set are reused
        cudaStream_t all[6] = {q->s_in, q->s_comp, q->s_out, q->s_aux[0], q->s_aux[1], q->s_aux[2]};
        for (cudaStream_t s : all) cudaStreamSynchronize(s);
      }
      for (void* p : pooled) cudaFreeAsync(p, q->s_in);
      if (!pooled.empty()) cudaStreamSynchronize(q->s_in);
      moa::host::checkin(q);
    }
    if (prev_device >= 0 && prev_device != device) cudaSetDevice(prev_device);
    if (std::getenv("MOA_HOST_TRACE"))
      fprintf(stderr, "[moa_host] cleanup=%.3f ms\n",
              std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
  }
};

int fail_cuda(cudaError_t e, const char* what) {
  moa::set_last_error(std::string(what) + ": " + cudaGetErrorString(e));
  return (int)e;
}

}  // namespace

extern "C" int moa_product_rows_host(int dtype, void* res, const void* a, const void* b,
                                     int64_t noproc, int64_t rowsinred, int64_t elsinop,
                                     int64_t lstride, int64_t rstride, int64_t restride,
                                     int combine_code, int reduce_code, int64_t start,
                                     int64_t step, uint32_t flags, int device) {
  // argument errors: the device entry point's checks, on a call with no work
  // (so nothing is launched); then the host-layout checks
  {
    const int64_t no_work_start = start < 0 ? start : (start > noproc ? start : noproc);
    const int rc = moa_product_rows(dtype, nullptr, nullptr, nullptr, noproc, rowsinred, elsinop,
                                    lstride, rstride, restride, combine_code, reduce_code,
                                    no_work_start, step, flags, nullptr);
    if (rc != 0) return rc;
  }
  if (start >= noproc || elsinop == 0) return 0;  // surplus worker / empty rows
  bool acc = (flags & MOA_FLAG_ACCUMULATE) != 0;
  const int64_t K = rowsinred, N = elsinop;
  if (K == 0 && acc) return 0;  // the empty fold leaves res as it is
  if (res == nullptr || (K > 0 && (a == nullptr || b == nullptr))) {
    moa::set_last_error("null operand pointer");
    return MOA_E_NULL;
  }
  if (restride * step < N) {
    moa::set_last_error("result rows of the row set overlap (restride*step < elsinop)");
    return MOA_E_BOUNDS;
  }
  const size_t esz = (dtype == MOA_DTYPE_F64 || dtype == MOA_DTYPE_I64) ? 8 : 4;
  const int64_t rows = (noproc - start + step - 1) / step;

  Trace tr;
  if (acc && (size_t)(rows * N) * esz >= kIdentityCheckBytes) {
    const char* rows0 = static_cast<const char*>(res) + (size_t)(start * restride) * esz;
    const size_t pitch = (size_t)(restride * step) * esz;
    const uint64_t pat = identity_bits(dtype, reduce_code);
    const bool ident = esz == 8 ? rows_hold<uint64_t>(rows0, pitch, rows, N, pat)
                                : rows_hold<uint32_t>(rows0, pitch, rows, N, (uint32_t)pat);
    if (ident) {  // the fold from res is the fold from the identity
      acc = false;
      flags &= ~(uint32_t)MOA_FLAG_ACCUMULATE;
    }
    tr.mark(ident ? "identity_res" : "res_checked");
  }
  Session ss;
  ss.device = device;
  int cur = 0;
  if (cudaGetDevice(&cur) == cudaSuccess) ss.prev_device = cur;
  if (cur != device) {
    if (cudaError_t e = cudaSetDevice(device); e != cudaSuccess) {
      (void)cudaGetLastError();  // not sticky: do not leave it for the next launch check
      return fail_cuda(e, "cudaSetDevice");
    }
  }
  {
    cudaError_t e = cudaSuccess;
    ss.q = moa::host::checkout(device, e);
    if (ss.q == nullptr) return fail_cuda(e, "stream creation");
    ss.pool = moa::host::device_pool(device, e);
    if (ss.pool == nullptr) return fail_cuda(e, "device memory pool");
  }
  moa::host::Queues& q = *ss.q;
  tr.mark("setup");

  // A rows of the set pack densely (lda = K) when the set's rows do not
  // overlap; otherwise the whole span of A goes over with its own strides
  const bool a_dense = K == 0 || lstride * step >= K;
  const bool b_dense = K == 0 || rstride >= N;
  const char* a_rows = static_cast<const char*>(a) + (size_t)(start * lstride) * esz;
  char* c_rows = static_cast<char*>(res) + (size_t)(start * restride) * esz;
  // page-locked host buffers move with asynchronous copies; pageable ones are
  // staged through page-locked slots by the copy threads (host_runtime.cu)
  const bool a_pin = K == 0 || moa::host::is_pinned(a);
  const bool b_pin = K == 0 || moa::host::is_pinned(b);
  const bool r_pin = moa::host::is_pinned(res);
  const size_t a_pitch = (size_t)(lstride * step) * esz, c_pitch = (size_t)(restride * step) * esz;

  const bool wide = dtype == MOA_DTYPE_F32 &&
                    (reduce_code == moa::R_ADD || reduce_code == moa::R_MUL || combine_code == moa::C_MUL ||
                     combine_code == moa::C_DIV);
  std::vector<Block> blocks = (a_dense && b_dense)
                                  ? plan_blocks(rows, rows * N * (int64_t)esz, K, (K + N) * (int64_t)esz)
                                  : std::vector<Block>{{0, rows}};
  const bool chunked = blocks.size() > 1 && !wide && K >= 2;
  // long contractions ramp their chunks (c4 through the C ABI 254.1 -> 249.6
  // ms, c5 215.4 -> 214.0); short ones keep eight equal chunks, as a ramp's
  // many thin first chunks each re-read and re-write the block's C rows
  // (c3, K = 256: 20.6 vs 25.2 ms; profiles/r02_e2e_chunk_ramp.log)
  const auto chunks = !chunked ? std::vector<std::pair<int64_t, int64_t>>{{0, K}}
                     : (chunk_ramp_enabled() && K >= 1024)
                         ? ramp_chunks(K, 16)
                         : k_chunks(K, blocks.size() >= 5 ? 8 : (int)blocks.size(), 16);

  int64_t max_rows = 0;
  for (const Block& bl : blocks) max_rows = bl.r1 - bl.r0 > max_rows ? bl.r1 - bl.r0 : max_rows;
  const int64_t a_span = a_dense ? max_rows * K : ((rows - 1) * lstride * step + K);
  const int64_t b_span = b_dense ? K * N : ((K - 1) * rstride + N);
  const int64_t lda = a_dense ? K : lstride * step, ldb = b_dense ? N : rstride;

  // A of the set (dense rows, or the whole strided span), B, onto the device
  // (a column range [k0, k1) of a block's rows lands chunk-major: the nr x
  // (k1-k0) panel densely at element nr*k0, so its device copy is one
  // contiguous run — row-wise 2-D copies of narrow rows cost the copy engine
  // ~2 us per row — and the chunk's kernel reads it with lda = k1 - k0)
  auto copy_a = [&](char* dst, int64_t r0, int64_t nr, int64_t k0, int64_t k1, cudaStream_t st) {
    if (a_dense && k1 - k0 < K)
      ss.check(moa::host::h2d(device, dst + (size_t)(nr * k0) * esz, (size_t)(k1 - k0) * esz,
                              a_rows + (size_t)r0 * a_pitch + (size_t)k0 * esz, a_pitch,
                              (size_t)(k1 - k0) * esz, (size_t)nr, a_pin, st));
    else if (a_dense)
      ss.check(moa::host::h2d(device, dst, (size_t)K * esz, a_rows + (size_t)r0 * a_pitch, a_pitch,
                              (size_t)K * esz, (size_t)nr, a_pin, st));
    else
      ss.check(moa::host::h2d(device, dst, (size_t)a_span * esz, a_rows, (size_t)a_span * esz,
                              (size_t)a_span * esz, 1, a_pin, st));
  };
  auto copy_b = [&](char* dst, int64_t k0, int64_t k1, cudaStream_t st) {
    if (b_dense)
      ss.check(moa::host::h2d(device, dst + (size_t)(k0 * N) * esz, (size_t)N * esz,
                              static_cast<const char*>(b) + (size_t)(k0 * rstride) * esz,
                              (size_t)rstride * esz, (size_t)N * esz, (size_t)(k1 - k0), b_pin, st));
    else
      ss.check(moa::host::h2d(device, dst, (size_t)b_span * esz, b, (size_t)b_span * esz,
                              (size_t)b_span * esz, 1, b_pin, st));
  };

  // ---- one block: in order on one queue (page-locked B copies in on a
  // second queue; a small write-only result goes straight into page-locked
  // res; a large one into page-locked res runs as row parts)
  if (blocks.size() == 1) {
    cudaStream_t st = q.s_comp;
    const size_t out_bytes = (size_t)(rows * N) * esz;
    const bool split_in = K > 0 && a_pin && b_pin;
    cudaStream_t sb = split_in ? q.s_in : st;
    char* c_direct = (!acc && r_pin && out_bytes <= direct_out_bytes())
                         ? static_cast<char*>(moa::host::device_view(c_rows))
                         : nullptr;
    char* a_dev = static_cast<char*>(ss.alloc(0, (size_t)(K > 0 ? a_span : 0) * esz, st));
    char* b_dev = static_cast<char*>(ss.alloc(1, (size_t)(K > 0 ? b_span : 0) * esz, sb));
    char* c_dev = c_direct ? c_direct : static_cast<char*>(ss.alloc(2, out_bytes, st));
    if (ss.err != cudaSuccess) return fail_cuda(ss.err, "device buffers");
    // A large result into page-locked res: the product runs as row parts,
    // each part's rows copied out on their own queue while the next part
    // computes (its A rows, and C rows when accumulating, copied in just
    // before it), so the copy-out starts after the first part instead of the
    // whole kernel.  Row parts never change the route or a bit (capi.cu
    // route() depends on K only).
    const bool parts = !c_direct && r_pin && rows >= 4 * kRowAlign && out_bytes >= (64ull << 20) &&
                       row_parts_enabled();
    if (parts) {
      // every copy in rides one queue in order (B, then each part's A rows /
      // C rows), each part's kernel waits for its own rows only
      cudaStream_t si = q.s_in;
      cudaEvent_t allocated = ss.event();  // buffers drawn on st are ready on si too
      ss.check(cudaEventRecord(allocated, st));
      ss.check(cudaStreamWaitEvent(si, allocated, 0));
      if (K > 0) {
        if (!a_dense) copy_a(a_dev, 0, rows, 0, K, si);
        copy_b(b_dev, 0, K, si);
      }
      int64_t per = (rows + 3) / 4;
      per += (kRowAlign - per % kRowAlign) % kRowAlign;
      for (int64_t r0 = 0; r0 < rows && ss.err == cudaSuccess; r0 += per) {
        const int64_t nr = r0 + per < rows ? per : rows - r0;
        char* c_part = c_dev + (size_t)(r0 * N) * esz;
        char* a_part = nullptr;
        if (K > 0) {
          if (a_dense) {
            a_part = a_dev + (size_t)(r0 * K) * esz;
            copy_a(a_part, r0, nr, 0, K, si);
          } else {
            a_part = a_dev + (size_t)(r0 * lda) * esz;
          }
        }
        if (acc)
          ss.check(moa::host::h2d(device, c_part, (size_t)N * esz, c_rows + (size_t)r0 * c_pitch,
                                  c_pitch, (size_t)N * esz, (size_t)nr, true, si));
        cudaEvent_t in = ss.event();
        ss.check(cudaEventRecord(in, si));
        ss.check(cudaStreamWaitEvent(st, in, 0));
        if (ss.err != cudaSuccess) break;
        const int rc = moa_product_rows(dtype, c_part, a_part, K > 0 ? b_dev : nullptr, nr, K, N,
                                        K > 0 ? lda : 0, K > 0 ? ldb : N, N, combine_code,
                                        reduce_code, 0, 1, flags, st);
        if (rc != 0) {
          ss.err = cudaErrorUnknown;  // drain before the queues are reused; message already set
          return rc;
        }
        cudaEvent_t done = ss.event();
        ss.check(cudaEventRecord(done, st));
        ss.check(cudaStreamWaitEvent(q.s_out, done, 0));
        ss.check(moa::host::d2h(device, c_rows + (size_t)r0 * c_pitch, c_pitch, c_part,
                                (size_t)N * esz, (size_t)N * esz, (size_t)nr, true, q.s_out));
      }
      tr.mark("parts_issued");
      ss.check(cudaStreamSynchronize(q.s_out));
      ss.check(cudaStreamSynchronize(st));
      tr.mark("out_parts");
      if (ss.err != cudaSuccess) return fail_cuda(ss.err, "host product");
      return 0;
    }
    if (K > 0) {
      copy_a(a_dev, 0, rows, 0, K, st);
      copy_b(b_dev, 0, K, sb);
      if (split_in) {
        cudaEvent_t b_in = ss.event();
        ss.check(cudaEventRecord(b_in, sb));
        ss.check(cudaStreamWaitEvent(st, b_in, 0));
      }
    }
    if (acc)
      ss.check(moa::host::h2d(device, c_dev, (size_t)N * esz, c_rows, c_pitch, (size_t)N * esz,
                              (size_t)rows, r_pin, st));
    if (ss.err != cudaSuccess) return fail_cuda(ss.err, "host product (copy in)");
    tr.mark("in");
    const int rc = moa_product_rows(dtype, c_dev, K > 0 ? a_dev : nullptr, K > 0 ? b_dev : nullptr,
                                    rows, K, N, K > 0 ? lda : 0, K > 0 ? ldb : N,
                                    c_direct ? restride * step : N, combine_code, reduce_code, 0, 1,
                                    flags, st);
    if (rc != 0) {
      ss.err = cudaErrorUnknown;  // drain before the queues are reused; message already set
      return rc;
    }
    tr.mark("launched");
    if (c_direct) {
      ss.check(cudaStreamSynchronize(st));
      tr.mark("out_direct");
    } else {
      ss.check(moa::host::d2h(device, c_rows, c_pitch, c_dev, (size_t)N * esz, (size_t)N * esz,
                              (size_t)rows, r_pin, st));
      ss.check(cudaStreamSynchronize(st));
    }
    tr.mark(r_pin ? "out_pinned" : "out_staged");
    if (ss.err != cudaSuccess) return fail_cuda(ss.err, "host product");
    return 0;
  }

  // ---- streamed row blocks (results of >= 1 GiB)
  char* a_buf[2] = {nullptr, nullptr};
  char* c_buf[2] = {nullptr, nullptr};
  for (int s = 0; s < 2; s++) {
    a_buf[s] = static_cast<char*>(ss.alloc(-1, (size_t)(K > 0 ? a_span : 0) * esz, q.s_in));
    c_buf[s] = static_cast<char*>(ss.alloc(-1, (size_t)(max_rows * N) * esz, q.s_in));
  }
  char* b_buf = static_cast<char*>(ss.alloc(-1, (size_t)(K > 0 ? b_span : 0) * esz, q.s_in));
  cudaEvent_t allocated = ss.event();
  ss.check(cudaEventRecord(allocated, q.s_in));
  ss.check(cudaStreamWaitEvent(q.s_comp, allocated, 0));
  ss.check(cudaStreamWaitEvent(q.s_out, allocated, 0));
  if (ss.err != cudaSuccess) return fail_cuda(ss.err, "device buffers");

  std::vector<cudaEvent_t> b_ready;
  struct RowPart {
    int64_t q0, q1;
    cudaEvent_t ready;
  };
  std::vector<RowPart> last_parts;  // the last block's row parts (if split)
  cudaEvent_t a_free[2] = {nullptr, nullptr}, c_free[2] = {nullptr, nullptr};
  std::vector<cudaEvent_t> done(blocks.size(), nullptr);

  // result rows of block i back into res: page-locked res over four copy
  // queues (asynchronous); pageable res staged by the copy threads (returns
  // when the rows are in res, while the next block computes)
  auto copy_out = [&](size_t i) {
    const Block& bl = blocks[i];
    const int slot = (int)(i % 2);
    const int64_t nr = bl.r1 - bl.r0;
    char* host_rows = c_rows + (size_t)bl.r0 * c_pitch;
    if (!r_pin) {
      ss.check(cudaStreamWaitEvent(q.s_out, done[i], 0));
      ss.check(moa::host::d2h(device, host_rows, c_pitch, c_buf[slot], (size_t)N * esz,
                              (size_t)N * esz, (size_t)nr, false, q.s_out));
    } else {
      const int parts = (nr >= 4 && nr * N * (int64_t)esz >= (64ll << 20)) ? 4 : 1;
      const int64_t per = (nr + parts - 1) / parts;
      std::vector<cudaEvent_t> joined;
      for (int p = 0; p < parts && ss.err == cudaSuccess; p++) {
        const int64_t q0 = p * per, q1 = (p + 1) * per < nr ? (p + 1) * per : nr;
        if (q0 >= q1) break;
        cudaStream_t st = p > 0 ? q.s_aux[p - 1] : q.s_out;
        ss.check(cudaStreamWaitEvent(st, done[i], 0));
        ss.check(moa::host::d2h(device, host_rows + (size_t)q0 * c_pitch, c_pitch,
                                c_buf[slot] + (size_t)(q0 * N) * esz, (size_t)N * esz,
                                (size_t)N * esz, (size_t)(q1 - q0), true, st));
        if (p > 0) {
          joined.push_back(ss.event());
          ss.check(cudaEventRecord(joined.back(), st));
        }
      }
      for (cudaEvent_t e : joined) ss.check(cudaStreamWaitEvent(q.s_out, e, 0));
    }
    c_free[slot] = ss.event();
    ss.check(cudaEventRecord(c_free[slot], q.s_out));
  };

  for (size_t i = 0; i < blocks.size() && ss.err == cudaSuccess; i++) {
    const Block& bl = blocks[i];
    const int slot = (int)(i % 2);
    const int64_t nr = bl.r1 - bl.r0;
    // --- in: this block's A rows (and res rows when accumulating), B behind block 0.
    // The first block, computed per k-chunk, takes its A rows in the same
    // k-chunks (2-D copies of a column range), each just ahead of the matching
    // B chunk, so the first kernel waits for one chunk of each, not all of A0.
    const bool a_by_chunk = i == 0 && chunks.size() > 1 && a_dense;
    if (a_free[slot]) ss.check(cudaStreamWaitEvent(q.s_in, a_free[slot], 0));
    if (K > 0 && !a_by_chunk) copy_a(a_buf[slot], bl.r0, nr, 0, K, q.s_in);
    if (acc) {
      if (c_free[slot]) ss.check(cudaStreamWaitEvent(q.s_in, c_free[slot], 0));
      ss.check(moa::host::h2d(device, c_buf[slot], (size_t)N * esz, c_rows + (size_t)bl.r0 * c_pitch,
                              c_pitch, (size_t)N * esz, (size_t)nr, r_pin, q.s_in));
    }
    cudaEvent_t a_ready = ss.event();
    ss.check(cudaEventRecord(a_ready, q.s_in));
    // --- compute, interleaved with B's chunks for the first block: each
    // chunk's kernel is issued as soon as its copies are, so a staged (host-
    // driven) transfer of B overlaps the chunks already computing
    ss.check(cudaStreamWaitEvent(q.s_comp, a_ready, 0));
    if (!acc && c_free[slot]) ss.check(cudaStreamWaitEvent(q.s_comp, c_free[slot], 0));
    if (ss.err != cudaSuccess) break;
    const bool per_chunk = i == 0 && chunks.size() > 1;
    auto launch = [&](int64_t k0, int64_t k1, bool accumulate) {
      const uint32_t f = (flags & ~MOA_FLAG_ACCUMULATE) | (accumulate ? MOA_FLAG_ACCUMULATE : 0u);
      // a_by_chunk: the chunk's A panel is dense at element nr*k0 (copy_a)
      const char* a_ptr = a_by_chunk ? a_buf[slot] + (size_t)(nr * k0) * esz
                                     : a_buf[slot] + (size_t)k0 * esz;
      return moa_product_rows(dtype, c_buf[slot], a_ptr, b_buf + (size_t)(k0 * ldb) * esz, nr,
                              k1 - k0, N, a_by_chunk ? k1 - k0 : lda, ldb, N, combine_code,
                              reduce_code, 0, 1, f, q.s_comp);
    };
    if (K > 0) {
      if (i == 0) {
        for (size_t j = 0; j < chunks.size(); j++) {
          const auto& ch = chunks[j];
          if (a_by_chunk) copy_a(a_buf[slot], bl.r0, nr, ch.first, ch.second, q.s_in);
          copy_b(b_buf, b_dense ? ch.first : 0, b_dense ? ch.second : K, q.s_in);
          b_ready.push_back(ss.event());
          ss.check(cudaEventRecord(b_ready.back(), q.s_in));
          if (per_chunk) {
            ss.check(cudaStreamWaitEvent(q.s_comp, b_ready.back(), 0));
            if (ss.err != cudaSuccess) break;
            if (const int rc = launch(ch.first, ch.second, acc || j > 0); rc != 0) {
              ss.err = cudaErrorUnknown;  // drain; message already set
              return rc;
            }
          }
        }
      }
      if (!per_chunk) {
        // blocks after the first read all of B: wait for its last chunk
        ss.check(cudaStreamWaitEvent(q.s_comp, b_ready.back(), 0));
        if (ss.err != cudaSuccess) break;
        // the last block of a DMMA product in row parts, so its copy-out (the
        // one copy left exposed) starts after a quarter of it: c4 through the
        // C ABI 249.7 -> 248.5 ms.  Not for the float32 fast folds: each part
        // re-scans B and a quarter of c5's last block is under one wave of
        // 128x128 tiles (213.7 -> 215.8 ms; profiles/r02_e2e_last_parts.log).
        const bool dmma_route = dtype == MOA_DTYPE_F64 && combine_code == moa::C_MUL &&
                                reduce_code == moa::R_ADD && !(flags & MOA_FLAG_EXACT) && K >= 8;
        if (i + 1 == blocks.size() && i > 0 && nr >= 4 * kRowAlign && dmma_route &&
            row_parts_enabled()) {
          int64_t per = (nr + 3) / 4;
          per += (kRowAlign - per % kRowAlign) % kRowAlign;
          const uint32_t f = (flags & ~MOA_FLAG_ACCUMULATE) | (acc ? MOA_FLAG_ACCUMULATE : 0u);
          for (int64_t q0 = 0; q0 < nr; q0 += per) {
            const int64_t q1 = q0 + per < nr ? q0 + per : nr;
            const int rc = moa_product_rows(dtype, c_buf[slot] + (size_t)(q0 * N) * esz,
                                            a_buf[slot] + (size_t)(q0 * lda) * esz, b_buf, q1 - q0, K,
                                            N, lda, ldb, N, combine_code, reduce_code, 0, 1, f,
                                            q.s_comp);
            if (rc != 0) {
              ss.err = cudaErrorUnknown;
              return rc;
            }
            last_parts.push_back({q0, q1, ss.event()});
            ss.check(cudaEventRecord(last_parts.back().ready, q.s_comp));
          }
        } else if (const int rc = launch(0, K, acc); rc != 0) {
          ss.err = cudaErrorUnknown;
          return rc;
        }
      }
    } else {
      const int rc = moa_product_rows(dtype, c_buf[slot], nullptr, nullptr, nr, 0, N, 0, N, N,
                                      combine_code, reduce_code, 0, 1, flags, q.s_comp);
      if (rc != 0) {
        ss.err = cudaErrorUnknown;
        return rc;
      }
    }
    done[i] = ss.event();
    ss.check(cudaEventRecord(done[i], q.s_comp));
    a_free[slot] = done[i];
    // --- out: the previous block's rows (issued after this block's kernel,
    // so a staged copy into pageable memory runs while the GPU computes)
    tr.mark("blk_issued");
    if (i > 0) {
      copy_out(i - 1);
      tr.mark("blk_out");
    }
  }
  if (ss.err == cudaSuccess && !last_parts.empty()) {
    // the last block's rows part by part, each as soon as its kernel is done
    const size_t i = blocks.size() - 1;
    char* host_rows = c_rows + (size_t)blocks[i].r0 * c_pitch;
    for (const RowPart& rp : last_parts) {
      if (ss.err != cudaSuccess) break;
      ss.check(cudaStreamWaitEvent(q.s_out, rp.ready, 0));
      ss.check(moa::host::d2h(device, host_rows + (size_t)rp.q0 * c_pitch, c_pitch,
                              c_buf[i % 2] + (size_t)(rp.q0 * N) * esz, (size_t)N * esz,
                              (size_t)N * esz, (size_t)(rp.q1 - rp.q0), r_pin, q.s_out));
    }
  } else if (ss.err == cudaSuccess) {
    copy_out(blocks.size() - 1);
  }
  if (ss.err == cudaSuccess) ss.check(cudaStreamSynchronize(q.s_out));
  if (ss.err == cudaSuccess) ss.check(cudaStreamSynchronize(q.s_comp));
  if (ss.err == cudaSuccess) ss.check(cudaStreamSynchronize(q.s_in));
  tr.mark("end");
  if (ss.err != cudaSuccess) return fail_cuda(ss.err, "host product");
  return 0;
}
