/*
 * moa_b200.h — C ABI of the B200 backend for the MoA generalized inner/outer
 * product (Raynolds & Mullin, arXiv 0907.0792).
 *
 * The boundary mirrors the reference backend's hot-loop contract
 *
 *   _ckernel.product_rows(res, a, b, noproc, rowsinred, elsinop,
 *                         lstride, rstride, restride,
 *                         combine_code, reduce_code, start, step)
 *   (/root/reference/pkg/src/moaprod/_ckernel.pyx:75-88, Python twin
 *    _purekernel.py:15-37, called only from kernel.py:164-165)
 *
 * argument for argument: the same loop bounds, the same flat strides, the same
 * operation codes (ops.py:52-66) and the same row set start, start+step, ...
 * The differences are the ones a device backend needs:
 *   - res/a/b are DEVICE pointers (any allocation visible to the current
 *     device; the caller owns them, as the reference's caller owns its numpy
 *     buffers, kernel.py:149);
 *   - an element type code (the reference is float64 only, arrays.py:77-78);
 *   - a flags word: by default res is WRITE-ONLY and every result element is
 *     folded from the reduce identity in registers, which is bit-identical to
 *     the reference's identity prefill (kernel.py:149) followed by the
 *     accumulate (_ckernel.pyx:51,70) but skips the prefill pass.  With
 *     MOA_FLAG_ACCUMULATE the fold starts from res's current contents exactly
 *     as the reference's product_rows does;
 *   - a cudaStream_t (as void*) on which all work is enqueued; the call is
 *     asynchronous with respect to the host, like any CUDA launch.
 *
 * Errors: 0 on success; MOA_E_* (< 0) for argument errors; a positive
 * cudaError_t value when the CUDA runtime reports one.  moa_last_error()
 * returns a thread-local message for the last failure on the calling thread.
 * Shape/plan validation stays in the host layer (kernel.py:111-135 analogue),
 * which raises the reference's exception classes before this is reached.
 *
 * All entry points are thread-safe and reentrant: there is no global mutable
 * state apart from an atomic launch counter.
 */
#ifndef MOA_B200_H
#define MOA_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* element types (the reference has float64 only, arrays.py:77-78).  Integer
   types compute exactly in two's complement: add/sub/mul wrap, divide
   truncates toward zero with x/0 = 0; min/max identities are the type's
   max/min. */
#define MOA_DTYPE_F64 0
#define MOA_DTYPE_F32 1
#define MOA_DTYPE_I32 2
#define MOA_DTYPE_I64 3

/* combine codes — identical to ops.py:52-59 and _ckernel.pyx:11-23 */
#define MOA_COMBINE_ADD 0
#define MOA_COMBINE_SUBTRACT 1
#define MOA_COMBINE_MULTIPLY 2
#define MOA_COMBINE_DIVIDE 3
#define MOA_COMBINE_MIN 4
#define MOA_COMBINE_MAX 5

/* reduce codes — identical to ops.py:61-66 and _ckernel.pyx:26-34 */
#define MOA_REDUCE_ADD 0
#define MOA_REDUCE_MULTIPLY 1
#define MOA_REDUCE_MIN 2
#define MOA_REDUCE_MAX 3

/* flags */
#define MOA_FLAG_ACCUMULATE 1u /* fold into res's existing values (reference semantics) */
#define MOA_FLAG_EXACT 2u      /* (multiply, add): reference rounding and fold order
                                  (separate multiply and add, l ascending) instead of
                                  the FP64 DMMA tensor-core path */

/* argument errors */
#define MOA_E_DTYPE (-1)
#define MOA_E_OPCODE (-2)
#define MOA_E_BOUNDS (-3) /* negative extent/stride, step < 1, start < 0 */
#define MOA_E_NULL (-4)   /* null operand pointer with non-empty work */

/*
 * Replaces _ckernel.product_rows (_ckernel.pyx:75-88).  Computes, for every
 * row i in {start, start+step, ...} below noproc and every j < elsinop,
 *
 *   res[i*restride + j] = fold_{l ascending < rowsinred} reduce(., combine(
 *                             a[l + i*lstride], b[l*rstride + j]))
 *
 * starting from the reduce identity (default) or from res (ACCUMULATE).
 * Bit-exact with the reference for every (combine, reduce) pair except
 * (multiply, add) float64 with rowsinred >= 8 and without MOA_FLAG_EXACT,
 * which runs on the FP64 tensor cores with fused multiply-adds and is
 * accurate to K*2^-52*max|A|*max|B| over the finite operands, with the
 * reference's NaN positions and infinities (signs included).  The one
 * exception to the latter is overflow near DBL_MAX: where the reference's
 * separately rounded product overflows to +-inf but the fused sum stays in
 * range (or the reverse), the two differ — MOA_FLAG_EXACT reproduces the
 * reference there too.  Below rowsinred = 8 (multiply, add) takes the exact
 * fold (the product is bound by writing res either way), so small products —
 * the reference's own random-case tests — return the reference's bits.
 * float32 operands follow the reference's upcast (arrays.py:77-78): the result
 * equals the reference's float64 result rounded to float32.
 */
int moa_product_rows(int dtype, void* res, const void* a, const void* b,
                     int64_t noproc, int64_t rowsinred, int64_t elsinop,
                     int64_t lstride, int64_t rstride, int64_t restride,
                     int combine_code, int reduce_code,
                     int64_t start, int64_t step,
                     uint32_t flags, void* stream);

/*
 * The same product with HOST buffers — the exact drop-in for
 * _ckernel.product_rows, whose res/a/b are host numpy arrays
 * (_ckernel.pyx:75-88): identical arguments and semantics to
 * moa_product_rows, with res/a/b in host memory and the CUDA device index in
 * place of the stream.  Copies the row set's A rows (packed by 2-D copies),
 * B, and with MOA_FLAG_ACCUMULATE the row set's res rows to the device, runs
 * the product, and writes back exactly res's rows start, start+step, ... (so
 * concurrent calls on disjoint row sets of one res are safe, as in the
 * reference's execute_parallel, parallel.py:26-43).  Large products are
 * streamed in row blocks with copies overlapping the kernels (page-locked host
 * buffers overlap fully; pageable ones are staged by the driver).  Blocks
 * until res holds the result.  MOA_E_BOUNDS also when the row set's result
 * rows would overlap (restride*step < elsinop).
 */
int moa_product_rows_host(int dtype, void* res, const void* a, const void* b,
                          int64_t noproc, int64_t rowsinred, int64_t elsinop,
                          int64_t lstride, int64_t rstride, int64_t restride,
                          int combine_code, int reduce_code,
                          int64_t start, int64_t step,
                          uint32_t flags, int device);

/*
 * Host memory for results (auxiliary; the reference has no counterpart — its
 * _Runner allocates res with np.full, kernel.py:149).  moa_host_alloc returns
 * `bytes` (rounded up to 2 MiB) of host memory backed by transparent huge
 * pages, first-touched by the library's copy threads and page-locked with
 * cudaHostRegister, so moa_product_rows_host writes results into it at link
 * speed without staging.  moa_host_free returns it to a process-wide cache of
 * idle blocks (reused by later allocations of a similar size; beyond
 * $MOA_HOST_CACHE_BYTES, default 4 GiB, the oldest are unregistered and
 * unmapped).  NULL on failure.  The memory is uninitialised.  Thread-safe.
 */
void* moa_host_alloc(size_t bytes);
void moa_host_free(void* p);

/* Message for the last failing call on this thread ("" if none). */
const char* moa_last_error(void);

/* ABI version (major*100 + minor). */
int moa_abi_version(void);

/* Number of CUDA devices visible to this process (0 if none or on error):
   lets a host binding spread the reference's execute_parallel workers over
   the GPUs (worker k -> device k mod count). */
int moa_device_count(void);

/* Number of CUDA kernels this library has launched in this process. */
uint64_t moa_launch_count(void);

/*
 * Which kernel moa_product_rows would run for these arguments, as a static
 * string ("outer", "fill", "dmma", "semiring_exact", "semiring_fast",
 * "semiring_dpx", "none").  "semiring_dpx": int32 (add|subtract) x (min|max),
 * exact, on the TMA tropical kernel with one DPX add-then-min/max per pair
 * when rows are 16-byte aligned (else the exact loop).
 * Host-only; launches nothing.  "semiring_fast" (float32 (add|subtract|
 * multiply) x (min|max), with or without MOA_FLAG_ACCUMULATE) means the
 * kernels that decide on the device, after a NaN/+-0/inf/sign pre-scan of the
 * operands (and of res when accumulating), whether a packed fast fold is
 * bit-exact for this data; otherwise the exact fold runs.
 */
const char* moa_plan_kernel(int dtype, int64_t noproc, int64_t rowsinred,
                            int64_t elsinop, int combine_code, int reduce_code,
                            uint32_t flags);

#ifdef __cplusplus
}
#endif

#endif /* MOA_B200_H */
