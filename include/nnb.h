/* nnb.h -- C ABI of the B200 runtime (libnnb.so) behind the CompiledNN path.
 *
 * The reference crosses into native code at exactly one place: the generated
 * x86 function  void f(float *arena, const float *pool)  that
 * CompiledNetwork.apply() calls through ctypes
 *   - pkg/src/nnjit/codegen/executable.py:28      ENTRY_SIGNATURE = CFUNCTYPE(None, c_void_p, c_void_p)
 *   - pkg/src/nnjit/codegen/executable.py:34-47   ExecutableBuffer(code): map RW, copy, flip RX
 *   - pkg/src/nnjit/codegen/executable.py:49-50   ExecutableBuffer.__call__(arena, pool)
 *   - pkg/src/nnjit/runtime.py:44-49              arena + constant-pool allocation
 *   - pkg/src/nnjit/runtime.py:71-73              CompiledNetwork.apply()
 *   - pkg/src/nnjit/codegen/hostcheck.py:9-23     check_host() capability gate
 * This header replaces that boundary one-for-one:
 *   check_host()              -> nnb_device_check()
 *   ExecutableBuffer(code)    -> nnb_compile() / nnb_create()  (NVRTC -> cubin -> module)
 *   arena / pool allocation   -> nnb_create()                  (device arena, weight pool upload)
 *   entry(arena, pool)        -> nnb_apply()                   (one CUDA-graph replay)
 *   arena views               -> nnb_arena_ptr()               (device pointers for tensor views)
 *   CompiledNetwork.run(xs)   -> nnb_run_host()                (H2D, replay, D2H)
 *   ExecutableBuffer.close()  -> nnb_destroy()
 * Plain C types only; no torch or CUDA types cross the boundary (streams are
 * passed as void*).  Every call returns an nnb_status; the message of the
 * last failure on the calling thread is available from nnb_last_error().
 */
#ifndef NNB_H_
#define NNB_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NNB_ABI_VERSION 6
#define NNB_MAX_TMAPS 6

typedef enum {
  NNB_OK = 0,
  NNB_ERR_ARGUMENT = 1,     /* bad argument / descriptor                  -> ValueError      */
  NNB_ERR_NO_DRIVER = 2,    /* libcuda.so.1 missing or cuInit failed       -> UnsupportedDevice */
  NNB_ERR_NO_DEVICE = 3,    /* device index out of range                   -> UnsupportedDevice */
  NNB_ERR_ARCH = 4,         /* device is not compute capability 10.0       -> UnsupportedDevice */
  NNB_ERR_NVRTC = 5,        /* libnvrtc missing or compilation failed      -> CompileError    */
  NNB_ERR_CUDA = 6,         /* a CUDA driver call failed                   -> DeviceError     */
  NNB_ERR_OOM = 7,          /* device allocation failed                    -> DeviceError     */
  NNB_ERR_BATCH = 8         /* batch outside [1, max_batch]                -> InputShapeMismatch */
} nnb_status;

/* A float32 TMA descriptor (rank 2..4) that the runtime encodes with
 * cuTensorMapEncodeTiled once the arena and pool addresses are known.
 * Coordinates outside the tensor are zero-filled by the hardware, which is
 * how the convolution kernels get TF 'same' padding for free. */
typedef struct {
  uint32_t space;            /* 1 = arena, 2 = weight pool                    */
  uint32_t swizzle;          /* 0 none, 3 = 128-byte swizzle                  */
  uint64_t offset;           /* byte offset inside the space                 */
  uint32_t rank;             /* 2..4                                          */
  uint32_t box[4];           /* box extent per dimension (innermost first)    */
  uint64_t dims[4];          /* elements per dimension (innermost first)      */
  uint64_t strides[3];       /* bytes between consecutive indices of dims 1.. */
} nnb_tmap;

/* One kernel launch of the schedule.  The grid is
 *   grid.x = min(ceil(n * items_per_image / items_per_block) * grid_mult, grid_cap)
 * for a replay over n images (grid_cap 0 = no cap); the launch is part of the
 * replay only when n_min <= n <= n_max.  Every kernel has the signature
 *   void k(const float *pool, float *arena, int n [, TmaDesc tm0, ..., tm5])
 * with the NNB_MAX_TMAPS tensor maps present iff n_tmaps > 0 (unused trailing
 * maps are passed zeroed). */
typedef struct {
  int32_t kernel;            /* index into the kernel-name list             */
  uint32_t block;            /* threads per block                           */
  uint32_t smem_bytes;       /* dynamic shared memory                       */
  uint32_t grid_mult;
  uint64_t items_per_image;
  uint64_t items_per_block;
  int32_t n_min, n_max;
  uint32_t grid_cap;
  uint32_t n_tmaps;
  nnb_tmap tmaps[NNB_MAX_TMAPS];
  uint32_t cluster;          /* thread-block cluster size along x (0/1: none);
                              * the grid is rounded down to a multiple of it */
  uint32_t cooperative;      /* 1: co-resident grid (cooperative launch)      */
  int64_t zero_offset;       /* >= 0: arena byte offset of a uint32 set to 0
                              * (stream-ordered) right before the launch      */
} nnb_launch;

/* A network I/O tensor: byte offset in the arena and bytes per image. */
typedef struct {
  uint64_t offset;
  uint64_t image_bytes;
} nnb_io;

typedef struct {
  int32_t device;
  /* kernels: CUDA C++ translation units (compiled by NVRTC in parallel, one
   * module each) and the extern "C" kernel names with their source index */
  const char *const *sources;
  int32_t n_sources;
  const char *include_dir;   /* directory of the kernel headers               */
  const char *cache_dir;     /* cubin cache directory, NULL = no cache        */
  const char *const *kernel_names;
  const int32_t *kernel_source;
  int32_t n_kernels;
  /* schedule */
  const nnb_launch *launches;
  int32_t n_launches;
  /* memory */
  const void *pool;          /* weight pool bytes (host)                     */
  uint64_t pool_bytes;
  uint64_t arena_bytes;      /* per-image arena * capacity                   */
  int32_t max_batch;
  const nnb_io *inputs;
  int32_t n_inputs;
  const nnb_io *outputs;
  int32_t n_outputs;
} nnb_net_desc;

typedef struct nnb_net nnb_net;

/* Capability gate (replaces hostcheck.check_host): driver present, device
 * index valid, compute capability 10.x.  Any output pointer may be NULL. */
nnb_status nnb_device_check(int32_t device, int32_t *cc_major, int32_t *cc_minor,
                            int32_t *sm_count);

/* Compile a translation unit to an sm_100a cubin with NVRTC (no GPU needed).
 * When cubin_out is non-NULL it receives a malloc'd buffer the caller frees
 * with nnb_free().  Used by nnb_create() and by the CPU build check. */
nnb_status nnb_compile(const char *source, const char *include_dir, const char *cache_dir,
                       void **cubin_out, uint64_t *cubin_bytes, double *compile_ms);

/* NVRTC over n_sources translation units on up to hardware_concurrency
 * threads -- the same job pool nnb_create uses (no GPU needed).  *wall_ms is
 * the wall time, *sum_ms the sum of the per-source times (either may be NULL).
 * The CPU test-suite bounds compile() time with it. */
nnb_status nnb_compile_parallel(const char *const *sources, int32_t n_sources,
                                const char *include_dir, const char *cache_dir, double *wall_ms,
                                double *sum_ms);

/* Build a network: compile (or load from cache) the kernels a replay over
 * max_batch images runs, upload the pool, allocate and zero the arena.  The
 * kernels of other batch sizes are compiled on their first replay (or every
 * kernel up front with NNB_EAGER=1); CUDA graphs are captured lazily per
 * batch size.  Graphs over n <= NNB_PREFETCH_MAX_N images (default 16, 0 =
 * off) carry a second branch that prefetches the constant pool into L2 while
 * the first launches run (cold-start latency); NNB_PDL=0 turns programmatic
 * dependent launch off. */
nnb_status nnb_create(const nnb_net_desc *desc, nnb_net **out);

/* Device address of arena byte `offset` (for zero-copy tensor views). */
nnb_status nnb_arena_ptr(nnb_net *net, uint64_t offset, void **dptr);

/* Replay the schedule over the first n images on `stream` (CUstream or NULL
 * for the legacy default stream).  Asynchronous. */
nnb_status nnb_apply(nnb_net *net, int32_t n, void *stream);

/* Host-buffer call: copy n images of every input in, replay, copy every
 * output out, wait for completion.  inputs[i] / outputs[i] are host
 * pointers (pinned memory is fastest, see nnb_host_alloc). */
nnb_status nnb_run_host(nnb_net *net, int32_t n, const void *const *inputs,
                        void *const *outputs, void *stream);

/* nnb_run_host without the final wait (the copies and the replay are queued
 * on `stream`; the caller synchronises). */
nnb_status nnb_enqueue_host(nnb_net *net, int32_t n, const void *const *inputs,
                            void *const *outputs, void *stream);

/* Pipelined host-buffer call over k networks compiled from the same model
 * (each for >= ceil(n/k) images, same device): image chunk j of the host
 * buffers goes through nets[j] on streams[j]; every chunk is queued before
 * any is waited for, so chunk j's H2D copy overlaps chunk j-1's replay and
 * D2H copy.  Returns when all chunks are done. */
nnb_status nnb_run_host_chunked(nnb_net *const *nets, const void *const *streams, int32_t k,
                                int64_t n, const void *const *inputs, void *const *outputs);

nnb_status nnb_sync(nnb_net *net, void *stream);

/* Seconds of the last replay measured with CUDA events on `stream`:
 * nnb_time_apply replays `iters` times between two events. */
nnb_status nnb_time_apply(nnb_net *net, int32_t n, int32_t iters, void *stream, double *ms);

/* Mean milliseconds of launch `index` of the schedule run alone `iters`
 * times (no graph) -- per-kernel roofline evidence for bench.py. */
nnb_status nnb_time_launch(nnb_net *net, int32_t index, int32_t n, int32_t iters, void *stream,
                           double *ms);

/* Per-launch mean milliseconds inside a full pass over n images: the
 * schedule is enqueued directly (no graph, no PDL) with a CUDA event between
 * consecutive launches, `iters` times; ms[i] = -1 for launches not in the
 * pass.  ms must hold one entry per launch of the schedule. */
nnb_status nnb_time_sequence(nnb_net *net, int32_t n, int32_t iters, void *stream, double *ms);

/* FP32 FFMA throughput of `device` (TFLOP/s, 2 flops per FMA): a
 * microbenchmark of 16 independent FMA chains per thread, 8 blocks of 256
 * threads per SM, `iters` iterations, best of 5 timed launches (CUDA
 * events).  The measured SIMT roofline denominator (roofline.py). */
nnb_status nnb_ffma_peak(int32_t device, int32_t iters, double *tflops, double *ms);

nnb_status nnb_host_alloc(uint64_t bytes, void **ptr);
void nnb_host_free(void *ptr);
void nnb_free(void *ptr);

/* Introspection */
nnb_status nnb_net_info(nnb_net *net, uint64_t *arena_bytes, uint64_t *pool_bytes,
                        int32_t *n_kernels, double *compile_ms, int32_t *cache_hit);

const char *nnb_last_error(void);
int32_t nnb_abi_version(void);
void nnb_destroy(nnb_net *net);

#ifdef __cplusplus
}
#endif
#endif /* NNB_H_ */
