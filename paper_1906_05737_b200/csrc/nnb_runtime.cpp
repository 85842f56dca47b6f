// nnb_runtime.cpp -- native runtime behind include/nnb.h.
//
// Responsibilities:
//   * capability gate           (replaces pkg/src/nnjit/codegen/hostcheck.py:9-23)
//   * NVRTC -> sm_100a cubin, with an on-disk cache keyed by the source, the
//     kernel headers, the NVRTC version and the options
//     (replaces the x86 encoder + ExecutableBuffer, codegen/executable.py:31-62)
//   * device weight pool upload and arena allocation (runtime.py:44-49)
//   * CUDA-graph capture per batch size and replay (runtime.py:71-73)
//   * host-buffer end-to-end call (runtime.py:75-87)
//
// libcuda and libnvrtc are opened with dlopen on first use, so the library
// loads (and reports a clean status) on machines without a GPU or driver --
// that is how the CPU test-suite checks the ABI.
#include "../../include/nnb.h"

#include <cuda.h>
#include <nvrtc.h>
#include <dirent.h>
#include <dlfcn.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <mutex>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

namespace {

thread_local std::string g_err;

nnb_status fail(nnb_status st, const char *fmt, ...) {
  char buf[4096];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}

#define XSTR(x) STR_(x)
#define STR_(x) #x

// ---------------------------------------------------------------- driver ----
struct Cu {
  void *h = nullptr;
  bool ok = false;
  std::string why;
#define CU_FN(name) decltype(&name) p_##name = nullptr;
  CU_FN(cuInit) CU_FN(cuDriverGetVersion) CU_FN(cuDeviceGet) CU_FN(cuDeviceGetCount)
  CU_FN(cuDeviceGetAttribute) CU_FN(cuDevicePrimaryCtxRetain) CU_FN(cuCtxSetCurrent)
  CU_FN(cuModuleLoadData) CU_FN(cuModuleUnload) CU_FN(cuModuleGetFunction)
  CU_FN(cuFuncSetAttribute) CU_FN(cuMemAlloc) CU_FN(cuMemFree) CU_FN(cuMemcpyHtoD)
  CU_FN(cuMemsetD8) CU_FN(cuMemAllocHost) CU_FN(cuMemFreeHost) CU_FN(cuMemcpyHtoDAsync)
  CU_FN(cuMemcpyDtoHAsync) CU_FN(cuLaunchKernel) CU_FN(cuStreamCreate) CU_FN(cuStreamDestroy)
  CU_FN(cuStreamSynchronize) CU_FN(cuStreamBeginCapture) CU_FN(cuStreamEndCapture)
  CU_FN(cuGraphInstantiateWithFlags) CU_FN(cuGraphLaunch) CU_FN(cuGraphDestroy)
  CU_FN(cuGraphExecDestroy) CU_FN(cuEventCreate) CU_FN(cuEventRecord)
  CU_FN(cuEventSynchronize) CU_FN(cuEventElapsedTime) CU_FN(cuEventDestroy)
  CU_FN(cuGetErrorString) CU_FN(cuTensorMapEncodeTiled) CU_FN(cuLaunchKernelEx)
  CU_FN(cuMemsetD32Async) CU_FN(cuCtxGetCurrent) CU_FN(cuStreamWaitEvent)
#undef CU_FN
  void load() {
    const char *names[] = {"libcuda.so.1", "libcuda.so"};
    for (const char *n : names) {
      h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
      if (h) break;
    }
    if (!h) { why = "libcuda.so.1 not found (no NVIDIA driver in this process)"; return; }
#define CU_LOAD(name)                                                        \
  p_##name = reinterpret_cast<decltype(&name)>(dlsym(h, XSTR(name)));        \
  if (!p_##name) { why = "libcuda lacks " XSTR(name); return; }
    CU_LOAD(cuInit) CU_LOAD(cuDriverGetVersion) CU_LOAD(cuDeviceGet) CU_LOAD(cuDeviceGetCount)
    CU_LOAD(cuDeviceGetAttribute) CU_LOAD(cuDevicePrimaryCtxRetain) CU_LOAD(cuCtxSetCurrent)
    CU_LOAD(cuModuleLoadData) CU_LOAD(cuModuleUnload) CU_LOAD(cuModuleGetFunction)
    CU_LOAD(cuFuncSetAttribute) CU_LOAD(cuMemAlloc) CU_LOAD(cuMemFree) CU_LOAD(cuMemcpyHtoD)
    CU_LOAD(cuMemsetD8) CU_LOAD(cuMemAllocHost) CU_LOAD(cuMemFreeHost) CU_LOAD(cuMemcpyHtoDAsync)
    CU_LOAD(cuMemcpyDtoHAsync) CU_LOAD(cuLaunchKernel) CU_LOAD(cuStreamCreate)
    CU_LOAD(cuStreamDestroy) CU_LOAD(cuStreamSynchronize) CU_LOAD(cuStreamBeginCapture)
    CU_LOAD(cuStreamEndCapture) CU_LOAD(cuGraphInstantiateWithFlags) CU_LOAD(cuGraphLaunch)
    CU_LOAD(cuGraphDestroy) CU_LOAD(cuGraphExecDestroy) CU_LOAD(cuEventCreate)
    CU_LOAD(cuEventRecord) CU_LOAD(cuEventSynchronize) CU_LOAD(cuEventElapsedTime)
    CU_LOAD(cuEventDestroy) CU_LOAD(cuGetErrorString) CU_LOAD(cuTensorMapEncodeTiled)
    CU_LOAD(cuLaunchKernelEx) CU_LOAD(cuMemsetD32Async) CU_LOAD(cuCtxGetCurrent)
    CU_LOAD(cuStreamWaitEvent)
#undef CU_LOAD
    CUresult r = p_cuInit(0);
    if (r != CUDA_SUCCESS) {
      why = "cuInit failed (code " + std::to_string((int)r) + ")";
      return;
    }
    ok = true;
  }
};

// ----------------------------------------------------------------- nvrtc ----
struct Nvrtc {
  void *h = nullptr;
  bool ok = false;
  std::string why;
#define NV_FN(name) decltype(&name) p_##name = nullptr;
  NV_FN(nvrtcVersion) NV_FN(nvrtcCreateProgram) NV_FN(nvrtcCompileProgram)
  NV_FN(nvrtcGetProgramLogSize) NV_FN(nvrtcGetProgramLog) NV_FN(nvrtcGetCUBINSize)
  NV_FN(nvrtcGetCUBIN) NV_FN(nvrtcDestroyProgram) NV_FN(nvrtcGetErrorString)
#undef NV_FN
  void load() {
    std::vector<std::string> cands;
    if (const char *e = getenv("NNB_NVRTC")) cands.push_back(e);
    if (const char *c = getenv("CUDA_HOME")) cands.push_back(std::string(c) + "/lib64/libnvrtc.so.12");
    cands.push_back("/usr/local/cuda/lib64/libnvrtc.so.12");
    cands.push_back("libnvrtc.so.12");
    cands.push_back("libnvrtc.so");
    for (auto &n : cands) {
      h = dlopen(n.c_str(), RTLD_NOW | RTLD_LOCAL);
      if (h) break;
    }
    if (!h) { why = "libnvrtc.so.12 not found"; return; }
#define NV_LOAD(name)                                                        \
  p_##name = reinterpret_cast<decltype(&name)>(dlsym(h, XSTR(name)));        \
  if (!p_##name) { why = "libnvrtc lacks " XSTR(name); return; }
    NV_LOAD(nvrtcVersion) NV_LOAD(nvrtcCreateProgram) NV_LOAD(nvrtcCompileProgram)
    NV_LOAD(nvrtcGetProgramLogSize) NV_LOAD(nvrtcGetProgramLog) NV_LOAD(nvrtcGetCUBINSize)
    NV_LOAD(nvrtcGetCUBIN) NV_LOAD(nvrtcDestroyProgram) NV_LOAD(nvrtcGetErrorString)
#undef NV_LOAD
    ok = true;
  }
};

std::once_flag g_cu_once, g_nv_once;
Cu g_cu;
Nvrtc g_nv;

Cu *cu() {
  std::call_once(g_cu_once, [] { g_cu.load(); });
  return &g_cu;
}
Nvrtc *nv() {
  std::call_once(g_nv_once, [] { g_nv.load(); });
  return &g_nv;
}

#define CU_CHECK(call)                                                          \
  do {                                                                          \
    CUresult r_ = (call);                                                       \
    if (r_ != CUDA_SUCCESS) {                                                   \
      const char *s_ = "?";                                                     \
      if (cu()->p_cuGetErrorString) cu()->p_cuGetErrorString(r_, &s_);          \
      return fail(r_ == CUDA_ERROR_OUT_OF_MEMORY ? NNB_ERR_OOM : NNB_ERR_CUDA,  \
                  "%s failed: %s (%d)", #call, s_, (int)r_);                    \
    }                                                                           \
  } while (0)

// ------------------------------------------------------------- hashing ----
uint64_t fnv1a(const std::string &s, uint64_t h = 1469598103934665603ull) {
  for (unsigned char c : s) { h ^= c; h *= 1099511628211ull; }
  return h;
}

std::string read_file(const std::string &p, bool *ok) {
  std::ifstream f(p, std::ios::binary);
  if (!f) { *ok = false; return {}; }
  std::stringstream ss;
  ss << f.rdbuf();
  *ok = true;
  return ss.str();
}

std::string headers_digest(const char *dir) {
  std::vector<std::string> names;
  if (DIR *d = opendir(dir)) {
    while (dirent *e = readdir(d)) {
      std::string n = e->d_name;
      if (n.size() > 4 && (n.substr(n.size() - 4) == ".cuh" || n.substr(n.size() - 2) == ".h"))
        names.push_back(n);
    }
    closedir(d);
  }
  std::sort(names.begin(), names.end());
  std::string all;
  for (auto &n : names) {
    bool ok;
    all += n + "\n" + read_file(std::string(dir) + "/" + n, &ok);
  }
  return all;
}

const char *kArchOpt = "--gpu-architecture=sm_100a";

nnb_status compile_cubin(const char *source, const char *include_dir, const char *cache_dir,
                         const std::string &digest, std::string *cubin, double *ms, bool *hit) {
  auto t0 = std::chrono::steady_clock::now();
  *hit = false;
  Nvrtc *N = nv();
  if (!N->ok) return fail(NNB_ERR_NVRTC, "%s", N->why.c_str());
  int vmaj = 0, vmin = 0;
  N->p_nvrtcVersion(&vmaj, &vmin);
  std::string inc = std::string("--include-path=") + (include_dir ? include_dir : ".");
  std::vector<std::string> opts = {kArchOpt, "--std=c++17", inc, "--generate-line-info",
                                   "-DNNB_NVRTC=1"};
  std::string key_src = std::string(source) + "\x1f" + digest;
  for (auto &o : opts) key_src += "\x1f" + o;
  key_src += "\x1f" + std::to_string(vmaj) + "." + std::to_string(vmin);
  char key[40];
  snprintf(key, sizeof key, "%016llx%016llx", (unsigned long long)fnv1a(key_src),
           (unsigned long long)fnv1a(key_src, 0x9e3779b97f4a7c15ull));
  std::string cpath;
  if (cache_dir && *cache_dir) {
    cpath = std::string(cache_dir) + "/" + key + ".cubin";
    bool ok;
    std::string c = read_file(cpath, &ok);
    if (ok && !c.empty()) {
      *cubin = c;
      *hit = true;
      *ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
      return NNB_OK;
    }
  }
  nvrtcProgram prog;
  nvrtcResult r = N->p_nvrtcCreateProgram(&prog, source, "nnb_net.cu", 0, nullptr, nullptr);
  if (r != NVRTC_SUCCESS) return fail(NNB_ERR_NVRTC, "nvrtcCreateProgram: %s", N->p_nvrtcGetErrorString(r));
  std::vector<const char *> copts;
  for (auto &o : opts) copts.push_back(o.c_str());
  r = N->p_nvrtcCompileProgram(prog, (int)copts.size(), copts.data());
  size_t logn = 0;
  N->p_nvrtcGetProgramLogSize(prog, &logn);
  std::string log(logn, '\0');
  if (logn) N->p_nvrtcGetProgramLog(prog, &log[0]);
  if (r != NVRTC_SUCCESS) {
    N->p_nvrtcDestroyProgram(&prog);
    if (log.size() > 3500) log = log.substr(0, 3500) + "...";
    return fail(NNB_ERR_NVRTC, "NVRTC compile failed: %s", log.c_str());
  }
  size_t n = 0;
  N->p_nvrtcGetCUBINSize(prog, &n);
  cubin->assign(n, '\0');
  N->p_nvrtcGetCUBIN(prog, &(*cubin)[0]);
  N->p_nvrtcDestroyProgram(&prog);
  if (!cpath.empty()) {
    mkdir(cache_dir, 0755);
    std::string tmp = cpath + ".tmp." + std::to_string(getpid()) + "." +
                      std::to_string(std::hash<std::thread::id>()(std::this_thread::get_id()));
    {
      std::ofstream f(tmp, std::ios::binary);
      f.write(cubin->data(), (std::streamsize)cubin->size());
    }
    rename(tmp.c_str(), cpath.c_str());
  }
  *ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return NNB_OK;
}

// Makes `ctx` current for the scope of an entry point and restores the
// caller's context on every exit path: the CUDA runtime (torch) follows the
// driver's current context, so leaving a replica's context bound would move
// the caller's default device.
struct CtxScope {
  CUcontext prev = nullptr;
  bool bound = false;
  CUresult r = CUDA_SUCCESS;
  explicit CtxScope(CUcontext ctx) {
    Cu *C = cu();
    r = C->p_cuCtxGetCurrent(&prev);
    if (r == CUDA_SUCCESS && prev != ctx) {
      r = C->p_cuCtxSetCurrent(ctx);
      bound = r == CUDA_SUCCESS;
    }
  }
  ~CtxScope() {
    if (bound) cu()->p_cuCtxSetCurrent(prev);
  }
};

#define CTX_SCOPE(ctx)                                                           \
  CtxScope ctx_scope_(ctx);                                                      \
  if (ctx_scope_.r != CUDA_SUCCESS)                                              \
    return fail(NNB_ERR_CUDA, "cannot make the network's context current (%d)", (int)ctx_scope_.r);

nnb_status device_ctx(int32_t device, CUcontext *ctx, CUdevice *dev) {
  Cu *C = cu();
  if (!C->ok) return fail(NNB_ERR_NO_DRIVER, "%s", C->why.c_str());
  int count = 0;
  CU_CHECK(C->p_cuDeviceGetCount(&count));
  if (device < 0 || device >= count)
    return fail(NNB_ERR_NO_DEVICE, "device %d out of range (%d visible)", device, count);
  CU_CHECK(C->p_cuDeviceGet(dev, device));
  int maj = 0;
  CU_CHECK(C->p_cuDeviceGetAttribute(&maj, CU_DEVICE_ATTRIBUTE_COMPUTE_CAPABILITY_MAJOR, *dev));
  if (maj != 10)
    return fail(NNB_ERR_ARCH, "device %d has compute capability %d.x; kernels target sm_100a", device, maj);
  CU_CHECK(C->p_cuDevicePrimaryCtxRetain(ctx, *dev));
  return NNB_OK;
}

}  // namespace

struct nnb_net {
  int device = 0;
  // Programmatic dependent launch: the next kernel's launch and prologue
  // overlap the previous kernel's tail; griddepcontrol.wait (no early
  // trigger) keeps full-completion ordering.  Measured: -3% batch-1 replay
  // on cfg3, neutral elsewhere; an early trigger was 3-10% slower.
  // NNB_PDL=0 disables it.
  bool pdl = true;
  std::vector<std::vector<CUtensorMap>> maps;   // per launch
  CUcontext ctx = nullptr;
  // kernels are compiled lazily per batch size: nnb_create compiles the
  // sources of the launches a replay over max_batch images runs; the
  // batch-size variants for smaller n (FFMA / split-K kernels) are compiled
  // the first time such an n is replayed or timed
  std::vector<std::string> sources;
  std::string include_dir, cache_dir, digest;
  std::vector<std::string> kernel_names;
  std::vector<int32_t> kernel_source;
  std::vector<CUmodule> mods;                    // per source, null until loaded
  std::vector<CUfunction> fns;                   // per kernel, null until loaded
  std::vector<nnb_launch> launches;
  CUdeviceptr arena = 0, pool = 0;
  uint64_t arena_bytes = 0, pool_bytes = 0;
  int max_batch = 1;
  std::vector<nnb_io> inputs, outputs;
  CUstream capture_stream = nullptr;
  std::map<int, CUgraphExec> graphs;
  double compile_ms = 0;
  bool cache_hit = false;
  CUevent ev0 = nullptr, ev1 = nullptr;
  // Weight prefetch (small batches): a replay over n <= prefetch_max_n images
  // is a chain of short launches, each of which starts by pulling its weights
  // from HBM when they are not in L2 (a cold start, or other work on the GPU
  // since the last replay).  Such graphs get a second branch next to the
  // chain: one small kernel that issues prefetch.global.L2 over the whole
  // constant pool, so later layers find their weights in L2 while the first
  // layers run.  NNB_PREFETCH_MAX_N (default 16, 0 = off).
  int prefetch_max_n = 16;
  CUstream side_stream = nullptr;
  CUevent fork_ev = nullptr, join_ev = nullptr;
  CUmodule pf_mod = nullptr;
  CUfunction pf_fn = nullptr;
};

namespace {

struct CompileJob { std::string cubin, err; nnb_status st = NNB_OK; double ms = 0; bool hit = false; };

// NVRTC over `srcs` on up to hardware_concurrency threads; returns the wall
// milliseconds in *wall_ms.
void compile_parallel(const std::vector<const char *> &srcs, const char *include_dir,
                      const char *cache_dir, const std::string &digest,
                      std::vector<CompileJob> &jobs, double *wall_ms) {
  jobs.assign(srcs.size(), CompileJob());
  auto t0 = std::chrono::steady_clock::now();
  unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  unsigned nthreads = std::min<unsigned>(hw, (unsigned)std::max<size_t>(srcs.size(), 1));
  std::vector<std::thread> pool;
  std::atomic<size_t> next{0};
  for (unsigned t = 0; t < nthreads; ++t)
    pool.emplace_back([&] {
      for (size_t i = next++; i < srcs.size(); i = next++) {
        CompileJob &j = jobs[i];
        j.st = compile_cubin(srcs[i], include_dir, cache_dir, digest, &j.cubin, &j.ms, &j.hit);
        if (j.st != NNB_OK) j.err = g_err;
      }
    });
  for (auto &th : pool) th.join();
  if (wall_ms)
    *wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

bool serves(const nnb_launch &l, int n) { return n >= l.n_min && n <= l.n_max; }

// Compile (or load from the cubin cache) and load every module the launches
// of a replay over n images need; n <= 0 loads everything.  Must not run
// inside a stream capture.
nnb_status ensure_loaded(nnb_net *net, int n, double *wall_ms = nullptr, bool *all_hit = nullptr) {
  Cu *C = cu();
  std::vector<int> need;
  std::vector<char> want(net->sources.size(), 0);
  for (const nnb_launch &l : net->launches)
    if (n <= 0 || serves(l, n)) want[net->kernel_source[l.kernel]] = 1;
  for (size_t i = 0; i < want.size(); ++i)
    if (want[i] && !net->mods[i]) need.push_back((int)i);
  if (wall_ms) *wall_ms = 0;
  if (all_hit) *all_hit = true;
  if (need.empty()) return NNB_OK;
  std::vector<const char *> srcs;
  for (int i : need) srcs.push_back(net->sources[i].c_str());
  std::vector<CompileJob> jobs;
  compile_parallel(srcs, net->include_dir.c_str(),
                   net->cache_dir.empty() ? nullptr : net->cache_dir.c_str(), net->digest, jobs,
                   wall_ms);
  for (auto &j : jobs) {
    if (j.st != NNB_OK) { g_err = j.err; return j.st; }
    if (all_hit) *all_hit = *all_hit && j.hit;
  }
  for (size_t k = 0; k < need.size(); ++k) {
    CUresult r = C->p_cuModuleLoadData(&net->mods[need[k]], jobs[k].cubin.data());
    if (r != CUDA_SUCCESS) return fail(NNB_ERR_CUDA, "cuModuleLoadData failed (%d)", (int)r);
  }
  for (size_t i = 0; i < net->fns.size(); ++i) {
    const int src = net->kernel_source[i];
    if (net->fns[i] || !net->mods[src]) continue;
    CUresult r = C->p_cuModuleGetFunction(&net->fns[i], net->mods[src], net->kernel_names[i].c_str());
    if (r != CUDA_SUCCESS) return fail(NNB_ERR_CUDA, "kernel %s not in module", net->kernel_names[i].c_str());
  }
  for (const nnb_launch &l : net->launches) {
    if (!net->fns[l.kernel] || l.smem_bytes <= 48 * 1024) continue;
    CUresult r = C->p_cuFuncSetAttribute(net->fns[l.kernel], CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES,
                                         (int)l.smem_bytes);
    if (r != CUDA_SUCCESS) return fail(NNB_ERR_CUDA, "smem %u bytes rejected", l.smem_bytes);
  }
  return NNB_OK;
}

// One launch of the schedule over n images (no-op when it is not part of
// the replay for n or its grid is empty).
nnb_status launch_one(nnb_net *net, size_t li, int n, CUstream s, bool pdl) {
  Cu *C = cu();
  const nnb_launch &l = net->launches[li];
  if (n < l.n_min || n > l.n_max) return NNB_OK;
  if (!net->fns[l.kernel]) return fail(NNB_ERR_ARGUMENT, "kernel %d is not loaded for batch %d", l.kernel, n);
  {
    uint64_t items = (uint64_t)n * l.items_per_image;
    uint64_t gx = (items + l.items_per_block - 1) / l.items_per_block * l.grid_mult;
    if (l.grid_cap && gx > l.grid_cap) gx = l.grid_cap;
    const uint32_t cl = l.cluster > 1 ? l.cluster : 1;
    if (cl > 1) gx = std::max<uint64_t>(cl, gx / cl * cl);   // whole clusters
    if (gx == 0) return NNB_OK;
    if (gx > 0x7fffffffull) return fail(NNB_ERR_ARGUMENT, "grid too large (%llu)", (unsigned long long)gx);
    CUdeviceptr pool = net->pool, arena = net->arena;
    int nn = n;
    void *args[3 + NNB_MAX_TMAPS] = {&pool, &arena, &nn};
    for (uint32_t k = 0; k < l.n_tmaps; ++k) args[3 + k] = &net->maps[li][k];
    if (l.zero_offset >= 0)      // the persistent kernel's barrier counter
      CU_CHECK(C->p_cuMemsetD32Async(net->arena + (CUdeviceptr)l.zero_offset, 0, 1, s));
    if (pdl || cl > 1 || l.cooperative) {
      // programmatic dependent launch: the next kernel's CTAs are scheduled while
      // this one drains; each kernel starts with griddepcontrol.wait.
      // Clusters: CTA pairs for the tcgen05 cta_group::2 GEMM.
      CUlaunchAttribute attr[3];
      unsigned na = 0;
      if (l.cooperative) {
        attr[na].id = CU_LAUNCH_ATTRIBUTE_COOPERATIVE;
        attr[na].value.cooperative = 1;
        ++na;
      }
      if (pdl) {
        attr[na].id = CU_LAUNCH_ATTRIBUTE_PROGRAMMATIC_STREAM_SERIALIZATION;
        attr[na].value.programmaticStreamSerializationAllowed = 1;
        ++na;
      }
      if (cl > 1) {
        attr[na].id = CU_LAUNCH_ATTRIBUTE_CLUSTER_DIMENSION;
        attr[na].value.clusterDim.x = cl;
        attr[na].value.clusterDim.y = 1;
        attr[na].value.clusterDim.z = 1;
        ++na;
      }
      CUlaunchConfig cfg = {};
      cfg.gridDimX = (unsigned)gx; cfg.gridDimY = 1; cfg.gridDimZ = 1;
      cfg.blockDimX = l.block; cfg.blockDimY = 1; cfg.blockDimZ = 1;
      cfg.sharedMemBytes = l.smem_bytes;
      cfg.hStream = s;
      cfg.attrs = attr;
      cfg.numAttrs = na;
      CU_CHECK(C->p_cuLaunchKernelEx(&cfg, net->fns[l.kernel], args, nullptr));
    } else {
      CU_CHECK(C->p_cuLaunchKernel(net->fns[l.kernel], (unsigned)gx, 1, 1, l.block, 1, 1,
                                   l.smem_bytes, s, args, nullptr));
    }
  }
  return NNB_OK;
}

nnb_status enqueue(nnb_net *net, int n, CUstream s) {
  for (size_t li = 0; li < net->launches.size(); ++li) {
    nnb_status st = launch_one(net, li, n, s, net->pdl);
    if (st != NNB_OK) return st;
  }
  return NNB_OK;
}

const char *kPrefetchSrc = R"(
extern "C" __global__ void __launch_bounds__(256) nnb_l2_prefetch(const char* p, unsigned long long bytes) {
  const unsigned long long step = (unsigned long long)gridDim.x * blockDim.x * 128ull;
  for (unsigned long long off = ((unsigned long long)blockIdx.x * blockDim.x + threadIdx.x) * 128ull;
       off < bytes; off += step)
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p + off));
}
)";

// The prefetch branch of a small-batch graph (see nnb_net): forked from the
// capture stream before the first launch.  Failures only disable it.
bool prefetch_branch(nnb_net *net, int n) {
  Cu *C = cu();
  if (n > net->prefetch_max_n || net->pool_bytes < 4096 || !C->p_cuStreamWaitEvent) return false;
  if (!net->pf_fn) {
    std::string cubin;
    double cms = 0;
    bool hit = false;
    if (compile_cubin(kPrefetchSrc, ".", net->cache_dir.empty() ? nullptr : net->cache_dir.c_str(), "",
                      &cubin, &cms, &hit) != NNB_OK ||
        C->p_cuModuleLoadData(&net->pf_mod, cubin.data()) != CUDA_SUCCESS ||
        C->p_cuModuleGetFunction(&net->pf_fn, net->pf_mod, "nnb_l2_prefetch") != CUDA_SUCCESS ||
        C->p_cuStreamCreate(&net->side_stream, CU_STREAM_NON_BLOCKING) != CUDA_SUCCESS ||
        C->p_cuEventCreate(&net->fork_ev, CU_EVENT_DISABLE_TIMING) != CUDA_SUCCESS ||
        C->p_cuEventCreate(&net->join_ev, CU_EVENT_DISABLE_TIMING) != CUDA_SUCCESS) {
      net->pf_fn = nullptr;
      net->prefetch_max_n = 0;
      return false;
    }
  }
  if (C->p_cuEventRecord(net->fork_ev, net->capture_stream) != CUDA_SUCCESS ||
      C->p_cuStreamWaitEvent(net->side_stream, net->fork_ev, 0) != CUDA_SUCCESS)
    return false;
  CUdeviceptr pool = net->pool;
  unsigned long long bytes = net->pool_bytes;
  void *args[] = {&pool, &bytes};
  const unsigned blocks = (unsigned)std::min<uint64_t>(32, (bytes / 128 + 255) / 256);
  C->p_cuLaunchKernel(net->pf_fn, blocks ? blocks : 1, 1, 1, 256, 1, 1, 0, net->side_stream, args, nullptr);
  // (the side stream is now part of the capture: it must be joined before
  // the capture ends)
  return C->p_cuEventRecord(net->join_ev, net->side_stream) == CUDA_SUCCESS;
}

nnb_status graph_for(nnb_net *net, int n, CUgraphExec *out) {
  auto it = net->graphs.find(n);
  if (it != net->graphs.end()) { *out = it->second; return NNB_OK; }
  Cu *C = cu();
  nnb_status lst = ensure_loaded(net, n);
  if (lst != NNB_OK) return lst;
  CU_CHECK(C->p_cuStreamBeginCapture(net->capture_stream, CU_STREAM_CAPTURE_MODE_THREAD_LOCAL));
  const bool forked = prefetch_branch(net, n);
  nnb_status st = enqueue(net, n, net->capture_stream);
  if (forked) C->p_cuStreamWaitEvent(net->capture_stream, net->join_ev, 0);
  CUgraph g = nullptr;
  CUresult r = C->p_cuStreamEndCapture(net->capture_stream, &g);
  if (st != NNB_OK) { if (g) C->p_cuGraphDestroy(g); return st; }
  if (r != CUDA_SUCCESS) return fail(NNB_ERR_CUDA, "cuStreamEndCapture failed (%d)", (int)r);
  CUgraphExec ex = nullptr;
  r = C->p_cuGraphInstantiateWithFlags(&ex, g, 0);
  C->p_cuGraphDestroy(g);
  if (r != CUDA_SUCCESS) return fail(NNB_ERR_CUDA, "cuGraphInstantiate failed (%d)", (int)r);
  net->graphs[n] = ex;
  *out = ex;
  return NNB_OK;
}

}  // namespace

extern "C" {

int32_t nnb_abi_version(void) { return NNB_ABI_VERSION; }

const char *nnb_last_error(void) { return g_err.c_str(); }

nnb_status nnb_device_check(int32_t device, int32_t *cc_major, int32_t *cc_minor, int32_t *sm_count) {
  Cu *C = cu();
  if (!C->ok) return fail(NNB_ERR_NO_DRIVER, "%s", C->why.c_str());
  int count = 0;
  CU_CHECK(C->p_cuDeviceGetCount(&count));
  if (device < 0 || device >= count)
    return fail(NNB_ERR_NO_DEVICE, "device %d out of range (%d visible)", device, count);
  CUdevice dev;
  CU_CHECK(C->p_cuDeviceGet(&dev, device));
  int maj = 0, mnr = 0, sms = 0;
  CU_CHECK(C->p_cuDeviceGetAttribute(&maj, CU_DEVICE_ATTRIBUTE_COMPUTE_CAPABILITY_MAJOR, dev));
  CU_CHECK(C->p_cuDeviceGetAttribute(&mnr, CU_DEVICE_ATTRIBUTE_COMPUTE_CAPABILITY_MINOR, dev));
  CU_CHECK(C->p_cuDeviceGetAttribute(&sms, CU_DEVICE_ATTRIBUTE_MULTIPROCESSOR_COUNT, dev));
  if (cc_major) *cc_major = maj;
  if (cc_minor) *cc_minor = mnr;
  if (sm_count) *sm_count = sms;
  if (maj != 10)
    return fail(NNB_ERR_ARCH, "device %d has compute capability %d.%d; kernels target sm_100a",
                device, maj, mnr);
  return NNB_OK;
}

nnb_status nnb_compile(const char *source, const char *include_dir, const char *cache_dir,
                       void **cubin_out, uint64_t *cubin_bytes, double *compile_ms) {
  if (!source) return fail(NNB_ERR_ARGUMENT, "source is NULL");
  std::string cubin;
  double ms = 0;
  bool hit = false;
  std::string digest = headers_digest(include_dir ? include_dir : ".");
  nnb_status st = compile_cubin(source, include_dir, cache_dir, digest, &cubin, &ms, &hit);
  if (st != NNB_OK) return st;
  if (cubin_bytes) *cubin_bytes = cubin.size();
  if (compile_ms) *compile_ms = ms;
  if (cubin_out) {
    void *p = malloc(cubin.size());
    if (!p) return fail(NNB_ERR_OOM, "malloc(%zu) failed", cubin.size());
    memcpy(p, cubin.data(), cubin.size());
    *cubin_out = p;
  }
  return NNB_OK;
}

nnb_status nnb_compile_parallel(const char *const *sources, int32_t n_sources,
                                const char *include_dir, const char *cache_dir, double *wall_ms,
                                double *sum_ms) {
  if (!sources || n_sources < 0) return fail(NNB_ERR_ARGUMENT, "bad arguments");
  std::vector<const char *> srcs(sources, sources + n_sources);
  for (auto p : srcs)
    if (!p) return fail(NNB_ERR_ARGUMENT, "source is NULL");
  std::string digest = headers_digest(include_dir ? include_dir : ".");
  std::vector<CompileJob> jobs;
  compile_parallel(srcs, include_dir, cache_dir, digest, jobs, wall_ms);
  double sum = 0;
  for (auto &j : jobs) {
    if (j.st != NNB_OK) { g_err = j.err; return j.st; }
    sum += j.ms;
  }
  if (sum_ms) *sum_ms = sum;
  return NNB_OK;
}

// FP32 FFMA throughput microbenchmark (the SIMT roofline denominator of
// roofline.py; SURVEY.md 8(d) asked for it to be measured, not derived).
// Every thread runs 16 independent FMA chains (no dependency stalls at 8
// warps per scheduler); 8 resident 256-thread blocks per SM, `waves` grids.
static const char *kFfmaSrc = R"(
extern "C" __global__ void __launch_bounds__(256) nnb_ffma_probe(float* out, int iters, float a, float b) {
  float x[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) x[j] = threadIdx.x * 1e-3f + j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) x[j] = fmaf(x[j], a, b);
  }
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < 16; ++j) s += x[j];
  if (s == 1234.5f) out[blockIdx.x] = s;
}
)";

nnb_status nnb_ffma_peak(int32_t device, int32_t iters, double *tflops, double *ms) {
  if (!tflops || iters < 1) return fail(NNB_ERR_ARGUMENT, "bad arguments");
  CUcontext ctx;
  CUdevice dev;
  nnb_status st = device_ctx(device, &ctx, &dev);
  if (st != NNB_OK) return st;
  CTX_SCOPE(ctx)
  Cu *C = cu();
  int sms = 0;
  CU_CHECK(C->p_cuDeviceGetAttribute(&sms, CU_DEVICE_ATTRIBUTE_MULTIPROCESSOR_COUNT, dev));
  std::string cubin;
  double cms = 0;
  bool hit = false;
  st = compile_cubin(kFfmaSrc, ".", nullptr, "", &cubin, &cms, &hit);
  if (st != NNB_OK) return st;
  CUmodule mod = nullptr;
  CU_CHECK(C->p_cuModuleLoadData(&mod, cubin.data()));
  CUfunction fn = nullptr;
  CUdeviceptr out = 0;
  CUevent e0 = nullptr, e1 = nullptr;
  float best = 1e30f;
  const unsigned blocks = (unsigned)sms * 8;
  CUresult r = C->p_cuModuleGetFunction(&fn, mod, "nnb_ffma_probe");
  if (r == CUDA_SUCCESS) r = C->p_cuMemAlloc(&out, 4 * blocks);
  if (r == CUDA_SUCCESS) r = C->p_cuEventCreate(&e0, CU_EVENT_DEFAULT);
  if (r == CUDA_SUCCESS) r = C->p_cuEventCreate(&e1, CU_EVENT_DEFAULT);
  for (int rep = 0; rep < 6 && r == CUDA_SUCCESS; ++rep) {
    float a = 0.999f, b = 1e-3f;
    int it = iters;
    void *args[] = {&out, &it, &a, &b};
    r = C->p_cuEventRecord(e0, nullptr);
    if (r == CUDA_SUCCESS) r = C->p_cuLaunchKernel(fn, blocks, 1, 1, 256, 1, 1, 0, nullptr, args, nullptr);
    if (r == CUDA_SUCCESS) r = C->p_cuEventRecord(e1, nullptr);
    if (r == CUDA_SUCCESS) r = C->p_cuEventSynchronize(e1);
    float f = 0;
    if (r == CUDA_SUCCESS) r = C->p_cuEventElapsedTime(&f, e0, e1);
    if (r == CUDA_SUCCESS && rep > 0) best = std::min(best, f);     // first run: warm-up
  }
  if (e0) C->p_cuEventDestroy(e0);
  if (e1) C->p_cuEventDestroy(e1);
  if (out) C->p_cuMemFree(out);
  C->p_cuModuleUnload(mod);
  if (r != CUDA_SUCCESS) return fail(NNB_ERR_CUDA, "ffma probe failed (%d)", (int)r);
  const double flops = 2.0 * 16.0 * iters * 256.0 * blocks;
  *tflops = flops / (best * 1e-3) / 1e12;
  if (ms) *ms = best;
  return NNB_OK;
}

void nnb_free(void *p) { free(p); }

nnb_status nnb_create(const nnb_net_desc *d, nnb_net **out) {
  if (!d || !out || !d->sources || d->n_sources < 1 || d->n_kernels < 0 || d->n_launches < 0 ||
      d->max_batch < 1)
    return fail(NNB_ERR_ARGUMENT, "invalid nnb_net_desc");
  for (int i = 0; i < d->n_launches; ++i) {
    const nnb_launch &l = d->launches[i];
    if (l.kernel < 0 || l.kernel >= d->n_kernels || l.block == 0 || l.block > 1024 ||
        l.items_per_block == 0 || l.grid_mult == 0)
      return fail(NNB_ERR_ARGUMENT, "launch %d is malformed", i);
  }
  Cu *C = cu();
  nnb_net *net = new nnb_net();
  net->device = d->device;
  net->max_batch = d->max_batch;
  if (const char *e = getenv("NNB_PDL")) net->pdl = atoi(e) != 0;
  if (const char *e = getenv("NNB_PREFETCH_MAX_N")) net->prefetch_max_n = atoi(e);
  CUdevice dev;
  nnb_status st = device_ctx(d->device, &net->ctx, &dev);
  if (st != NNB_OK) { delete net; return st; }
  CtxScope scope(net->ctx);
  if (scope.r != CUDA_SUCCESS) { delete net; return fail(NNB_ERR_CUDA, "cannot make device %d current", d->device); }

  auto bail = [&](nnb_status s) { nnb_destroy(net); return s; };
  for (int i = 0; i < d->n_sources; ++i) net->sources.emplace_back(d->sources[i]);
  net->include_dir = d->include_dir ? d->include_dir : ".";
  net->cache_dir = d->cache_dir ? d->cache_dir : "";
  net->digest = headers_digest(net->include_dir.c_str());
  for (int i = 0; i < d->n_kernels; ++i) {
    net->kernel_names.emplace_back(d->kernel_names[i]);
    const int src = d->kernel_source ? d->kernel_source[i] : 0;
    if (src < 0 || src >= d->n_sources) { fail(NNB_ERR_ARGUMENT, "kernel %d has no source", i); return bail(NNB_ERR_ARGUMENT); }
    net->kernel_source.push_back(src);
  }
  net->mods.assign(d->n_sources, nullptr);
  net->fns.assign(d->n_kernels, nullptr);
  net->launches.assign(d->launches, d->launches + d->n_launches);
  {
    // the sources a replay over max_batch images needs, compiled in parallel
    // (NNB_EAGER=1: every batch-size variant up front)
    const char *e = getenv("NNB_EAGER");
    const bool eager = e && atoi(e) != 0;
    nnb_status cst = ensure_loaded(net, eager ? 0 : net->max_batch, &net->compile_ms, &net->cache_hit);
    if (cst != NNB_OK) return bail(cst);
  }
  CUresult r;
  net->pool_bytes = d->pool_bytes;
  net->arena_bytes = d->arena_bytes;
  r = C->p_cuMemAlloc(&net->pool, std::max<uint64_t>(d->pool_bytes, 256));
  if (r != CUDA_SUCCESS) { fail(NNB_ERR_OOM, "pool alloc %llu bytes failed", (unsigned long long)d->pool_bytes); return bail(NNB_ERR_OOM); }
  if (d->pool_bytes) {
    r = C->p_cuMemcpyHtoD(net->pool, d->pool, d->pool_bytes);
    if (r != CUDA_SUCCESS) { fail(NNB_ERR_CUDA, "pool upload failed (%d)", (int)r); return bail(NNB_ERR_CUDA); }
  }
  r = C->p_cuMemAlloc(&net->arena, std::max<uint64_t>(d->arena_bytes, 256));
  if (r != CUDA_SUCCESS) { fail(NNB_ERR_OOM, "arena alloc %llu bytes failed", (unsigned long long)d->arena_bytes); return bail(NNB_ERR_OOM); }
  r = C->p_cuMemsetD8(net->arena, 0, std::max<uint64_t>(d->arena_bytes, 256));
  if (r != CUDA_SUCCESS) { fail(NNB_ERR_CUDA, "arena memset failed (%d)", (int)r); return bail(NNB_ERR_CUDA); }
  net->maps.resize(net->launches.size());
  for (size_t i = 0; i < net->launches.size(); ++i) {
    const nnb_launch &l = net->launches[i];
    if (l.zero_offset >= 0 && ((uint64_t)l.zero_offset + 4 > net->arena_bytes || l.zero_offset % 4)) {
      fail(NNB_ERR_ARGUMENT, "launch %zu: zero_offset outside the arena", i);
      return bail(NNB_ERR_ARGUMENT);
    }
    if (l.n_tmaps != 0 && l.n_tmaps != NNB_MAX_TMAPS) { fail(NNB_ERR_ARGUMENT, "launch %zu: n_tmaps must be 0 or %d", i, NNB_MAX_TMAPS); return bail(NNB_ERR_ARGUMENT); }
    net->maps[i].resize(l.n_tmaps);
    for (uint32_t k = 0; k < l.n_tmaps; ++k) {
      const nnb_tmap &t = l.tmaps[k];
      CUdeviceptr base = t.space == 1 ? net->arena : net->pool;
      uint64_t limit = t.space == 1 ? net->arena_bytes : net->pool_bytes;
      bool bad = (t.space != 1 && t.space != 2) || t.rank < 2 || t.rank > 4 || t.offset % 16;
      uint64_t last = t.offset + 4 * t.dims[0];
      for (uint32_t d = 1; d < t.rank && !bad; ++d) {
        bad = t.strides[d - 1] % 16 != 0 || t.box[d] == 0 || t.box[d] > 256;
        last += (t.dims[d] - 1) * t.strides[d - 1];
      }
      if (bad || last > limit || t.box[0] * 4 > 128) {
        fail(NNB_ERR_ARGUMENT, "launch %zu: tensor map %u malformed or out of range", i, k);
        return bail(NNB_ERR_ARGUMENT);
      }
      cuuint64_t dims[4], strides[3];
      cuuint32_t box[4], estr[4] = {1, 1, 1, 1};
      for (uint32_t d = 0; d < t.rank; ++d) { dims[d] = t.dims[d]; box[d] = t.box[d]; }
      for (uint32_t d = 0; d + 1 < t.rank; ++d) strides[d] = t.strides[d];
      r = C->p_cuTensorMapEncodeTiled(&net->maps[i][k], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, t.rank,
                                      reinterpret_cast<void *>(base + t.offset), dims, strides, box, estr,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE,
                                      t.swizzle == 3 ? CU_TENSOR_MAP_SWIZZLE_128B
                                      : t.swizzle == 2 ? CU_TENSOR_MAP_SWIZZLE_64B
                                      : t.swizzle == 1 ? CU_TENSOR_MAP_SWIZZLE_32B
                                                       : CU_TENSOR_MAP_SWIZZLE_NONE,
                                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) { fail(NNB_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d) for launch %zu map %u", (int)r, i, k); return bail(NNB_ERR_CUDA); }
    }
  }
  net->inputs.assign(d->inputs, d->inputs + d->n_inputs);
  net->outputs.assign(d->outputs, d->outputs + d->n_outputs);
  r = C->p_cuStreamCreate(&net->capture_stream, CU_STREAM_NON_BLOCKING);
  if (r != CUDA_SUCCESS) { fail(NNB_ERR_CUDA, "stream create failed"); return bail(NNB_ERR_CUDA); }
  C->p_cuEventCreate(&net->ev0, CU_EVENT_DEFAULT);
  C->p_cuEventCreate(&net->ev1, CU_EVENT_DEFAULT);
  *out = net;
  return NNB_OK;
}

nnb_status nnb_arena_ptr(nnb_net *net, uint64_t offset, void **dptr) {
  if (!net || !dptr || offset > net->arena_bytes) return fail(NNB_ERR_ARGUMENT, "bad arena offset");
  *dptr = reinterpret_cast<void *>(net->arena + offset);
  return NNB_OK;
}

nnb_status nnb_apply(nnb_net *net, int32_t n, void *stream) {
  if (!net) return fail(NNB_ERR_ARGUMENT, "net is NULL");
  if (n < 1 || n > net->max_batch)
    return fail(NNB_ERR_BATCH, "batch %d outside [1, %d]", n, net->max_batch);
  Cu *C = cu();
  CTX_SCOPE(net->ctx)
  CUgraphExec ex;
  nnb_status st = graph_for(net, n, &ex);
  if (st != NNB_OK) return st;
  CU_CHECK(C->p_cuGraphLaunch(ex, reinterpret_cast<CUstream>(stream)));
  return NNB_OK;
}

nnb_status nnb_sync(nnb_net *net, void *stream) {
  if (!net) return fail(NNB_ERR_ARGUMENT, "net is NULL");
  CTX_SCOPE(net->ctx)
  CU_CHECK(cu()->p_cuStreamSynchronize(reinterpret_cast<CUstream>(stream)));
  return NNB_OK;
}

// H2D of images [first, first + n) of every host input into the arena's
// first n rows, one replay, D2H of the outputs to the same image range of the
// host outputs; all on `stream`, nothing waited for.
static nnb_status enqueue_host(nnb_net *net, int32_t n, int64_t first, const void *const *inputs,
                               void *const *outputs, CUstream s) {
  if (!net) return fail(NNB_ERR_ARGUMENT, "net is NULL");
  if (n < 1 || n > net->max_batch)
    return fail(NNB_ERR_BATCH, "batch %d outside [1, %d]", n, net->max_batch);
  Cu *C = cu();
  CTX_SCOPE(net->ctx)
  for (size_t i = 0; i < net->inputs.size(); ++i) {
    const uint64_t b = net->inputs[i].image_bytes;
    CU_CHECK(C->p_cuMemcpyHtoDAsync(net->arena + net->inputs[i].offset,
                                    static_cast<const char *>(inputs[i]) + first * b, (size_t)n * b, s));
  }
  nnb_status st = nnb_apply(net, n, s);
  if (st != NNB_OK) return st;
  for (size_t i = 0; i < net->outputs.size(); ++i) {
    const uint64_t b = net->outputs[i].image_bytes;
    CU_CHECK(C->p_cuMemcpyDtoHAsync(static_cast<char *>(outputs[i]) + first * b,
                                    net->arena + net->outputs[i].offset, (size_t)n * b, s));
  }
  return NNB_OK;
}

nnb_status nnb_run_host(nnb_net *net, int32_t n, const void *const *inputs, void *const *outputs,
                        void *stream) {
  CUstream s = reinterpret_cast<CUstream>(stream);
  nnb_status st = enqueue_host(net, n, 0, inputs, outputs, s);
  if (st != NNB_OK) return st;
  CTX_SCOPE(net->ctx)
  CU_CHECK(cu()->p_cuStreamSynchronize(s));
  return NNB_OK;
}

nnb_status nnb_enqueue_host(nnb_net *net, int32_t n, const void *const *inputs,
                            void *const *outputs, void *stream) {
  return enqueue_host(net, n, 0, inputs, outputs, reinterpret_cast<CUstream>(stream));
}

nnb_status nnb_run_host_chunked(nnb_net *const *nets, const void *const *streams, int32_t k,
                                int64_t n, const void *const *inputs, void *const *outputs) {
  if (!nets || !streams || k < 1 || n < 1) return fail(NNB_ERR_ARGUMENT, "bad arguments");
  for (int32_t j = 0; j < k; ++j)
    if (!nets[j]) return fail(NNB_ERR_ARGUMENT, "net %d is NULL", j);
  const int64_t per = (n + k - 1) / k;
  // every chunk is enqueued before anything is waited for: chunk j's H2D
  // overlaps chunk j-1's replay and D2H (copy engines vs SMs)
  int32_t used = 0;
  for (int64_t first = 0; first < n; first += per, ++used) {
    const int32_t m = (int32_t)(n - first < per ? n - first : per);
    nnb_status st = enqueue_host(nets[used], m, first, inputs, outputs,
                                 reinterpret_cast<CUstream>(const_cast<void *>(streams[used])));
    if (st != NNB_OK) return st;
  }
  for (int32_t j = 0; j < used; ++j) {
    CTX_SCOPE(nets[j]->ctx)
    CU_CHECK(cu()->p_cuStreamSynchronize(reinterpret_cast<CUstream>(const_cast<void *>(streams[j]))));
  }
  return NNB_OK;
}

nnb_status nnb_time_apply(nnb_net *net, int32_t n, int32_t iters, void *stream, double *ms) {
  if (!net || iters < 1 || !ms) return fail(NNB_ERR_ARGUMENT, "bad arguments");
  if (n < 1 || n > net->max_batch)
    return fail(NNB_ERR_BATCH, "batch %d outside [1, %d]", n, net->max_batch);
  Cu *C = cu();
  CTX_SCOPE(net->ctx)
  CUstream s = reinterpret_cast<CUstream>(stream);
  CUgraphExec ex;
  nnb_status st = graph_for(net, n, &ex);
  if (st != NNB_OK) return st;
  CU_CHECK(C->p_cuEventRecord(net->ev0, s));
  for (int i = 0; i < iters; ++i) CU_CHECK(C->p_cuGraphLaunch(ex, s));
  CU_CHECK(C->p_cuEventRecord(net->ev1, s));
  CU_CHECK(C->p_cuEventSynchronize(net->ev1));
  float f = 0;
  CU_CHECK(C->p_cuEventElapsedTime(&f, net->ev0, net->ev1));
  *ms = f / iters;
  return NNB_OK;
}

nnb_status nnb_time_launch(nnb_net *net, int32_t index, int32_t n, int32_t iters, void *stream,
                           double *ms) {
  if (!net || iters < 1 || !ms || index < 0 || index >= (int32_t)net->launches.size())
    return fail(NNB_ERR_ARGUMENT, "bad arguments");
  if (n < 1 || n > net->max_batch)
    return fail(NNB_ERR_BATCH, "batch %d outside [1, %d]", n, net->max_batch);
  Cu *C = cu();
  CTX_SCOPE(net->ctx)
  CUstream s = reinterpret_cast<CUstream>(stream);
  nnb_status lst = ensure_loaded(net, n);
  if (lst != NNB_OK) return lst;
  CU_CHECK(C->p_cuEventRecord(net->ev0, s));
  for (int i = 0; i < iters; ++i) {
    nnb_status st = launch_one(net, (size_t)index, n, s, false);
    if (st != NNB_OK) return st;
  }
  CU_CHECK(C->p_cuEventRecord(net->ev1, s));
  CU_CHECK(C->p_cuEventSynchronize(net->ev1));
  float f = 0;
  CU_CHECK(C->p_cuEventElapsedTime(&f, net->ev0, net->ev1));
  *ms = f / iters;
  return NNB_OK;
}

nnb_status nnb_time_sequence(nnb_net *net, int32_t n, int32_t iters, void *stream, double *ms) {
  if (!net || iters < 1 || !ms) return fail(NNB_ERR_ARGUMENT, "bad arguments");
  if (n < 1 || n > net->max_batch)
    return fail(NNB_ERR_BATCH, "batch %d outside [1, %d]", n, net->max_batch);
  Cu *C = cu();
  CTX_SCOPE(net->ctx)
  CUstream s = reinterpret_cast<CUstream>(stream);
  const size_t L = net->launches.size();
  nnb_status st = ensure_loaded(net, n);
  if (st != NNB_OK) return st;
  std::vector<CUevent> ev(L + 1, nullptr);
  for (auto &e : ev)
    if (C->p_cuEventCreate(&e, CU_EVENT_DEFAULT) != CUDA_SUCCESS) st = fail(NNB_ERR_CUDA, "cuEventCreate failed");
  std::vector<double> acc(L, 0.0);
  for (int it = 0; it < iters && st == NNB_OK; ++it) {
    // same order and inputs as a replay; events between consecutive launches
    if (C->p_cuEventRecord(ev[0], s) != CUDA_SUCCESS) { st = fail(NNB_ERR_CUDA, "cuEventRecord failed"); break; }
    for (size_t li = 0; li < L && st == NNB_OK; ++li) {
      st = launch_one(net, li, n, s, false);
      if (st == NNB_OK && C->p_cuEventRecord(ev[li + 1], s) != CUDA_SUCCESS)
        st = fail(NNB_ERR_CUDA, "cuEventRecord failed");
    }
    if (st != NNB_OK) break;
    if (C->p_cuEventSynchronize(ev[L]) != CUDA_SUCCESS) { st = fail(NNB_ERR_CUDA, "kernel failed"); break; }
    for (size_t li = 0; li < L; ++li) {
      float f = 0;
      C->p_cuEventElapsedTime(&f, ev[li], ev[li + 1]);
      acc[li] += f;
    }
  }
  for (auto &e : ev)
    if (e) C->p_cuEventDestroy(e);
  if (st != NNB_OK) return st;
  for (size_t li = 0; li < L; ++li) {
    const nnb_launch &l = net->launches[li];
    ms[li] = (n < l.n_min || n > l.n_max) ? -1.0 : acc[li] / iters;
  }
  return NNB_OK;
}

nnb_status nnb_host_alloc(uint64_t bytes, void **ptr) {
  Cu *C = cu();
  if (!C->ok) return fail(NNB_ERR_NO_DRIVER, "%s", C->why.c_str());
  // page-locked memory needs a context: device 0's primary one when the
  // calling thread has none yet (it is portable across contexts anyway)
  CUcontext cur = nullptr;
  CU_CHECK(C->p_cuCtxGetCurrent(&cur));
  if (!cur) {
    CUdevice dev;
    CU_CHECK(C->p_cuDeviceGet(&dev, 0));
    CU_CHECK(C->p_cuDevicePrimaryCtxRetain(&cur, dev));
    CU_CHECK(C->p_cuCtxSetCurrent(cur));
  }
  CU_CHECK(C->p_cuMemAllocHost(ptr, bytes));
  return NNB_OK;
}

void nnb_host_free(void *ptr) {
  if (ptr && cu()->ok) cu()->p_cuMemFreeHost(ptr);
}

nnb_status nnb_net_info(nnb_net *net, uint64_t *arena_bytes, uint64_t *pool_bytes, int32_t *n_kernels,
                        double *compile_ms, int32_t *cache_hit) {
  if (!net) return fail(NNB_ERR_ARGUMENT, "net is NULL");
  if (arena_bytes) *arena_bytes = net->arena_bytes;
  if (pool_bytes) *pool_bytes = net->pool_bytes;
  if (n_kernels) *n_kernels = (int32_t)net->fns.size();
  if (compile_ms) *compile_ms = net->compile_ms;
  if (cache_hit) *cache_hit = net->cache_hit ? 1 : 0;
  return NNB_OK;
}

void nnb_destroy(nnb_net *net) {
  if (!net) return;
  Cu *C = cu();
  if (C->ok) {
    CtxScope scope(net->ctx);
    for (auto &kv : net->graphs) C->p_cuGraphExecDestroy(kv.second);
    if (net->ev0) C->p_cuEventDestroy(net->ev0);
    if (net->ev1) C->p_cuEventDestroy(net->ev1);
    if (net->capture_stream) C->p_cuStreamDestroy(net->capture_stream);
    if (net->side_stream) C->p_cuStreamDestroy(net->side_stream);
    if (net->fork_ev) C->p_cuEventDestroy(net->fork_ev);
    if (net->join_ev) C->p_cuEventDestroy(net->join_ev);
    if (net->pf_mod) C->p_cuModuleUnload(net->pf_mod);
    if (net->arena) C->p_cuMemFree(net->arena);
    if (net->pool) C->p_cuMemFree(net->pool);
    for (CUmodule m : net->mods)
      if (m) C->p_cuModuleUnload(m);
  }
  delete net;
}

}  // extern "C"
