// sgm_runtime.cpp — C-ABI runtime of libsgm.so (see include/sgm.h).
//
// * CUDA driver API resolved with dlopen("libcuda.so.1") at sgm_init, so the
//   library loads (and exports its symbols) on a machine without a GPU.
// * Kernels are generated per candidate (sgm_codegen.cpp), compiled with NVRTC
//   for sm_100a and cached on disk as cubins keyed by a hash of the source, so
//   re-runs and multi-rank sweeps are compile-free (checkpoint/resume of tuning).
// * Timing uses CUDA events around a CUDA graph of back-to-back launches with
//   rotating input sets (inputs miss L2 between launches).

#include <cuda.h>
#include <dlfcn.h>
#include <nvrtc.h>
#include <sys/stat.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <cinttypes>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <mutex>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/sgm.h"
#include "sgm_codegen.h"

namespace sgm {
// host mirror of sgm::Args in sgm_dev.cuh (kernel parameter block)
struct alignas(64) TmaDesc {
  uint64_t w[16];
};
struct Args {
  const void* in[16];
  void* out[16];
  void* scratch;
  TmaDesc tm[4];
};
static_assert(sizeof(TmaDesc) == sizeof(CUtensorMap), "TmaDesc mirrors CUtensorMap");
}  // namespace sgm

namespace {

const char* kDevHeader =
#include "sgm_dev_embed.inc"
    ;
const char* kUtilHeader =
#include "sgm_util_embed.inc"
    ;

thread_local std::string g_err;
std::atomic<long long> g_launches{0};

int set_err(int st, const char* fmt, ...) {
  char buf[2048];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}

// ---------------------------------------------------------------- driver API
struct Driver {
  bool ok = false;
  void* h = nullptr;
#define SGM_FN(name, ...) CUresult (*name)(__VA_ARGS__) = nullptr;
  SGM_FN(cuInit, unsigned)
  SGM_FN(cuDeviceGet, CUdevice*, int)
  SGM_FN(cuDeviceGetAttribute, int*, CUdevice_attribute, CUdevice)
  SGM_FN(cuDevicePrimaryCtxRetain, CUcontext*, CUdevice)
  SGM_FN(cuCtxSetCurrent, CUcontext)
  SGM_FN(cuCtxGetCurrent, CUcontext*)
  SGM_FN(cuModuleLoadData, CUmodule*, const void*)
  SGM_FN(cuModuleUnload, CUmodule)
  SGM_FN(cuModuleGetFunction, CUfunction*, CUmodule, const char*)
  SGM_FN(cuModuleGetGlobal, CUdeviceptr*, size_t*, CUmodule, const char*)
  SGM_FN(cuFuncSetAttribute, CUfunction, CUfunction_attribute, int)
  SGM_FN(cuFuncGetAttribute, int*, CUfunction_attribute, CUfunction)
  SGM_FN(cuLaunchKernel, CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, CUstream,
         void**, void**)
  SGM_FN(cuLaunchKernelEx, const CUlaunchConfig*, CUfunction, void**, void**)
  SGM_FN(cuMemAlloc, CUdeviceptr*, size_t)
  SGM_FN(cuMemFree, CUdeviceptr)
  SGM_FN(cuMemHostAlloc, void**, size_t, unsigned)
  SGM_FN(cuMemFreeHost, void*)
  SGM_FN(cuMemcpyHtoDAsync, CUdeviceptr, const void*, size_t, CUstream)
  SGM_FN(cuMemcpyDtoHAsync, void*, CUdeviceptr, size_t, CUstream)
  SGM_FN(cuMemcpyDtoH, void*, CUdeviceptr, size_t)
  SGM_FN(cuCtxSynchronize)
  SGM_FN(cuMemsetD32Async, CUdeviceptr, unsigned, size_t, CUstream)
  SGM_FN(cuStreamSynchronize, CUstream)
  SGM_FN(cuStreamCreate, CUstream*, unsigned)
  SGM_FN(cuStreamDestroy, CUstream)
  SGM_FN(cuEventCreate, CUevent*, unsigned)
  SGM_FN(cuEventDestroy, CUevent)
  SGM_FN(cuEventRecord, CUevent, CUstream)
  SGM_FN(cuEventSynchronize, CUevent)
  SGM_FN(cuEventElapsedTime, float*, CUevent, CUevent)
  SGM_FN(cuStreamBeginCapture, CUstream, CUstreamCaptureMode)
  SGM_FN(cuStreamEndCapture, CUstream, CUgraph*)
  SGM_FN(cuGraphInstantiateWithFlags, CUgraphExec*, CUgraph, unsigned long long)
  SGM_FN(cuGraphLaunch, CUgraphExec, CUstream)
  SGM_FN(cuGraphExecDestroy, CUgraphExec)
  SGM_FN(cuGraphDestroy, CUgraph)
  SGM_FN(cuOccupancyMaxActiveClusters, int*, CUfunction, const CUlaunchConfig*)
  SGM_FN(cuOccupancyMaxActiveBlocksPerMultiprocessor, int*, CUfunction, int, size_t)
  SGM_FN(cuTensorMapEncodeTiled, CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
         const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
         CUtensorMapL2promotion, CUtensorMapFloatOOBfill)
#undef SGM_FN
  CUresult (*cuGetErrorString)(CUresult, const char**) = nullptr;

  template <class F> bool sym(F& f, const char* a, const char* b = nullptr) {
    void* p = dlsym(h, a);
    if (!p && b) p = dlsym(h, b);
    f = reinterpret_cast<F>(p);
    return p != nullptr;
  }
  bool load() {
    if (ok) return true;
    h = dlopen("libcuda.so.1", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libcuda.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return false;
    bool g = true;
    g &= sym(cuInit, "cuInit");
    g &= sym(cuDeviceGet, "cuDeviceGet");
    g &= sym(cuDeviceGetAttribute, "cuDeviceGetAttribute");
    g &= sym(cuDevicePrimaryCtxRetain, "cuDevicePrimaryCtxRetain");
    g &= sym(cuCtxSetCurrent, "cuCtxSetCurrent");
    g &= sym(cuCtxGetCurrent, "cuCtxGetCurrent");
    g &= sym(cuModuleLoadData, "cuModuleLoadData");
    g &= sym(cuModuleUnload, "cuModuleUnload");
    g &= sym(cuModuleGetFunction, "cuModuleGetFunction");
    g &= sym(cuModuleGetGlobal, "cuModuleGetGlobal_v2");
    g &= sym(cuFuncSetAttribute, "cuFuncSetAttribute");
    g &= sym(cuFuncGetAttribute, "cuFuncGetAttribute");
    g &= sym(cuLaunchKernel, "cuLaunchKernel");
    sym(cuLaunchKernelEx, "cuLaunchKernelEx");  // optional: programmatic dependent launch
    g &= sym(cuMemAlloc, "cuMemAlloc_v2");
    g &= sym(cuMemFree, "cuMemFree_v2");
    g &= sym(cuMemHostAlloc, "cuMemHostAlloc");
    g &= sym(cuMemFreeHost, "cuMemFreeHost");
    g &= sym(cuMemcpyHtoDAsync, "cuMemcpyHtoDAsync_v2");
    g &= sym(cuMemcpyDtoHAsync, "cuMemcpyDtoHAsync_v2");
    g &= sym(cuMemcpyDtoH, "cuMemcpyDtoH_v2");
    g &= sym(cuCtxSynchronize, "cuCtxSynchronize");
    g &= sym(cuMemsetD32Async, "cuMemsetD32Async");
    g &= sym(cuStreamSynchronize, "cuStreamSynchronize");
    g &= sym(cuStreamCreate, "cuStreamCreate");
    g &= sym(cuStreamDestroy, "cuStreamDestroy_v2");
    g &= sym(cuEventCreate, "cuEventCreate");
    g &= sym(cuEventDestroy, "cuEventDestroy_v2");
    g &= sym(cuEventRecord, "cuEventRecord");
    g &= sym(cuEventSynchronize, "cuEventSynchronize");
    g &= sym(cuEventElapsedTime, "cuEventElapsedTime");
    g &= sym(cuStreamBeginCapture, "cuStreamBeginCapture_v2");
    g &= sym(cuStreamEndCapture, "cuStreamEndCapture");
    g &= sym(cuGraphInstantiateWithFlags, "cuGraphInstantiateWithFlags");
    g &= sym(cuGraphLaunch, "cuGraphLaunch");
    g &= sym(cuGraphExecDestroy, "cuGraphExecDestroy");
    g &= sym(cuGraphDestroy, "cuGraphDestroy");
    g &= sym(cuTensorMapEncodeTiled, "cuTensorMapEncodeTiled");
    sym(cuOccupancyMaxActiveClusters, "cuOccupancyMaxActiveClusters");
    sym(cuOccupancyMaxActiveBlocksPerMultiprocessor, "cuOccupancyMaxActiveBlocksPerMultiprocessor");
    sym(cuGetErrorString, "cuGetErrorString");
    ok = g;
    return ok;
  }
};
Driver D;
std::mutex g_init_mu;

struct DevState {
  bool init = false;
  CUdevice dev = 0;
  CUcontext ctx = nullptr;
  int sms = 148;
  int cc_major = 10, cc_minor = 0;
  CUmodule util = nullptr;
  CUfunction f_fill64, f_fill32, f_fill16, f_ff_fill, f_cmp, f_re64, f_re32, f_re16, f_rex32, f_rex16, f_n64, f_n32, f_n16;
  CUdeviceptr red = 0;  // 4 x u64 reduction scratch
  // host-buffer (e2e) staging shared by every plan of this device: pinned host
  // memory + one device buffer, grown on demand (sgm_plan_run_host)
  std::mutex io_mu;
  void* pinned = nullptr;
  CUdeviceptr dev_io = 0;
  size_t io_bytes = 0;
};
DevState g_dev[16];
thread_local int t_device = -1;
std::string g_cache_dir;
std::mutex g_cache_mu;

int cu_check(CUresult r, const char* what) {
  if (r == CUDA_SUCCESS) return SGM_OK;
  const char* s = "?";
  if (D.cuGetErrorString) D.cuGetErrorString(r, &s);
  return set_err(SGM_ERR_CUDA, "%s failed: %s (%d)", what, s, (int)r);
}
#define CU(call)                                            \
  do {                                                      \
    int _st = cu_check((call), #call);                      \
    if (_st != SGM_OK) return _st;                          \
  } while (0)

std::string default_cache_dir() {
  if (const char* e = getenv("SGM_CACHE_DIR")) return e;
  Dl_info info;
  if (dladdr((void*)&default_cache_dir, &info) && info.dli_fname) {
    std::string p = info.dli_fname;
    size_t at = p.find_last_of('/');
    if (at != std::string::npos) return p.substr(0, at) + "/.cubin_cache";
  }
  return "/tmp/sgm_cubin_cache";
}

std::string cache_dir() {
  std::lock_guard<std::mutex> lk(g_cache_mu);
  if (g_cache_dir.empty()) g_cache_dir = default_cache_dir();
  return g_cache_dir;
}

bool read_file(const std::string& path, std::string& out) {
  std::ifstream f(path, std::ios::binary);
  if (!f) return false;
  std::ostringstream ss;
  ss << f.rdbuf();
  out = ss.str();
  return !out.empty();
}

void write_file_atomic(const std::string& path, const std::string& data) {
  std::string dir = path.substr(0, path.find_last_of('/'));
  mkdir(dir.c_str(), 0755);
  char tmp[64];
  snprintf(tmp, sizeof tmp, ".tmp.%d.%p", (int)getpid(), (void*)&data);
  std::string t = path + tmp;
  {
    std::ofstream f(t, std::ios::binary);
    if (!f) return;
    f.write(data.data(), (std::streamsize)data.size());
  }
  rename(t.c_str(), path.c_str());
}

const char* kArch = "-arch=sm_100a";

// Compile `src` (which #includes sgm_dev.cuh / sgm_util.cuh) to a cubin, with the disk cache.
int compile_cubin(const std::string& src, std::string& cubin, double& ms, int& hit) {
  int maj = 0, minr = 0;
  nvrtcVersion(&maj, &minr);
  std::string key_src = src + "|" + kArch + "|nvrtc" + std::to_string(maj) + "." + std::to_string(minr) + "|" +
                        std::to_string(sgmcg::fnv1a(kDevHeader)) + std::to_string(sgmcg::fnv1a(kUtilHeader));
  if (const char* e = getenv("SGM_NVRTC_OPTS")) key_src += std::string("|opts:") + e;  // experiments: own cache keys
  char name[64];
  snprintf(name, sizeof name, "%016" PRIx64 ".cubin", sgmcg::fnv1a(key_src));
  std::string path = cache_dir() + "/" + name;
  if (read_file(path, cubin)) {
    ms = 0;
    hit = 1;
    return SGM_OK;
  }
  hit = 0;
  auto t0 = std::chrono::steady_clock::now();
  nvrtcProgram prog;
  const char* hdrs[2] = {kDevHeader, kUtilHeader};
  const char* hnames[2] = {"sgm_dev.cuh", "sgm_util.cuh"};
  if (nvrtcCreateProgram(&prog, src.c_str(), "sgm_kernel.cu", 2, hdrs, hnames) != NVRTC_SUCCESS)
    return set_err(SGM_ERR_NVRTC, "nvrtcCreateProgram failed");
  std::vector<const char*> opts = {kArch, "-std=c++17", "-lineinfo", "-DNDEBUG", "--extra-device-vectorization",
                                   "-diag-suppress=177,550"};
  static std::vector<std::string> extra = [] {  // experiments: SGM_NVRTC_OPTS="-a -b"
    std::vector<std::string> v;
    if (const char* e = getenv("SGM_NVRTC_OPTS")) {
      std::istringstream ss(e);
      std::string w;
      while (ss >> w) v.push_back(w);
    }
    return v;
  }();
  for (auto& e : extra) opts.push_back(e.c_str());
  nvrtcResult r = nvrtcCompileProgram(prog, (int)opts.size(), opts.data());
  if (r != NVRTC_SUCCESS) {
    size_t ls = 0;
    nvrtcGetProgramLogSize(prog, &ls);
    std::string log(ls, '\0');
    nvrtcGetProgramLog(prog, &log[0]);
    nvrtcDestroyProgram(&prog);
    if (const char* dump = getenv("SGM_DUMP_FAILED")) {  // debugging aid: keep the failing source
      std::ofstream f(dump);
      f << src;
    }
    if (log.size() > 1800) log = log.substr(0, 1800);
    return set_err(SGM_ERR_NVRTC, "NVRTC: %s\n%s", nvrtcGetErrorString(r), log.c_str());
  }
  size_t cs = 0;
  nvrtcGetCUBINSize(prog, &cs);
  cubin.assign(cs, '\0');
  nvrtcGetCUBIN(prog, &cubin[0]);
  nvrtcDestroyProgram(&prog);
  ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  write_file_atomic(path, cubin);
  return SGM_OK;
}

int ensure_ctx() {
  if (t_device < 0 || !g_dev[t_device].init) return set_err(SGM_ERR_NOT_INIT, "sgm_init(device) not called on this thread");
  CU(D.cuCtxSetCurrent(g_dev[t_device].ctx));
  return SGM_OK;
}

int launch_1d(CUfunction f, int64_t n, CUstream s, void** params) {
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  CU(D.cuLaunchKernel(f, (unsigned)blocks, 1, 1, 256, 1, 1, 0, s, params, nullptr));
  g_launches++;
  return SGM_OK;
}

size_t esize(int ns) { return ns == SGM_F64 ? 8 : ns == SGM_BF16 ? 2 : 4; }

}  // namespace

struct sgm_plan {
  sgmcg::GenResult gen;
  int device = 0;
  CUmodule mod = nullptr;
  CUfunction fn = nullptr;
  CUdeviceptr scratch = 0;
  int numsys = 0;
  int64_t launch_ctas = 0;   // persistent grid: min(work CTAs, co-resident CTAs)
  int occ_per_sm = 0;        // occupancy API: CTAs per SM (cluster 1)
  int regs = 0, static_smem = 0;
  int n_in = 0, n_out = 0;
  size_t in_bytes[SGM_MAX_SLOTS] = {0};
  size_t out_bytes[SGM_MAX_SLOTS] = {0};
  int64_t out_elems[SGM_MAX_SLOTS] = {0};
  double compile_ms = 0;
  int cache_hit = 0;
  // TMA descriptors of the streamed operands, re-encoded when an input pointer changes
  CUtensorMap tmaps[4];
  const void* tmap_ptr[4] = {nullptr, nullptr, nullptr, nullptr};
  CUstream tstream = nullptr;
  // cached CUDA graph of `graph_rot` launches over one rotation of input sets
  CUgraph graph = nullptr;
  CUgraphExec gexec = nullptr;
  std::vector<const void*> graph_key;
  int graph_rot = 0;
  int graph_pdl = -1;        // PDL setting the cached graph was captured with
  CUdeviceptr wd_flag = 0;   // the module's sgm_wd_flag (watchdog, sgm_dev.cuh)
  std::string cubin;         // compile-only plans keep their sm_100a cubin (sgm_plan_cubin)
};

// programmatic dependent launch: on unless SGM_NO_PDL is set; sgm_set_pdl overrides
static std::atomic<int> g_pdl{-1};
static bool pdl_on() {
  int v = g_pdl.load();
  if (v < 0) {
    v = getenv("SGM_NO_PDL") == nullptr ? 1 : 0;
    g_pdl.store(v);
  }
  return v != 0;
}

struct sgm_timer {
  int cap = 0;
  int device = 0;
  std::vector<CUevent> ev;      // 2 per slot
  std::vector<int> launches;    // kernel launches timed in each slot
  int last = -1;
};

extern "C" {

int sgm_abi_version(void) { return SGM_ABI_VERSION; }
long long sgm_launch_count(void) { return g_launches.load(); }
const char* sgm_last_error(void) { return g_err.c_str(); }

int sgm_set_cache_dir(const char* path) {
  std::lock_guard<std::mutex> lk(g_cache_mu);
  g_cache_dir = path ? path : "";
  return SGM_OK;
}

int sgm_init(int device) {
  std::lock_guard<std::mutex> lk(g_init_mu);
  if (device < 0 || device >= 16) return set_err(SGM_ERR_INVALID, "bad device %d", device);
  if (!D.load()) return set_err(SGM_ERR_CUDA, "cannot load libcuda.so.1 (no NVIDIA driver on this machine)");
  DevState& S = g_dev[device];
  if (!S.init) {
    CU(D.cuInit(0));
    CU(D.cuDeviceGet(&S.dev, device));
    CU(D.cuDevicePrimaryCtxRetain(&S.ctx, S.dev));
    CU(D.cuCtxSetCurrent(S.ctx));
    D.cuDeviceGetAttribute(&S.sms, CU_DEVICE_ATTRIBUTE_MULTIPROCESSOR_COUNT, S.dev);
    D.cuDeviceGetAttribute(&S.cc_major, CU_DEVICE_ATTRIBUTE_COMPUTE_CAPABILITY_MAJOR, S.dev);
    D.cuDeviceGetAttribute(&S.cc_minor, CU_DEVICE_ATTRIBUTE_COMPUTE_CAPABILITY_MINOR, S.dev);
    if (S.cc_major != 10 || S.cc_minor != 0)
      return set_err(SGM_ERR_CUDA, "device %d is sm_%d%d; libsgm targets sm_100a (B200) only", device, S.cc_major,
                     S.cc_minor);
    std::string cubin;
    double ms;
    int hit;
    int st = compile_cubin("#include \"sgm_util.cuh\"\n", cubin, ms, hit);
    if (st) return st;
    CU(D.cuModuleLoadData(&S.util, cubin.data()));
    CU(D.cuModuleGetFunction(&S.f_fill64, S.util, "sgm_fill64"));
    CU(D.cuModuleGetFunction(&S.f_fill32, S.util, "sgm_fill32"));
    CU(D.cuModuleGetFunction(&S.f_fill16, S.util, "sgm_fill16"));
    CU(D.cuModuleGetFunction(&S.f_ff_fill, S.util, "sgm_ff_fill"));
    CU(D.cuModuleGetFunction(&S.f_cmp, S.util, "sgm_cmp_u32"));
    CU(D.cuModuleGetFunction(&S.f_re64, S.util, "sgm_relerr_f64"));
    CU(D.cuModuleGetFunction(&S.f_re32, S.util, "sgm_relerr_f32"));
    CU(D.cuModuleGetFunction(&S.f_re16, S.util, "sgm_relerr_bf16"));
    CU(D.cuModuleGetFunction(&S.f_rex32, S.util, "sgm_relerr_x_f32"));
    CU(D.cuModuleGetFunction(&S.f_rex16, S.util, "sgm_relerr_x_bf16"));
    CU(D.cuModuleGetFunction(&S.f_n64, S.util, "sgm_normal_f64"));
    CU(D.cuModuleGetFunction(&S.f_n32, S.util, "sgm_normal_f32"));
    CU(D.cuModuleGetFunction(&S.f_n16, S.util, "sgm_normal_bf16"));
    CU(D.cuMemAlloc(&S.red, 64));
    S.init = true;
  }
  t_device = device;
  CU(D.cuCtxSetCurrent(S.ctx));
  return SGM_OK;
}

int sgm_plan_create(const sgm_plan_desc* desc, sgm_plan** out) {
  if (!desc || !out) return set_err(SGM_ERR_INVALID, "null argument");
  *out = nullptr;
  int sms = (t_device >= 0 && g_dev[t_device].init) ? g_dev[t_device].sms : 148;
  sgmcg::GenResult gr = sgmcg::generate(*desc, sms);
  if (gr.status != SGM_OK) return set_err(gr.status, "%s", gr.error.c_str());
  sgm_plan* p = new sgm_plan();
  p->gen = gr;
  p->numsys = desc->numsys;
  p->n_in = desc->n_inputs;
  p->n_out = desc->n_outputs;
  for (int k = 0; k < desc->n_inputs; ++k) {
    int64_t n = 1;
    for (int j = 0; j < desc->inputs[k].rank; ++j) n *= desc->inputs[k].dims[j];
    p->in_bytes[k] = (size_t)n * esize(desc->numsys);
  }
  for (int k = 0; k < desc->n_outputs; ++k) {
    int64_t n = 1;
    for (int j = 0; j < desc->outputs[k].rank; ++j) n *= desc->outputs[k].dims[j];
    p->out_elems[k] = n;
    p->out_bytes[k] = (size_t)n * esize(desc->numsys);
  }
  std::string cubin;
  int st = compile_cubin(gr.source, cubin, p->compile_ms, p->cache_hit);
  if (st) {
    delete p;
    return st;
  }
  if (t_device < 0) {  // compile-only use (no device bound): keep the source + cubin, no module
    p->cubin = std::move(cubin);
    *out = p;
    return SGM_OK;
  }
  p->device = t_device;
  if ((st = ensure_ctx())) { delete p; return st; }
  CUresult r = D.cuModuleLoadData(&p->mod, cubin.data());
  if (r != CUDA_SUCCESS) { delete p; return cu_check(r, "cuModuleLoadData"); }
  r = D.cuModuleGetFunction(&p->fn, p->mod, gr.kernel_name.c_str());
  if (r != CUDA_SUCCESS) { sgm_plan_destroy(p); return cu_check(r, "cuModuleGetFunction"); }
  {
    size_t wsz = 0;
    if (D.cuModuleGetGlobal(&p->wd_flag, &wsz, p->mod, "sgm_wd_flag") != CUDA_SUCCESS) p->wd_flag = 0;
  }
  // prefer the largest shared-memory carveout: the planner counts on two CTAs per SM
  // at ~110 KB each, which the default carveout does not always grant
  D.cuFuncSetAttribute(p->fn, CU_FUNC_ATTRIBUTE_PREFERRED_SHARED_MEMORY_CARVEOUT, 100);
  if (gr.smem_bytes > 0) {  // dynamic + static smem may cross the 48 KB default even below it
    r = D.cuFuncSetAttribute(p->fn, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, gr.smem_bytes);
    if (r != CUDA_SUCCESS) { sgm_plan_destroy(p); return cu_check(r, "cuFuncSetAttribute(smem)"); }
  }
  if (gr.cluster > 8) {
    r = D.cuFuncSetAttribute(p->fn, CU_FUNC_ATTRIBUTE_NON_PORTABLE_CLUSTER_SIZE_ALLOWED, 1);
    if (r != CUDA_SUCCESS) { sgm_plan_destroy(p); return cu_check(r, "cuFuncSetAttribute(cluster)"); }
  }
  {
    // persistent launch: at most the CTAs (whole clusters) that can be co-resident
    int64_t resident = 0;
    if (gr.cluster > 1 && D.cuOccupancyMaxActiveClusters) {
      CUlaunchAttribute attr;
      memset(&attr, 0, sizeof attr);
      attr.id = CU_LAUNCH_ATTRIBUTE_CLUSTER_DIMENSION;
      attr.value.clusterDim.x = (unsigned)gr.cluster;
      attr.value.clusterDim.y = 1;
      attr.value.clusterDim.z = 1;
      CUlaunchConfig cfg;
      memset(&cfg, 0, sizeof cfg);
      cfg.gridDimX = (unsigned)gr.ctas;
      cfg.gridDimY = cfg.gridDimZ = 1;
      cfg.blockDimX = (unsigned)gr.threads;
      cfg.blockDimY = cfg.blockDimZ = 1;
      cfg.sharedMemBytes = (unsigned)gr.smem_bytes;
      cfg.attrs = &attr;
      cfg.numAttrs = 1;
      int ncl = 0;
      if (D.cuOccupancyMaxActiveClusters(&ncl, p->fn, &cfg) == CUDA_SUCCESS && ncl > 0) resident = (int64_t)ncl * gr.cluster;
    } else if (gr.cluster == 1 && D.cuOccupancyMaxActiveBlocksPerMultiprocessor) {
      int nb = 0;
      if (D.cuOccupancyMaxActiveBlocksPerMultiprocessor(&nb, p->fn, gr.threads, (size_t)gr.smem_bytes) == CUDA_SUCCESS &&
          nb > 0)
        resident = (int64_t)nb * g_dev[t_device].sms;
      // the occupancy API counts a TMEM-allocating kernel as one CTA per SM, but the
      // hardware co-schedules two that each take at most half of TMEM (the planner
      // pairs only those): trust the plan there
      if (gr.ctas_per_sm > nb && gr.n_tcgen05 > 0 && gr.smem_bytes <= 113 * 1024) {
        nb = gr.ctas_per_sm;
        resident = (int64_t)nb * g_dev[t_device].sms;
      }
      p->occ_per_sm = nb;
      if (getenv("SGM_OCC_DEBUG"))
        for (int kb : {16, 32, 48, 64, 80, 90, 96, 100, 104, 108, 112}) {
          int n2 = 0;
          D.cuOccupancyMaxActiveBlocksPerMultiprocessor(&n2, p->fn, gr.threads, (size_t)kb * 1024);
          int n3 = 0;
          D.cuOccupancyMaxActiveBlocksPerMultiprocessor(&n3, p->fn, 128, (size_t)kb * 1024);
          fprintf(stderr, "occ: %d KB dyn -> %d CTAs/SM at %d threads, %d at 128 threads\n", kb, n2, gr.threads, n3);
        }
      D.cuFuncGetAttribute(&p->regs, CU_FUNC_ATTRIBUTE_NUM_REGS, p->fn);
      D.cuFuncGetAttribute(&p->static_smem, CU_FUNC_ATTRIBUTE_SHARED_SIZE_BYTES, p->fn);
    }
    p->launch_ctas = gr.ctas;
    if (resident > 0 && resident < gr.ctas) p->launch_ctas = resident / gr.cluster * gr.cluster;
    if (p->launch_ctas < gr.cluster) p->launch_ctas = gr.cluster;
  }
  if (gr.scratch_bytes > 0) {
    r = D.cuMemAlloc(&p->scratch, (size_t)gr.scratch_bytes);
    if (r != CUDA_SUCCESS) { sgm_plan_destroy(p); return cu_check(r, "cuMemAlloc(scratch)"); }
    // gsplit counters (and trace) start at zero; the kernels leave the counters at zero
    r = D.cuMemsetD32Async(p->scratch, 0, (size_t)(gr.scratch_bytes + 3) / 4, nullptr);
    if (r == CUDA_SUCCESS) r = D.cuCtxSynchronize();
    if (r != CUDA_SUCCESS) { sgm_plan_destroy(p); return cu_check(r, "zero scratch"); }
  }
  *out = p;
  return SGM_OK;
}

int sgm_plan_feasible(const sgm_plan_desc* desc, sgm_plan_info* info) {
  if (!desc) return set_err(SGM_ERR_INVALID, "null argument");
  int sms = (t_device >= 0 && g_dev[t_device].init) ? g_dev[t_device].sms : 148;
  sgmcg::GenResult gr = sgmcg::generate(*desc, sms);
  if (gr.status != SGM_OK) return set_err(gr.status, "%s", gr.error.c_str());
  if (info) {
    memset(info, 0, sizeof *info);
    info->logical_blocks = gr.logical_blocks;
    info->ctas = gr.ctas;
    info->cluster = gr.cluster;
    info->threads = gr.threads;
    info->smem_bytes = gr.smem_bytes;
    info->loop_parts = gr.loop_parts;
    info->free_parts = gr.free_parts;
    info->scratch_bytes = gr.scratch_bytes;
    info->n_tcgen05 = gr.n_tcgen05;
    info->source_hash = sgmcg::fnv1a(gr.source);
    snprintf(info->kernel_name, sizeof info->kernel_name, "%s", gr.kernel_name.c_str());
    snprintf(info->plan_summary, sizeof info->plan_summary, "%s", gr.summary.c_str());
  }
  return SGM_OK;
}

int sgm_plan_info_get(const sgm_plan* p, sgm_plan_info* info) {
  if (!p || !info) return set_err(SGM_ERR_INVALID, "null argument");
  memset(info, 0, sizeof *info);
  info->logical_blocks = p->gen.logical_blocks;
  info->ctas = p->gen.ctas;
  info->cluster = p->gen.cluster;
  info->threads = p->gen.threads;
  info->smem_bytes = p->gen.smem_bytes;
  info->loop_parts = p->gen.loop_parts;
  info->free_parts = p->gen.free_parts;
  info->scratch_bytes = p->gen.scratch_bytes;
  info->compile_ms = p->compile_ms;
  info->cache_hit = p->cache_hit;
  info->n_tcgen05 = p->gen.n_tcgen05;
  info->source_hash = sgmcg::fnv1a(p->gen.source);
  snprintf(info->kernel_name, sizeof info->kernel_name, "%s", p->gen.kernel_name.c_str());
  snprintf(info->plan_summary, sizeof info->plan_summary, "grid=%lld occ=%d regs=%d sstat=%d %s",
           (long long)p->launch_ctas, p->occ_per_sm, p->regs, p->static_smem, p->gen.summary.c_str());
  return SGM_OK;
}

int sgm_plan_cubin(const sgm_plan* p, void* buf, size_t cap, size_t* len) {
  if (!p) return set_err(SGM_ERR_INVALID, "null plan");
  if (p->cubin.empty()) return set_err(SGM_ERR_INVALID, "cubin is kept only for compile-only plans (no device bound)");
  if (len) *len = p->cubin.size();
  if (buf && cap) memcpy(buf, p->cubin.data(), std::min(cap, p->cubin.size()));
  return SGM_OK;
}

int sgm_plan_source(const sgm_plan* p, char* buf, size_t cap, size_t* len) {
  if (!p) return set_err(SGM_ERR_INVALID, "null plan");
  if (len) *len = p->gen.source.size();
  if (buf && cap) {
    size_t n = std::min(cap - 1, p->gen.source.size());
    memcpy(buf, p->gen.source.data(), n);
    buf[n] = 0;
  }
  return SGM_OK;
}

int sgm_plan_trace(const sgm_plan* p, uint64_t* host, int64_t cap, int64_t* n) {
  if (!p || !n) return set_err(SGM_ERR_INVALID, "null argument");
  if (p->gen.trace_off < 0 || !p->scratch) return set_err(SGM_ERR_INVALID, "plan was not created with hints.trace");
  int st = ensure_ctx();
  if (st) return st;
  *n = p->launch_ctas * SGM_TRACE_N;
  if (!host || cap <= 0) return SGM_OK;
  CU(D.cuCtxSynchronize());
  for (int64_t c = 0; c < p->launch_ctas && (c + 1) * SGM_TRACE_N <= cap; ++c)
    CU(D.cuMemcpyDtoH(host + c * SGM_TRACE_N * 2, p->scratch + (CUdeviceptr)(c * p->gen.scratch_per_cta + p->gen.trace_off),
                      SGM_TRACE_N * 16));
  return SGM_OK;
}

int sgm_plan_destroy(sgm_plan* p) {
  if (!p) return SGM_OK;
  if (p->mod || p->scratch || p->tstream || p->gexec || p->graph) {
    if (D.ok && p->device >= 0 && g_dev[p->device].init) D.cuCtxSetCurrent(g_dev[p->device].ctx);
    if (p->mod) D.cuModuleUnload(p->mod);
    if (p->scratch) D.cuMemFree(p->scratch);
    if (p->tstream) D.cuStreamDestroy(p->tstream);
    if (p->gexec) D.cuGraphExecDestroy(p->gexec);
    if (p->graph) D.cuGraphDestroy(p->graph);
  }
  delete p;
  return SGM_OK;
}

static int fill_nan(int ns, CUdeviceptr p, int64_t n, CUstream s) {
  DevState& S = g_dev[t_device];
  if (ns == SGM_F64) {
    uint64_t v = 0x7ff8000000000000ull;
    void* a[] = {&p, &n, &v};
    return launch_1d(S.f_fill64, n, s, a);
  } else if (ns == SGM_BF16) {
    uint16_t v = 0x7fc0;
    void* a[] = {&p, &n, &v};
    return launch_1d(S.f_fill16, n, s, a);
  }
  uint32_t v = ns == SGM_FF ? 0xFFFFFFFFu : 0x7fc00000u;
  void* a[] = {&p, &n, &v};
  return launch_1d(S.f_fill32, n, s, a);
}

static int encode_tmap(sgm_plan* p, int i, const void* ptr) {
  const sgmcg::TmaSpec& t = p->gen.tmaps[i];
  if (((uintptr_t)ptr & 15) != 0) return set_err(SGM_ERR_INVALID, "TMA operand (input slot %d) is not 16-byte aligned", t.slot);
  cuuint64_t gdim[4] = {(cuuint64_t)t.dims[3], (cuuint64_t)t.dims[2], (cuuint64_t)t.dims[1], (cuuint64_t)t.dims[0]};
  cuuint64_t es = (cuuint64_t)t.elem_bytes;
  cuuint64_t gstride[3] = {gdim[0] * es, gdim[0] * gdim[1] * es, gdim[0] * gdim[1] * gdim[2] * es};
  cuuint32_t box[4] = {(cuuint32_t)t.box0, (cuuint32_t)t.box1, (cuuint32_t)t.box2, (cuuint32_t)t.box3};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = D.cuTensorMapEncodeTiled(&p->tmaps[i],
                                        t.elem_bytes == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                        : t.u32          ? CU_TENSOR_MAP_DATA_TYPE_UINT32
                                                         : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                                        4, const_cast<void*>(ptr), gdim, gstride, box, estr,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE,
                                        t.swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return cu_check(r, "cuTensorMapEncodeTiled");
  p->tmap_ptr[i] = ptr;
  return SGM_OK;
}

static int launch_plan(sgm_plan* p, const void* const* inputs, void* const* outputs, CUstream s) {
  // generated kernels move rows with 16-byte vectors wherever the strides allow
  // (and column strips, TMA boxes): every tensor base must be 16-byte aligned
  for (int k = 0; k < p->n_in; ++k)
    if ((uintptr_t)inputs[k] & 15) return set_err(SGM_ERR_INVALID, "input %d is not 16-byte aligned", k);
  for (int k = 0; k < p->n_out; ++k)
    if ((uintptr_t)outputs[k] & 15) return set_err(SGM_ERR_INVALID, "output %d is not 16-byte aligned", k);
  sgm::Args args;
  memset(&args, 0, sizeof args);
  for (int i = 0; i < (int)p->gen.tmaps.size() && i < 4; ++i) {
    const void* ptr = inputs[p->gen.tmaps[i].slot];
    if (ptr != p->tmap_ptr[i]) {
      int st = encode_tmap(p, i, ptr);
      if (st) return st;
    }
    memcpy(&args.tm[i], &p->tmaps[i], sizeof(CUtensorMap));
  }
  for (int k = 0; k < p->n_in; ++k) args.in[k] = inputs[k];
  for (int k = 0; k < p->n_out; ++k) args.out[k] = outputs[k];
  args.scratch = (void*)p->scratch;
  void* params[] = {&args};
  if (pdl_on() && D.cuLaunchKernelEx) {
    // programmatic stream serialization: this grid may launch while the previous
    // kernel in the stream drains; the generated code's griddepcontrol.wait keeps
    // every global access after that kernel's completion
    CUlaunchAttribute attr;
    memset(&attr, 0, sizeof attr);
    attr.id = CU_LAUNCH_ATTRIBUTE_PROGRAMMATIC_STREAM_SERIALIZATION;
    attr.value.programmaticStreamSerializationAllowed = 1;
    CUlaunchConfig cfg;
    memset(&cfg, 0, sizeof cfg);
    cfg.gridDimX = (unsigned)p->launch_ctas;
    cfg.gridDimY = cfg.gridDimZ = 1;
    cfg.blockDimX = (unsigned)p->gen.threads;
    cfg.blockDimY = cfg.blockDimZ = 1;
    cfg.sharedMemBytes = (unsigned)p->gen.smem_bytes;
    cfg.hStream = s;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    CU(D.cuLaunchKernelEx(&cfg, p->fn, params, nullptr));
  } else {
    CU(D.cuLaunchKernel(p->fn, (unsigned)p->launch_ctas, 1, 1, (unsigned)p->gen.threads, 1, 1,
                        (unsigned)p->gen.smem_bytes, s, params, nullptr));
  }
  g_launches++;  // during graph capture this counts the captured node once
  return SGM_OK;
}

int sgm_plan_run(sgm_plan* p, const void* const* inputs, void* const* outputs, int init_outputs, void* stream) {
  if (!p) return set_err(SGM_ERR_INVALID, "null plan");
  if (!p->fn) return set_err(SGM_ERR_NOT_INIT, "plan was created without a device (call sgm_init first)");
  int st = ensure_ctx();
  if (st) return st;
  CUstream s = (CUstream)stream;
  if (init_outputs)
    for (int k = 0; k < p->n_out; ++k)
      if ((st = fill_nan(p->numsys, (CUdeviceptr)outputs[k], p->out_elems[k], s))) return st;
  return launch_plan(p, inputs, outputs, s);
}

int sgm_plan_run_host(sgm_plan* p, const void* const* host_inputs, void* const* host_outputs, void* stream) {
  if (!p || !p->fn) return set_err(SGM_ERR_INVALID, "null plan / no device");
  int st = ensure_ctx();
  if (st) return st;
  size_t tot = 0;
  for (int k = 0; k < p->n_in; ++k) tot += (p->in_bytes[k] + 255) / 256 * 256;
  for (int k = 0; k < p->n_out; ++k) tot += (p->out_bytes[k] + 255) / 256 * 256;
  DevState& S = g_dev[p->device];
  std::lock_guard<std::mutex> lk(S.io_mu);
  if (tot > S.io_bytes) {
    if (S.pinned) D.cuMemFreeHost(S.pinned);
    if (S.dev_io) D.cuMemFree(S.dev_io);
    S.pinned = nullptr;
    S.dev_io = 0;
    S.io_bytes = 0;
    CU(D.cuMemHostAlloc(&S.pinned, tot, 0));
    CU(D.cuMemAlloc(&S.dev_io, tot));
    S.io_bytes = tot;
  }
  CUstream s = (CUstream)stream;
  const void* din[SGM_MAX_SLOTS];
  void* dout[SGM_MAX_SLOTS];
  size_t off = 0;
  for (int k = 0; k < p->n_in; ++k) {
    memcpy((char*)S.pinned + off, host_inputs[k], p->in_bytes[k]);
    CU(D.cuMemcpyHtoDAsync(S.dev_io + off, (char*)S.pinned + off, p->in_bytes[k], s));
    din[k] = (const void*)(S.dev_io + off);
    off += (p->in_bytes[k] + 255) / 256 * 256;
  }
  size_t out0 = off;
  for (int k = 0; k < p->n_out; ++k) {
    dout[k] = (void*)(S.dev_io + off);
    if ((st = fill_nan(p->numsys, (CUdeviceptr)dout[k], p->out_elems[k], s))) return st;
    off += (p->out_bytes[k] + 255) / 256 * 256;
  }
  if ((st = launch_plan(p, din, dout, s))) return st;
  off = out0;
  for (int k = 0; k < p->n_out; ++k) {
    CU(D.cuMemcpyDtoHAsync((char*)S.pinned + off, (CUdeviceptr)dout[k], p->out_bytes[k], s));
    off += (p->out_bytes[k] + 255) / 256 * 256;
  }
  CU(D.cuStreamSynchronize(s));
  off = out0;
  for (int k = 0; k < p->n_out; ++k) {
    memcpy(host_outputs[k], (char*)S.pinned + off, p->out_bytes[k]);
    off += (p->out_bytes[k] + 255) / 256 * 256;
  }
  return SGM_OK;
}

static int plan_graph(sgm_plan* p, const void* const* inputs, void* const* outputs, int rot);

int sgm_plan_time(sgm_plan* p, const void* const* inputs, void* const* outputs, int rot, int warmup, int iters,
                  void* stream, double* mean_us) {
  if (!p || !p->fn || !mean_us) return set_err(SGM_ERR_INVALID, "null plan / no device");
  int st = ensure_ctx();
  if (st) return st;
  if (rot < 1) rot = 1;
  if (iters < 1) iters = 1;
  CUstream user = (CUstream)stream;
  if (user) CU(D.cuStreamSynchronize(user));
  if ((st = plan_graph(p, inputs, outputs, rot))) return st;
  CUstream s = p->tstream;
  for (int w = 0; w < warmup; ++w)
    if ((st = launch_plan(p, inputs + (size_t)(w % rot) * p->n_in, outputs, s))) return st;
  const int reps = (iters + rot - 1) / rot;
  CUevent e0, e1;
  CU(D.cuEventCreate(&e0, 0));
  CU(D.cuEventCreate(&e1, 0));
  CU(D.cuGraphLaunch(p->gexec, s));  // warm the graph once
  CU(D.cuEventRecord(e0, s));
  for (int r = 0; r < reps; ++r) CU(D.cuGraphLaunch(p->gexec, s));
  CU(D.cuEventRecord(e1, s));
  CU(D.cuEventSynchronize(e1));
  g_launches += (long long)rot * (reps + 1);
  float ms = 0;
  CU(D.cuEventElapsedTime(&ms, e0, e1));
  *mean_us = (double)ms * 1000.0 / ((double)reps * rot);
  D.cuEventDestroy(e0);
  D.cuEventDestroy(e1);
  return SGM_OK;
}

// (Re)build the plan's cached graph: `rot` launches, launch i reading input set i.
static int plan_graph(sgm_plan* p, const void* const* inputs, void* const* outputs, int rot) {
  std::vector<const void*> key(inputs, inputs + (size_t)rot * p->n_in);
  key.insert(key.end(), outputs, outputs + p->n_out);
  const int pdl = pdl_on() ? 1 : 0;
  if (p->gexec && p->graph_rot == rot && p->graph_pdl == pdl && key == p->graph_key) return SGM_OK;
  if (p->gexec) { D.cuGraphExecDestroy(p->gexec); p->gexec = nullptr; }
  if (p->graph) { D.cuGraphDestroy(p->graph); p->graph = nullptr; }
  if (!p->tstream) CU(D.cuStreamCreate(&p->tstream, CU_STREAM_NON_BLOCKING));
  CU(D.cuStreamBeginCapture(p->tstream, CU_STREAM_CAPTURE_MODE_THREAD_LOCAL));
  int st = SGM_OK;
  for (int i = 0; i < rot && !st; ++i) st = launch_plan(p, inputs + (size_t)i * p->n_in, outputs, p->tstream);
  CUgraph g = nullptr;
  CUresult r = D.cuStreamEndCapture(p->tstream, &g);
  if (st) { if (g) D.cuGraphDestroy(g); return st; }
  if (r != CUDA_SUCCESS) return cu_check(r, "cuStreamEndCapture");
  r = D.cuGraphInstantiateWithFlags(&p->gexec, g, 0);
  if (r != CUDA_SUCCESS) { D.cuGraphDestroy(g); return cu_check(r, "cuGraphInstantiate"); }
  p->graph = g;
  p->graph_key = key;
  p->graph_rot = rot;
  p->graph_pdl = pdl;
  return SGM_OK;
}

int sgm_timer_create(int capacity, sgm_timer** out) {
  int st = ensure_ctx();
  if (st) return st;
  if (capacity < 1 || !out) return set_err(SGM_ERR_INVALID, "bad timer capacity");
  sgm_timer* t = new sgm_timer();
  t->cap = capacity;
  t->device = t_device;
  t->ev.resize((size_t)capacity * 2, nullptr);
  t->launches.assign(capacity, 0);
  for (auto& e : t->ev) {
    CUresult r = D.cuEventCreate(&e, 0);
    if (r != CUDA_SUCCESS) { sgm_timer_destroy(t); return cu_check(r, "cuEventCreate"); }
  }
  *out = t;
  return SGM_OK;
}

int sgm_timer_enqueue(sgm_timer* t, int slot, sgm_plan* p, const void* const* inputs, void* const* outputs, int rot,
                      int warmup, int reps, void* stream) {
  if (!t || !p || !p->fn || slot < 0 || slot >= t->cap) return set_err(SGM_ERR_INVALID, "bad timer / plan / slot");
  int st = ensure_ctx();
  if (st) return st;
  if (rot < 1) rot = 1;
  if (reps < 1) reps = 1;
  if ((st = plan_graph(p, inputs, outputs, rot))) return st;
  CUstream s = (CUstream)stream;
  for (int w = 0; w < warmup; ++w) CU(D.cuGraphLaunch(p->gexec, s));  // instruction cache, TMA descriptors
  CU(D.cuEventRecord(t->ev[2 * slot], s));
  for (int r = 0; r < reps; ++r) CU(D.cuGraphLaunch(p->gexec, s));
  CU(D.cuEventRecord(t->ev[2 * slot + 1], s));
  g_launches += (long long)rot * (reps + (warmup > 0 ? warmup : 0));
  t->launches[slot] = rot * reps;
  if (slot > t->last) t->last = slot;
  return SGM_OK;
}

int sgm_timer_read(sgm_timer* t, int n, double* us) {
  if (!t || !us || n < 0 || n > t->cap) return set_err(SGM_ERR_INVALID, "bad timer read");
  int st = ensure_ctx();
  if (st) return st;
  for (int k = 0; k < n; ++k) {
    if (!t->launches[k]) { us[k] = -1.0; continue; }
    CU(D.cuEventSynchronize(t->ev[2 * k + 1]));
    float ms = 0;
    CU(D.cuEventElapsedTime(&ms, t->ev[2 * k], t->ev[2 * k + 1]));
    us[k] = (double)ms * 1000.0 / t->launches[k];
  }
  return SGM_OK;
}

int sgm_timer_destroy(sgm_timer* t) {
  if (!t) return SGM_OK;
  for (auto e : t->ev)
    if (e) D.cuEventDestroy(e);
  delete t;
  return SGM_OK;
}

int sgm_compare_u32_acc(const uint32_t* a, const uint32_t* b, int64_t n, void* stream, int64_t* dev_counter) {
  int st = ensure_ctx();
  if (st) return st;
  DevState& S = g_dev[t_device];
  CUdeviceptr pa = (CUdeviceptr)a, pb = (CUdeviceptr)b, pc = (CUdeviceptr)dev_counter;
  void* args[] = {&pa, &pb, &n, &pc};
  return launch_1d(S.f_cmp, n, (CUstream)stream, args);
}

int sgm_ff_fill(uint32_t* dst, int64_t n, uint64_t seed, uint64_t salt, void* stream) {
  int st = ensure_ctx();
  if (st) return st;
  auto mix = [](uint64_t z) {
    z ^= z >> 30; z *= 0xbf58476d1ce4e5b9ULL;
    z ^= z >> 27; z *= 0x94d049bb133111ebULL;
    z ^= z >> 31;
    return z;
  };
  uint64_t key = mix(seed ^ mix(salt));
  CUdeviceptr p = (CUdeviceptr)dst;
  void* a[] = {&p, &n, &key};
  return launch_1d(g_dev[t_device].f_ff_fill, n, (CUstream)stream, a);
}

int sgm_compare_u32(const uint32_t* a, const uint32_t* b, int64_t n, void* stream, int64_t* mismatches) {
  int st = ensure_ctx();
  if (st) return st;
  DevState& S = g_dev[t_device];
  CUstream s = (CUstream)stream;
  CU(D.cuMemsetD32Async(S.red, 0, 16, s));
  CUdeviceptr pa = (CUdeviceptr)a, pb = (CUdeviceptr)b;
  void* args[] = {&pa, &pb, &n, &S.red};
  if ((st = launch_1d(S.f_cmp, n, s, args))) return st;
  uint64_t c = 0;
  CU(D.cuMemcpyDtoHAsync(&c, S.red, 8, s));
  CU(D.cuStreamSynchronize(s));
  *mismatches = (int64_t)c;
  return SGM_OK;
}

int sgm_rel_err(const void* a, const void* b, int64_t n, int numsys, void* stream, double* out) {
  int st = ensure_ctx();
  if (st) return st;
  DevState& S = g_dev[t_device];
  CUstream s = (CUstream)stream;
  CU(D.cuMemsetD32Async(S.red, 0, 16, s));
  CUdeviceptr pa = (CUdeviceptr)a, pb = (CUdeviceptr)b;
  void* args[] = {&pa, &pb, &n, &S.red};
  CUfunction f = numsys == SGM_F64 ? S.f_re64 : numsys == SGM_BF16 ? S.f_re16 : S.f_re32;
  if (numsys == SGM_FF) return set_err(SGM_ERR_INVALID, "rel_err is undefined for finite-field buffers");
  if ((st = launch_1d(f, n, s, args))) return st;
  uint64_t r[3] = {0, 0, 0};
  CU(D.cuMemcpyDtoHAsync(r, S.red, 24, s));
  CU(D.cuStreamSynchronize(s));
  double md, mb;
  memcpy(&md, &r[0], 8);
  memcpy(&mb, &r[1], 8);
  *out = r[2] ? INFINITY : md / (1.0 + mb);
  return SGM_OK;
}

int sgm_plan_watchdog(sgm_plan* p, void* stream, int reset, int* tripped) {
  if (!p || !p->fn || !tripped) return set_err(SGM_ERR_INVALID, "null plan / no device");
  int st = ensure_ctx();
  if (st) return st;
  *tripped = 0;
  if (!p->wd_flag) return SGM_OK;
  CUstream s = (CUstream)stream;
  unsigned v = 0;
  CU(D.cuMemcpyDtoHAsync(&v, p->wd_flag, 4, s));
  CU(D.cuStreamSynchronize(s));
  *tripped = v != 0;
  if (v && reset) {
    CU(D.cuMemsetD32Async(p->wd_flag, 0, 1, s));
    CU(D.cuStreamSynchronize(s));
  }
  return SGM_OK;
}

int sgm_set_pdl(int on) {
  g_pdl.store(on ? 1 : 0);
  return SGM_OK;
}

int sgm_rel_err_acc(const void* a, int numsys, const double* b, int64_t n, void* stream, uint64_t* dev_slot) {
  int st = ensure_ctx();
  if (st) return st;
  DevState& S = g_dev[t_device];
  if (numsys == SGM_FF) return set_err(SGM_ERR_INVALID, "rel_err is undefined for finite-field buffers");
  CUdeviceptr pa = (CUdeviceptr)a, pb = (CUdeviceptr)b, pc = (CUdeviceptr)dev_slot;
  void* args[] = {&pa, &pb, &n, &pc};
  CUfunction f = numsys == SGM_F64 ? S.f_re64 : numsys == SGM_BF16 ? S.f_rex16 : S.f_rex32;
  return launch_1d(f, n, (CUstream)stream, args);
}

int sgm_fill_normal(void* dst, int64_t n, int numsys, uint64_t seed, void* stream) {
  int st = ensure_ctx();
  if (st) return st;
  DevState& S = g_dev[t_device];
  CUdeviceptr p = (CUdeviceptr)dst;
  void* a[] = {&p, &n, &seed};
  CUfunction f = numsys == SGM_F64 ? S.f_n64 : numsys == SGM_BF16 ? S.f_n16 : S.f_n32;
  if (numsys == SGM_FF) return sgm_ff_fill((uint32_t*)dst, n, seed, 0, stream);
  return launch_1d(f, n, (CUstream)stream, a);
}

}  // extern "C"
