// Run-time compilation of user combination integrals (CombinationIntegral / pairwise /
// combine_integrate / integrate_single, integrate.py:51-203, matrix.py:273-283).
//
// The reference evaluates an arbitrary Python callable once per rectangle.  Here the
// Python layer (jit.py) translates the callable into a C expression; this file compiles
// pcf_jit_kernels.cuh with those definitions through NVRTC for sm_100a (--fmad=false, so
// arithmetic integrands reproduce the reference bit for bit), loads the CUBIN with the
// driver API and launches its kernels on the caller's stream.  libnvrtc and libcuda are
// opened at run time (dlopen), so the library still loads on machines without a driver.
#include <dlfcn.h>
#include <stdio.h>
#include <string.h>
#include <cmath>
#include <mutex>
#include <string>
#include <vector>
#include "pcf_internal.h"

namespace pcfb {
namespace {

const char* kJitSource =
#include "pcf_jit_src.inc"
    ;
const char* kCommonSource =
#include "pcf_common_src.inc"
    ;
const char* kTilesSource =
#include "pcf_tiles_src.inc"
    ;

// ---- NVRTC (subset of nvrtc.h)
typedef int nvrtcResult;
typedef struct _nvrtcProgram* nvrtcProgram;
struct Nvrtc {
  bool ok = false;
  std::string why;
  nvrtcResult (*create)(nvrtcProgram*, const char*, const char*, int, const char* const*,
                        const char* const*) = nullptr;
  nvrtcResult (*compile)(nvrtcProgram, int, const char* const*) = nullptr;
  nvrtcResult (*log_size)(nvrtcProgram, size_t*) = nullptr;
  nvrtcResult (*log)(nvrtcProgram, char*) = nullptr;
  nvrtcResult (*cubin_size)(nvrtcProgram, size_t*) = nullptr;
  nvrtcResult (*cubin)(nvrtcProgram, char*) = nullptr;
  nvrtcResult (*destroy)(nvrtcProgram*) = nullptr;
  const char* (*err)(nvrtcResult) = nullptr;
  nvrtcResult (*add_name)(nvrtcProgram, const char*) = nullptr;
  nvrtcResult (*lowered)(nvrtcProgram, const char*, const char**) = nullptr;
};

// ---- driver API (subset of cuda.h)
typedef int CUresult;
typedef struct CUmod_st* CUmodule;
typedef struct CUfunc_st* CUfunction;
typedef struct CUstream_st* CUstream;
struct Driver {
  bool ok = false;
  std::string why;
  CUresult (*load)(CUmodule*, const void*) = nullptr;
  CUresult (*unload)(CUmodule) = nullptr;
  CUresult (*getfn)(CUfunction*, CUmodule, const char*) = nullptr;
  CUresult (*launch)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned,
                     unsigned, CUstream, void**, void**) = nullptr;
  CUresult (*errstr)(CUresult, const char**) = nullptr;
  CUresult (*setattr)(CUfunction, int, int) = nullptr;
};

std::once_flag g_nvrtc_once, g_drv_once;
Nvrtc g_nvrtc;
Driver g_drv;

void* open_first(const char* const* names, std::string* why) {
  for (const char* const* n = names; *n; ++n) {
    void* h = dlopen(*n, RTLD_NOW | RTLD_LOCAL);
    if (h) return h;
  }
  const char* e = dlerror();
  *why = e ? e : "dlopen failed";
  return nullptr;
}

template <typename F>
bool sym(void* h, const char* name, F* out, std::string* why) {
  *out = reinterpret_cast<F>(dlsym(h, name));
  if (!*out) {
    *why = std::string("missing symbol ") + name;
    return false;
  }
  return true;
}

void init_nvrtc() {
  static const char* names[] = {"libnvrtc.so.12", "libnvrtc.so",
                                "/usr/local/cuda/lib64/libnvrtc.so.12", nullptr};
  void* h = open_first(names, &g_nvrtc.why);
  if (!h) return;
  g_nvrtc.ok = sym(h, "nvrtcCreateProgram", &g_nvrtc.create, &g_nvrtc.why) &&
               sym(h, "nvrtcCompileProgram", &g_nvrtc.compile, &g_nvrtc.why) &&
               sym(h, "nvrtcGetProgramLogSize", &g_nvrtc.log_size, &g_nvrtc.why) &&
               sym(h, "nvrtcGetProgramLog", &g_nvrtc.log, &g_nvrtc.why) &&
               sym(h, "nvrtcGetCUBINSize", &g_nvrtc.cubin_size, &g_nvrtc.why) &&
               sym(h, "nvrtcGetCUBIN", &g_nvrtc.cubin, &g_nvrtc.why) &&
               sym(h, "nvrtcDestroyProgram", &g_nvrtc.destroy, &g_nvrtc.why) &&
               sym(h, "nvrtcGetErrorString", &g_nvrtc.err, &g_nvrtc.why) &&
               sym(h, "nvrtcAddNameExpression", &g_nvrtc.add_name, &g_nvrtc.why) &&
               sym(h, "nvrtcGetLoweredName", &g_nvrtc.lowered, &g_nvrtc.why);
}

void init_driver() {
  static const char* names[] = {"libcuda.so.1", "libcuda.so", nullptr};
  void* h = open_first(names, &g_drv.why);
  if (!h) return;
  g_drv.ok = sym(h, "cuModuleLoadData", &g_drv.load, &g_drv.why) &&
             sym(h, "cuModuleUnload", &g_drv.unload, &g_drv.why) &&
             sym(h, "cuModuleGetFunction", &g_drv.getfn, &g_drv.why) &&
             sym(h, "cuLaunchKernel", &g_drv.launch, &g_drv.why) &&
             sym(h, "cuGetErrorString", &g_drv.errstr, &g_drv.why) &&
             sym(h, "cuFuncSetAttribute", &g_drv.setattr, &g_drv.why);
}

int drv_fail(CUresult r, const char* where) {
  const char* s = nullptr;
  if (g_drv.errstr) g_drv.errstr(r, &s);
  set_error("%s: CUDA driver error %d (%s)", where, r, s ? s : "?");
  return PCF_ERR_CUDA;
}

struct JitModule {
  CUmodule mod = nullptr;
  CUfunction matrix = nullptr, pairs = nullptr, single = nullptr;
};

// NVRTC: source (+ the embedded headers pcf_common.cuh / pcf_tiles.cuh) -> sm_100a CUBIN;
// `names` are template instantiations to export, their mangled names go to `lowered`
int compile_src(const std::string& src, const std::vector<std::string>& names,
                std::vector<char>* cubin, std::vector<std::string>* lowered, char* log,
                int64_t logcap) {
  std::call_once(g_nvrtc_once, init_nvrtc);
  if (!g_nvrtc.ok) {
    set_error("pcf_jit: NVRTC unavailable: %s", g_nvrtc.why.c_str());
    return PCF_ERR_CUDA;
  }
  nvrtcProgram prog = nullptr;
  const char* hdrs[] = {kCommonSource, kTilesSource};
  const char* hnames[] = {"pcf_common.cuh", "pcf_tiles.cuh"};
  nvrtcResult r = g_nvrtc.create(&prog, src.c_str(), "pcf_jit.cu", 2, hdrs, hnames);
  if (r) {
    set_error("pcf_jit: nvrtcCreateProgram: %s", g_nvrtc.err(r));
    return PCF_ERR_CUDA;
  }
  for (const auto& n : names) g_nvrtc.add_name(prog, n.c_str());
  const char* opts[] = {"--gpu-architecture=sm_100a", "--fmad=false", "--std=c++17",
                        "-default-device"};
  r = g_nvrtc.compile(prog, 4, opts);
  size_t ls = 0;
  g_nvrtc.log_size(prog, &ls);
  std::string lg(ls ? ls : 1, '\0');
  if (ls) g_nvrtc.log(prog, &lg[0]);
  if (log && logcap > 0) {
    const size_t n = std::min<size_t>(strlen(lg.c_str()), (size_t)logcap - 1);
    memcpy(log, lg.c_str(), n);
    log[n] = '\0';
  }
  if (r) {
    set_error("pcf_jit: compile failed: %.400s", lg.c_str());
    g_nvrtc.destroy(&prog);
    return PCF_ERR_ARG;
  }
  size_t n = 0;
  g_nvrtc.cubin_size(prog, &n);
  cubin->resize(n);
  g_nvrtc.cubin(prog, cubin->data());
  if (lowered) {
    lowered->clear();
    for (const auto& nm : names) {
      const char* low = nullptr;
      g_nvrtc.lowered(prog, nm.c_str(), &low);
      lowered->push_back(low ? std::string(low) : std::string());
    }
  }
  g_nvrtc.destroy(&prog);
  return PCF_OK;
}

int compile_cubin(const char* defs, std::vector<char>* cubin, char* log, int64_t logcap) {
  return compile_src(std::string(defs) + "\n" + kJitSource, {}, cubin, nullptr, log, logcap);
}

// The tile kernels (K1, K1c, K1r, K1g) instantiated with HK = H_USER for one record kind,
// both bound kinds: f[kernel][bounded], kernel 0 = K1, 1 = K1c, 2 = K1r, 3 = K1g, 4 = K1s.
struct JitTiles {
  CUmodule mod = nullptr;
  CUfunction f[5][2] = {};
  int f32 = 0;
};

std::string tiles_source(const char* defs, int f32) {
  std::string src = std::string(defs) + "\n" + kJitSource;
  src +=
      "\nnamespace pcfb {\n"
      "constexpr int kTileThreads = 512;\n"
      "struct PcfWorkItem { int row0, nrows, col0, col1, logC, log2G, smem_mode, cost_hi; };\n"
      "__device__ double pcf_user_h(double x, double y) { return ::pcf_h(x, y); }\n";
  src += "#if PCF_HAS_R\n__device__ double pcf_user_r(double x) { return ::pcf_r(x); }\n"
         "#else\n__device__ double pcf_user_r(double x) { return x; }\n#endif\n}\n";
  src += "#include \"pcf_tiles.cuh\"\n";
  (void)f32;
  return src;
}

std::vector<std::string> tiles_names(int f32) {
  const char* out = f32 ? "float" : "double";
  const char* rec = f32 ? "pcfb::Rec32" : "pcfb::Rec";
  const char* gw = f32 ? "16" : "8";
  std::vector<std::string> v;
  for (int b = 0; b < 2; ++b) {
    const char* bd = b ? "true" : "false";
    char buf[256];
    snprintf(buf, sizeof buf, "pcfb::k_fill_tiles_smem<5, %s, %s, %s, %s>", bd, out, rec, gw);
    v.push_back(buf);
    snprintf(buf, sizeof buf, "pcfb::k_fill_colgroups<5, %s, %s, %s, %s>", bd, out, rec, gw);
    v.push_back(buf);
    snprintf(buf, sizeof buf, "pcfb::k_fill_rowres<5, %s, %s, %s>", bd, out, rec);
    v.push_back(buf);
    snprintf(buf, sizeof buf, "pcfb::k_fill_tiles_global<5, %s, %s, %s>", bd, out, rec);
    v.push_back(buf);
    snprintf(buf, sizeof buf, "pcfb::k_fill_rows_staged<5, %s, %s, %s, %s>", bd, out, rec, gw);
    v.push_back(buf);
  }
  return v;
}

unsigned grid_for(long long n, int threads, unsigned cap) {
  long long g = (n + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (unsigned)g;
}

}  // namespace
}  // namespace pcfb

using namespace pcfb;

extern "C" {

int pcf_jit_cubin(const char* defs, void* cubin_out, int64_t cap, int64_t* size, char* log,
                  int64_t logcap) {
  if (!defs || !size) {
    set_error("pcf_jit_cubin: bad arguments");
    return PCF_ERR_ARG;
  }
  std::vector<char> cubin;
  int rc = compile_cubin(defs, &cubin, log, logcap);
  if (rc) return rc;
  *size = (int64_t)cubin.size();
  if (cubin_out && cap >= (int64_t)cubin.size()) memcpy(cubin_out, cubin.data(), cubin.size());
  return PCF_OK;
}

int pcf_jit_load(const char* defs, void** module, char* log, int64_t logcap) {
  if (!defs || !module) {
    set_error("pcf_jit_load: bad arguments");
    return PCF_ERR_ARG;
  }
  *module = nullptr;
  std::vector<char> cubin;
  int rc = compile_cubin(defs, &cubin, log, logcap);
  if (rc) return rc;
  std::call_once(g_drv_once, init_driver);
  if (!g_drv.ok) {
    set_error("pcf_jit: CUDA driver unavailable: %s", g_drv.why.c_str());
    return PCF_ERR_CUDA;
  }
  cudaFree(0);  // the runtime's primary context becomes current for the driver API
  JitModule* m = new JitModule();
  CUresult r = g_drv.load(&m->mod, cubin.data());
  if (r) {
    delete m;
    return drv_fail(r, "pcf_jit_load cuModuleLoadData");
  }
  if ((r = g_drv.getfn(&m->matrix, m->mod, "pcf_jit_matrix")) ||
      (r = g_drv.getfn(&m->pairs, m->mod, "pcf_jit_pairs"))) {
    g_drv.unload(m->mod);
    delete m;
    return drv_fail(r, "pcf_jit_load cuModuleGetFunction");
  }
  // pcf_jit_single exists only for integrate_single definitions (PCF_HAS_U 1)
  if (!strstr(defs, "#define PCF_HAS_U 1") ||
      g_drv.getfn(&m->single, m->mod, "pcf_jit_single"))
    m->single = nullptr;
  *module = m;
  return PCF_OK;
}

int pcf_jit_tiles_cubin(const char* defs, int is_f32, int64_t* size, char* log, int64_t logcap) {
  if (!defs || !size) {
    set_error("pcf_jit_tiles_cubin: bad arguments");
    return PCF_ERR_ARG;
  }
  *size = 0;
  const auto names = tiles_names(is_f32);
  std::vector<char> cubin;
  std::vector<std::string> low;
  int rc = compile_src(tiles_source(defs, is_f32), names, &cubin, &low, log, logcap);
  if (rc) return rc;
  for (size_t k = 0; k < names.size(); ++k)
    if (low[k].empty()) {
      set_error("pcf_jit_tiles_cubin: no lowered name for %s", names[k].c_str());
      return PCF_ERR_CUDA;
    }
  *size = (int64_t)cubin.size();
  return PCF_OK;
}

int pcf_jit_tiles_load(const char* defs, int is_f32, void** module, char* log, int64_t logcap) {
  if (!defs || !module) {
    set_error("pcf_jit_tiles_load: bad arguments");
    return PCF_ERR_ARG;
  }
  *module = nullptr;
  const auto names = tiles_names(is_f32);
  std::vector<char> cubin;
  std::vector<std::string> low;
  int rc = compile_src(tiles_source(defs, is_f32), names, &cubin, &low, log, logcap);
  if (rc) return rc;
  std::call_once(g_drv_once, init_driver);
  if (!g_drv.ok) {
    set_error("pcf_jit: CUDA driver unavailable: %s", g_drv.why.c_str());
    return PCF_ERR_CUDA;
  }
  cudaFree(0);
  JitTiles* m = new JitTiles();
  m->f32 = is_f32;
  CUresult r = g_drv.load(&m->mod, cubin.data());
  if (r) {
    delete m;
    return drv_fail(r, "pcf_jit_tiles_load cuModuleLoadData");
  }
  for (int b = 0; b < 2; ++b)
    for (int k = 0; k < 5; ++k) {
      const std::string& ln = low[b * 5 + k];
      if (ln.empty() || (r = g_drv.getfn(&m->f[k][b], m->mod, ln.c_str()))) {
        g_drv.unload(m->mod);
        delete m;
        return r ? drv_fail(r, "pcf_jit_tiles_load cuModuleGetFunction")
                 : (set_error("pcf_jit_tiles_load: no lowered name for %s", names[b * 5 + k].c_str()),
                    PCF_ERR_CUDA);
      }
    }
  *module = m;
  return PCF_OK;
}

void pcf_jit_tiles_release(void* module) {
  JitTiles* m = (JitTiles*)module;
  if (!m) return;
  if (g_drv.ok && m->mod) g_drv.unload(m->mod);
  delete m;
}

int pcf_jit_fill_tiles(void* module, int smem_mode, const void* recs_dev, const void* recsg_dev,
                       const int64_t* soff_dev, const int64_t* goff_dev, const int32_t* perm_dev,
                       int64_t M, const void* items_dev, int64_t n_items, int32_t smem_bytes,
                       int32_t* counter_dev, int has_r, double a, double b, void* out_dev,
                       int64_t ld, unsigned long long* err_dev, void* stream) {
  JitTiles* m = (JitTiles*)module;
  if (!m || !recs_dev || !soff_dev || !perm_dev || !items_dev || !counter_dev || !out_dev ||
      !err_dev || ld < M || !(a >= 0.0) || !(a < b) || n_items > 0x7fffffff ||
      smem_mode < 0 || smem_mode > 4 ||
      ((smem_mode == 1 || smem_mode == 3 || smem_mode == 4) && (!recsg_dev || !goff_dev))) {
    set_error("pcf_jit_fill_tiles: bad arguments");
    return PCF_ERR_ARG;
  }
  if (n_items <= 0) return PCF_OK;
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t ce = cudaMemsetAsync(counter_dev, 0, sizeof(int32_t), st);
  if (ce != cudaSuccess) {
    set_error("pcf_jit_fill_tiles: %s", cudaGetErrorString(ce));
    return PCF_ERR_CUDA;
  }
  const int kern = smem_mode == 1 ? 0
                   : (smem_mode == 3 ? 1 : (smem_mode == 2 ? 2 : (smem_mode == 4 ? 4 : 3)));
  const int bounded = std::isinf(b) ? 0 : 1;
  CUfunction fn = m->f[kern][bounded];
  int dev = 0, nsm = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const unsigned grid = (unsigned)(kern == 3 ? 2 * nsm : nsm);
  const unsigned smem = kern == 3 ? 0u : (unsigned)smem_bytes;
  if (smem > 48 * 1024) {
    CUresult ra = g_drv.setattr(fn, 8 /* MAX_DYNAMIC_SHARED_SIZE_BYTES */, (int)smem);
    if (ra) return drv_fail(ra, "pcf_jit_fill_tiles smem attribute");
  }
  int n_ = (int)n_items, apply = has_r ? 1 : 0;
  double p = 0.0;
  long long ld_ = ld, M_ = M;
  const void* null_tag = nullptr;
  void* null_done = nullptr;
  CUresult r;
  if (kern <= 1 || kern == 4) {
    void* args[] = {&recs_dev, &recsg_dev, &soff_dev, &goff_dev, &perm_dev, &items_dev, &n_,
                    &counter_dev, &p, &a, &b, &apply, &out_dev, &ld_, &M_, &err_dev, &null_tag,
                    &null_done};
    const unsigned nthr = kern == 4 ? (unsigned)kK1sThreads : 512u;  // K1s: 20 warps
    r = g_drv.launch(fn, grid, 1, 1, nthr, 1, 1, smem, (CUstream)stream, args, nullptr);
  } else {
    void* args[] = {&recs_dev, &soff_dev, &perm_dev, &items_dev, &n_, &counter_dev, &p, &a, &b,
                    &apply, &out_dev, &ld_, &M_, &err_dev, &null_tag, &null_done};
    r = g_drv.launch(fn, grid, 1, 1, 512, 1, 1, smem, (CUstream)stream, args, nullptr);
  }
  return r ? drv_fail(r, "pcf_jit_fill_tiles launch") : PCF_OK;
}

void pcf_jit_release(void* module) {
  JitModule* m = (JitModule*)module;
  if (!m) return;
  if (g_drv.ok && m->mod) g_drv.unload(m->mod);
  delete m;
}

int pcf_jit_matrix(void* module, const void* recs_dev, const int64_t* soff_dev,
                   const int32_t* perm_dev, int64_t M, int sym, double a, double b,
                   void* out_dev, int out_f32, int64_t ld, int64_t r0, int64_t r1,
                   unsigned long long* errs_dev, void* stream) {
  JitModule* m = (JitModule*)module;
  if (!m || !m->matrix || !recs_dev || !soff_dev || !perm_dev || !out_dev || !errs_dev ||
      M < 1 || ld < M || r0 < 0 || r1 > M || !(a >= 0.0) || !(a < b)) {
    set_error("pcf_jit_matrix: bad arguments");
    return PCF_ERR_ARG;
  }
  if (r1 <= r0) return PCF_OK;
  long long M_ = M, ld_ = ld, r0_ = r0, r1_ = r1;
  int sym_ = sym ? 1 : 0, f32_ = out_f32 ? 1 : 0;
  void* args[] = {&recs_dev, &soff_dev, &perm_dev, &M_, &sym_, &a, &b, &out_dev, &f32_,
                  &ld_, &r0_, &r1_, &errs_dev};
  const unsigned gx = grid_for(M, 128, 1024);
  const long long rows = r1 - r0;
  const unsigned gy = (unsigned)(rows > 65535 ? 65535 : rows);
  CUresult r = g_drv.launch(m->matrix, gx, gy, 1, 128, 1, 1, 0, (CUstream)stream, args, nullptr);
  return r ? drv_fail(r, "pcf_jit_matrix launch") : PCF_OK;
}

int pcf_jit_pairs(void* module, const void* recs_dev, const int64_t* soff_dev,
                  const int64_t* pairs_dev, int64_t npairs, double a, double b, int out_f32,
                  double* res_dev, int32_t* status_dev, void* stream) {
  JitModule* m = (JitModule*)module;
  if (!m || !m->pairs || !recs_dev || !soff_dev || !pairs_dev || !res_dev || !status_dev ||
      npairs < 0 || !(a >= 0.0) || !(a < b)) {
    set_error("pcf_jit_pairs: bad arguments");
    return PCF_ERR_ARG;
  }
  if (npairs == 0) return PCF_OK;
  long long n_ = npairs;
  int f32_ = out_f32 ? 1 : 0;
  void* args[] = {&recs_dev, &soff_dev, &pairs_dev, &n_, &a, &b, &f32_, &res_dev, &status_dev};
  CUresult r = g_drv.launch(m->pairs, grid_for(npairs, 128, 8192), 1, 1, 128, 1, 1, 0,
                            (CUstream)stream, args, nullptr);
  return r ? drv_fail(r, "pcf_jit_pairs launch") : PCF_OK;
}

int pcf_jit_single(void* module, const void* recs_dev, const int64_t* soff_dev, int64_t M,
                   double a, double b, int out_f32, double* res_dev, int32_t* status_dev,
                   void* stream) {
  JitModule* m = (JitModule*)module;
  if (!m || !m->single || !recs_dev || !soff_dev || !res_dev || !status_dev || M < 0 ||
      !(a >= 0.0) || !(a < b)) {
    set_error("pcf_jit_single: bad arguments (module compiled without a single integrand?)");
    return PCF_ERR_ARG;
  }
  if (M == 0) return PCF_OK;
  long long M_ = M;
  int f32_ = out_f32 ? 1 : 0;
  void* args[] = {&recs_dev, &soff_dev, &M_, &a, &b, &f32_, &res_dev, &status_dev};
  CUresult r = g_drv.launch(m->single, grid_for(M, 128, 8192), 1, 1, 128, 1, 1, 0,
                            (CUstream)stream, args, nullptr);
  return r ? drv_fail(r, "pcf_jit_single launch") : PCF_OK;
}

}  // extern "C"
