// Runtime specialisation: compile generated CUDA C for sm_100a with NVRTC.
//
// The engine generates kernels for region shapes whose generic execution
// would be interpretive (pointwise programs, arbitrary loop nests): every
// stride, trip count and the op sequence become compile-time constants, so
// the kernel is straight-line native code.  NVRTC is loaded with dlopen
// (libnvrtc.so.12 ships with the CUDA toolkit in this image) and modules are
// loaded / launched through driver entry points obtained from the runtime
// (cudaGetDriverEntryPoint), so libb200k.so has no extra link dependency.
// Compilation is -arch=sm_100a, --fmad=false (the generated code also uses
// explicit __f*_rn intrinsics so f32 ops are never contracted).
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <mutex>
#include <string>
#include <vector>

#include "../../include/b200k.h"

namespace {

typedef int nvrtcResult_;
typedef struct _nvrtcProgram *nvrtcProgram_;
typedef nvrtcResult_ (*PCreate)(nvrtcProgram_ *, const char *, const char *, int,
                                const char *const *, const char *const *);
typedef nvrtcResult_ (*PCompile)(nvrtcProgram_, int, const char *const *);
typedef nvrtcResult_ (*PGetSize)(nvrtcProgram_, size_t *);
typedef nvrtcResult_ (*PGetData)(nvrtcProgram_, char *);
typedef nvrtcResult_ (*PDestroy)(nvrtcProgram_ *);

struct Nvrtc {
  bool ok = false;
  PCreate create;
  PCompile compile;
  PGetSize log_size, cubin_size;
  PGetData log, cubin;
  PDestroy destroy;
};

typedef CUresult (*PModLoad)(CUmodule *, const void *);
typedef CUresult (*PGetFunc)(CUfunction *, CUmodule, const char *);
typedef CUresult (*PLaunch)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned,
                            unsigned, unsigned, CUstream, void **, void **);
typedef CUresult (*PFuncSetAttr)(CUfunction, CUfunction_attribute, int);

struct Driver {
  bool ok = false;
  PModLoad load;
  PGetFunc get;
  PLaunch launch;
  PFuncSetAttr set_attr;
};

std::mutex g_mu;
Nvrtc g_nv;
Driver g_drv;
std::string g_log;

bool init_nvrtc() {
  if (g_nv.ok) return true;
  const char *names[] = {"libnvrtc.so.12", "libnvrtc.so", "/usr/local/cuda/lib64/libnvrtc.so.12"};
  void *h = nullptr;
  for (const char *n : names)
    if ((h = dlopen(n, RTLD_NOW | RTLD_GLOBAL))) break;
  if (!h) {
    g_log = "dlopen(libnvrtc.so.12) failed";
    return false;
  }
  g_nv.create = (PCreate)dlsym(h, "nvrtcCreateProgram");
  g_nv.compile = (PCompile)dlsym(h, "nvrtcCompileProgram");
  g_nv.log_size = (PGetSize)dlsym(h, "nvrtcGetProgramLogSize");
  g_nv.log = (PGetData)dlsym(h, "nvrtcGetProgramLog");
  g_nv.cubin_size = (PGetSize)dlsym(h, "nvrtcGetCUBINSize");
  g_nv.cubin = (PGetData)dlsym(h, "nvrtcGetCUBIN");
  g_nv.destroy = (PDestroy)dlsym(h, "nvrtcDestroyProgram");
  g_nv.ok = g_nv.create && g_nv.compile && g_nv.log_size && g_nv.log && g_nv.cubin_size &&
            g_nv.cubin && g_nv.destroy;
  if (!g_nv.ok) g_log = "libnvrtc is missing symbols";
  return g_nv.ok;
}

template <typename F>
bool entry(const char *name, F &fn) {
  void *p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess)
    return false;
  fn = reinterpret_cast<F>(p);
  return true;
}

bool init_driver() {
  if (g_drv.ok) return true;
  cudaFree(nullptr);  // make sure the primary context is current
  g_drv.ok = entry("cuModuleLoadData", g_drv.load) && entry("cuModuleGetFunction", g_drv.get) &&
             entry("cuLaunchKernel", g_drv.launch) &&
             entry("cuFuncSetAttribute", g_drv.set_attr);
  if (!g_drv.ok) g_log = "driver entry points unavailable";
  return g_drv.ok;
}

// NVRTC: `src` -> sm_100a cubin (caller holds g_mu).
int compile_cubin(const char *src, std::vector<char> &cubin) {
  if (!init_nvrtc()) return B200_EUNSUPPORTED;
  nvrtcProgram_ prog;
  if (g_nv.create(&prog, src, "b200_jit.cu", 0, nullptr, nullptr) != 0) return B200_EINVAL;
  const char *opts[] = {"-arch=sm_100a", "--fmad=false", "-std=c++17", "-default-device",
                        "-lineinfo"};
  const int rc = g_nv.compile(prog, 5, opts);
  size_t n = 0;
  g_nv.log_size(prog, &n);
  g_log.assign(n, '\0');
  if (n) g_nv.log(prog, &g_log[0]);
  if (rc != 0) {
    g_nv.destroy(&prog);
    return B200_EINVAL;
  }
  size_t cn = 0;
  g_nv.cubin_size(prog, &cn);
  cubin.resize(cn);
  g_nv.cubin(prog, cubin.data());
  g_nv.destroy(&prog);
  return B200_OK;
}

// cubin image -> CUfunction (caller holds g_mu).
int load_cubin(const void *image, const char *kernel, void **fn) {
  if (!init_driver()) return B200_EUNSUPPORTED;
  CUmodule mod;
  if (g_drv.load(&mod, image) != CUDA_SUCCESS) {
    g_log = "cuModuleLoadData failed";
    return B200_ELAUNCH;
  }
  CUfunction f;
  if (g_drv.get(&f, mod, kernel) != CUDA_SUCCESS) {
    g_log = "cuModuleGetFunction failed";
    return B200_ELAUNCH;
  }
  *fn = reinterpret_cast<void *>(f);
  return B200_OK;
}

}  // namespace

// Compile `src` and return the CUfunction for `kernel` in *fn (opaque).
extern "C" int b200_jit_compile(const char *src, const char *kernel, void **fn) {
  std::lock_guard<std::mutex> lock(g_mu);
  if (!init_nvrtc() || !init_driver()) return B200_EUNSUPPORTED;
  std::vector<char> cubin;
  const int rc = compile_cubin(src, cubin);
  return rc != B200_OK ? rc : load_cubin(cubin.data(), kernel, fn);
}

// Compile `src` to an sm_100a cubin without loading it (no GPU needed): the
// image is copied into out (capacity cap bytes); *size receives its length
// (B200_EINVAL with *size set when cap is too small).
extern "C" int b200_jit_cubin(const char *src, void *out, size_t cap, size_t *size) {
  std::lock_guard<std::mutex> lock(g_mu);
  std::vector<char> cubin;
  const int rc = compile_cubin(src, cubin);
  if (rc != B200_OK) return rc;
  *size = cubin.size();
  if (cubin.size() > cap) return B200_EINVAL;
  memcpy(out, cubin.data(), cubin.size());
  return B200_OK;
}

// Load a cubin produced by b200_jit_cubin (e.g. from the on-disk kernel
// cache) and return the CUfunction for `kernel`.
extern "C" int b200_jit_load(const void *image, const char *kernel, void **fn) {
  std::lock_guard<std::mutex> lock(g_mu);
  return load_cubin(image, kernel, fn);
}


// The compiler log of the last b200_jit_compile (for diagnostics).
extern "C" const char *b200_jit_log(void) { return g_log.c_str(); }

// Launch a compiled kernel: args is an array of pointers to the argument values.
extern "C" int b200_jit_launch(void *fn, uint32_t gx, uint32_t gy, uint32_t gz, uint32_t bx,
                               uint32_t by, uint32_t bz, uint32_t smem, void **args,
                               void *stream) {
  if (!g_drv.ok && !init_driver()) return B200_EUNSUPPORTED;
  CUfunction f = reinterpret_cast<CUfunction>(fn);
  if (smem > 48 * 1024)
    g_drv.set_attr(f, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, (int)smem);
  CUresult r = g_drv.launch(f, gx, gy, gz, bx, by, bz, smem, static_cast<CUstream>(stream), args,
                            nullptr);
  return r == CUDA_SUCCESS ? B200_OK : B200_ELAUNCH;
}
