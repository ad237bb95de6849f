// Driver-API entry points resolved at run time through the CUDA runtime
// (cudaGetDriverEntryPoint) rather than linked against libcuda: the library
// must load — and report "no GPU" cleanly — on machines without a driver.
#include "lgp_internal.h"

namespace lgp {
namespace drv {
namespace {
template <class F>
F resolve(const char* name) {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &fn, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || fn == nullptr) {
    cudaGetLastError();
    throw Error(LGP_E_CUDA, std::string("driver entry point unavailable: ") + name);
  }
  return reinterpret_cast<F>(fn);
}
}  // namespace

#define LGP_DRV(name, ret, params, args)                         \
  ret name params {                                              \
    static auto fn = resolve<ret(*) params>("cu" #name);         \
    return fn args;                                              \
  }

LGP_DRV(ModuleLoadData, CUresult, (CUmodule * m, const void* image), (m, image))
LGP_DRV(ModuleUnload, CUresult, (CUmodule m), (m))
LGP_DRV(ModuleGetFunction, CUresult, (CUfunction * f, CUmodule m, const char* name), (f, m, name))
LGP_DRV(FuncSetAttribute, CUresult, (CUfunction f, CUfunction_attribute a, int v), (f, a, v))
LGP_DRV(FuncGetAttribute, CUresult, (int* v, CUfunction_attribute a, CUfunction f), (v, a, f))
LGP_DRV(OccupancyMaxActiveBlocksPerMultiprocessor, CUresult,
        (int* n, CUfunction f, int bs, size_t smem), (n, f, bs, smem))
LGP_DRV(LaunchKernel, CUresult,
        (CUfunction f, unsigned gx, unsigned gy, unsigned gz, unsigned bx, unsigned by,
         unsigned bz, unsigned smem, CUstream s, void** params, void** extra),
        (f, gx, gy, gz, bx, by, bz, smem, s, params, extra))
LGP_DRV(GetErrorString, CUresult, (CUresult r, const char** s), (r, s))

}  // namespace drv
}  // namespace lgp
