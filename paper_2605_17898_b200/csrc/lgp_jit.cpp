// NVRTC JIT for sm_100a with an in-memory cache per context and an on-disk
// cubin cache (LGP_JIT_CACHE, default <package>/_lib/jit_cache) keyed by a
// hash of (source, options, NVRTC version). NVRTC runs on the host, so the
// cache can be warmed in a GPU-less build container and shipped with the
// package.
#include <dlfcn.h>
#include <nvrtc.h>
#include <sys/stat.h>
#include <unistd.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <atomic>
#include <mutex>
#include <vector>
#include <sstream>

#include "lgp_internal.h"

namespace lgp {
namespace {

// NVRTC is dlopen'ed by absolute path (RTLD_LOCAL): PyTorch wheels ship their
// own libnvrtc.so.12 (an older minor), and a soname-based dependency would
// bind to whichever copy the process loaded first.
struct NvrtcApi {
  void* h = nullptr;
  nvrtcResult (*Version)(int*, int*);
  nvrtcResult (*CreateProgram)(nvrtcProgram*, const char*, const char*, int, const char* const*,
                               const char* const*);
  nvrtcResult (*CompileProgram)(nvrtcProgram, int, const char* const*);
  nvrtcResult (*GetProgramLogSize)(nvrtcProgram, size_t*);
  nvrtcResult (*GetProgramLog)(nvrtcProgram, char*);
  nvrtcResult (*GetCUBINSize)(nvrtcProgram, size_t*);
  nvrtcResult (*GetCUBIN)(nvrtcProgram, char*);
  nvrtcResult (*DestroyProgram)(nvrtcProgram*);
  const char* (*GetErrorString)(nvrtcResult);
};

NvrtcApi& nvrtc() {
  static NvrtcApi a;
  static std::once_flag once;
  std::call_once(once, [] {
    std::vector<std::string> cands;
    if (const char* e = std::getenv("LGP_NVRTC")) cands.push_back(e);
    cands.push_back("/usr/local/cuda/lib64/libnvrtc.so.12");
    cands.push_back("libnvrtc.so.12");
    for (auto& c : cands) {
      a.h = dlopen(c.c_str(), RTLD_NOW | RTLD_LOCAL);
      if (a.h) break;
    }
    if (!a.h) return;
#define LGP_NVRTC_SYM(f) a.f = (decltype(a.f))dlsym(a.h, "nvrtc" #f)
    LGP_NVRTC_SYM(Version);
    LGP_NVRTC_SYM(CreateProgram);
    LGP_NVRTC_SYM(CompileProgram);
    LGP_NVRTC_SYM(GetProgramLogSize);
    LGP_NVRTC_SYM(GetProgramLog);
    LGP_NVRTC_SYM(GetCUBINSize);
    LGP_NVRTC_SYM(GetCUBIN);
    LGP_NVRTC_SYM(DestroyProgram);
    LGP_NVRTC_SYM(GetErrorString);
#undef LGP_NVRTC_SYM
  });
  if (!a.h || !a.CompileProgram || !a.GetCUBIN)
    throw Error(LGP_E_COMPILE, "libnvrtc.so.12 could not be loaded (set LGP_NVRTC)");
  return a;
}

const char* kOpts[] = {"--gpu-architecture=sm_100a", "-lineinfo", "--std=c++17",
                       "--ftz=true", "--ptxas-options=-v", "-default-device"};
const int kNumOpts = sizeof(kOpts) / sizeof(kOpts[0]);

uint64_t fnv1a(const std::string& s, uint64_t h = 1469598103934665603ull) {
  for (unsigned char c : s) {
    h ^= c;
    h *= 1099511628211ull;
  }
  return h;
}

std::string cache_dir() {
  if (const char* e = std::getenv("LGP_JIT_CACHE")) return e;
  // <dir of this .so>/jit_cache
  Dl_info info;
  if (dladdr((void*)&cache_dir, &info) && info.dli_fname) {
    std::string p = info.dli_fname;
    auto pos = p.rfind('/');
    if (pos != std::string::npos) return p.substr(0, pos) + "/jit_cache";
  }
  return "";
}

bool read_file(const std::string& path, std::string& out) {
  std::ifstream f(path, std::ios::binary);
  if (!f) return false;
  std::ostringstream ss;
  ss << f.rdbuf();
  out = ss.str();
  return !out.empty();
}

void write_file_atomic(const std::string& dir, const std::string& path, const std::string& data) {
  mkdir(dir.c_str(), 0755);
  // unique per process AND per call: concurrent contexts in one process (host
  // threads) may compile the same tree at the same time
  static std::atomic<unsigned long long> seq{0};
  const std::string tmp = path + ".tmp" + std::to_string(getpid()) + "." + std::to_string(seq++);
  {
    std::ofstream f(tmp, std::ios::binary);
    if (!f) return;
    f.write(data.data(), (std::streamsize)data.size());
  }
  rename(tmp.c_str(), path.c_str());
}

}  // namespace

// Compile `source` to a sm_100a cubin (host-only; no GPU needed).
std::string jit_compile(const std::string& source, std::string* log_out) {
  int maj = 0, min = 0;
  nvrtc().Version(&maj, &min);
  std::string key = source;
  for (int i = 0; i < kNumOpts; ++i) key += kOpts[i];
  key += std::to_string(maj) + "." + std::to_string(min);
  char hex[32];
  snprintf(hex, sizeof hex, "%016llx", (unsigned long long)fnv1a(key));
  const std::string dir = cache_dir();
  const std::string path = dir.empty() ? "" : dir + "/" + hex + ".cubin";
  std::string cubin;
  if (!path.empty() && read_file(path, cubin)) {
    if (log_out) {
      read_file(dir + "/" + hex + ".log", *log_out);
      while (!log_out->empty() && log_out->back() == '\0') log_out->pop_back();
    }
    return cubin;
  }
  nvrtcProgram prog;
  if (nvrtc().CreateProgram(&prog, source.c_str(), "lgp_tree.cu", 0, nullptr, nullptr) !=
      NVRTC_SUCCESS)
    throw Error(LGP_E_COMPILE, "nvrtcCreateProgram failed");
  nvrtcResult rc = nvrtc().CompileProgram(prog, kNumOpts, kOpts);
  size_t logn = 0;
  nvrtc().GetProgramLogSize(prog, &logn);
  std::string log(logn, '\0');
  if (logn) nvrtc().GetProgramLog(prog, &log[0]);
  while (!log.empty() && log.back() == '\0') log.pop_back();
  if (rc != NVRTC_SUCCESS) {
    nvrtc().DestroyProgram(&prog);
    throw Error(LGP_E_COMPILE, std::string("NVRTC: ") + nvrtc().GetErrorString(rc) + "\n" + log);
  }
  size_t n = 0;
  nvrtc().GetCUBINSize(prog, &n);
  cubin.resize(n);
  nvrtc().GetCUBIN(prog, &cubin[0]);
  nvrtc().DestroyProgram(&prog);
  if (!path.empty()) {
    write_file_atomic(dir, path, cubin);
    write_file_atomic(dir, dir + "/" + hex + ".log", log);
    write_file_atomic(dir, dir + "/" + hex + ".cu", source);
  }
  if (log_out) *log_out = log;
  return cubin;
}

Module* get_module(Context* ctx, const Plan& plan) {
  auto it = ctx->modules.find(plan.key);
  if (it != ctx->modules.end()) return it->second.get();
  std::unique_ptr<Module> m(new Module);
  const std::string cubin = jit_compile(plan.source, &m->log);
  LGP_CU_CHECK(drv::ModuleLoadData(&m->mod, cubin.data()));
  m->tc = plan.tc;
  if (plan.tc) {
    LGP_CU_CHECK(drv::ModuleGetFunction(&m->prep, m->mod, "lgp_tc_prep"));
    LGP_CU_CHECK(drv::ModuleGetFunction(&m->matvec, m->mod, "lgp_matvec_tc"));
    {
      LGP_CU_CHECK(drv::ModuleGetFunction(&m->tcsym, m->mod, "lgp_matvec_tcsym"));
      if (plan.smem_tcsym > 0)
        LGP_CU_CHECK(drv::FuncSetAttribute(m->tcsym, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES,
                                           (int)plan.smem_tcsym));
    }
  } else {
    LGP_CU_CHECK(drv::ModuleGetFunction(&m->prep, m->mod, "lgp_prep"));
    LGP_CU_CHECK(drv::ModuleGetFunction(&m->matvec, m->mod, "lgp_matvec"));
    LGP_CU_CHECK(drv::ModuleGetFunction(&m->gram, m->mod, "lgp_gram"));
    LGP_CU_CHECK(drv::ModuleGetFunction(&m->diag, m->mod, "lgp_diag"));
    LGP_CU_CHECK(drv::ModuleGetFunction(&m->matvec_sym, m->mod, "lgp_matvec_sym"));
    const size_t sym_smem = plan.smem_bytes + (size_t)(plan.tune.threads / 32) * plan.tune.cc *
                                                  plan.tune.tb * 8;
    LGP_CU_CHECK(drv::FuncSetAttribute(m->matvec_sym,
                                       CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES,
                                       (int)sym_smem));
  }
  LGP_CU_CHECK(drv::FuncSetAttribute(m->matvec, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES,
                                  (int)plan.smem_bytes));
  LGP_CU_CHECK(drv::FuncGetAttribute(&m->regs, CU_FUNC_ATTRIBUTE_NUM_REGS, m->matvec));
  int nb = 0;
  LGP_CU_CHECK(drv::OccupancyMaxActiveBlocksPerMultiprocessor(&nb, m->matvec, plan.tune.threads,
                                                           plan.smem_bytes));
  if (nb < 1) throw Error(LGP_E_UNSUPPORTED, "matvec kernel does not fit on an SM");
  m->blocks_per_sm = nb;
  Module* raw = m.get();
  ctx->modules[plan.key] = std::move(m);
  return raw;
}

}  // namespace lgp
