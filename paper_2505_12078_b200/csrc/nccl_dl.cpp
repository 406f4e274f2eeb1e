// dlopen'ed NCCL (nccl_dl.hpp).
#include "nccl_dl.hpp"

#include <dlfcn.h>

#include <mutex>
#include <stdexcept>
#include <string>

namespace spock {

const NcclDl& nccl_dl() {
  static NcclDl t;
  static std::once_flag once;
  static std::string err;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      err = std::string("spock-b200: cannot load libnccl.so.2: ") + dlerror();
      return;
    }
    auto sym = [&](const char* name) {
      void* p = dlsym(h, name);
      if (!p && err.empty()) err = std::string("spock-b200: libnccl.so.2 has no ") + name;
      return p;
    };
    t.GetUniqueId = reinterpret_cast<decltype(t.GetUniqueId)>(sym("ncclGetUniqueId"));
    t.CommInitRank = reinterpret_cast<decltype(t.CommInitRank)>(sym("ncclCommInitRank"));
    t.AllGather = reinterpret_cast<decltype(t.AllGather)>(sym("ncclAllGather"));
    t.AllReduce = reinterpret_cast<decltype(t.AllReduce)>(sym("ncclAllReduce"));
    t.CommDestroy = reinterpret_cast<decltype(t.CommDestroy)>(sym("ncclCommDestroy"));
    t.GetErrorString = reinterpret_cast<decltype(t.GetErrorString)>(sym("ncclGetErrorString"));
  });
  if (!err.empty()) throw std::runtime_error(err);
  return t;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return;
  const NcclDl& d = nccl_dl();
  throw std::runtime_error(std::string("NCCL error in ") + what + ": " +
                           (d.GetErrorString ? d.GetErrorString(r) : "unknown"));
}

}  // namespace spock
