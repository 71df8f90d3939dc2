#include "nccl_shim.h"

#include <dlfcn.h>

#include <cstdlib>
#include <mutex>

#include "common.h"

namespace ss {

const NcclApi *nccl_api() {
    static NcclApi api{};
    static bool ok = false;
    static std::once_flag once;
    std::call_once(once, [] {
        void *h = nullptr;
        // already loaded by the host process (torch links libnccl.so.2)?
        h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) {
            const char *env = std::getenv("SS_NCCL_LIB");
            if (env) h = dlopen(env, RTLD_NOW);
        }
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW);
        if (!h) return;
        auto sym = [&](const char *n) { return dlsym(h, n); };
        api.getUniqueId = (decltype(api.getUniqueId))sym("ncclGetUniqueId");
        api.commInitRank = (decltype(api.commInitRank))sym("ncclCommInitRank");
        api.commDestroy = (decltype(api.commDestroy))sym("ncclCommDestroy");
        api.groupStart = (decltype(api.groupStart))sym("ncclGroupStart");
        api.groupEnd = (decltype(api.groupEnd))sym("ncclGroupEnd");
        api.send = (decltype(api.send))sym("ncclSend");
        api.recv = (decltype(api.recv))sym("ncclRecv");
        api.getErrorString = (decltype(api.getErrorString))sym("ncclGetErrorString");
        ok = api.getUniqueId && api.commInitRank && api.commDestroy && api.groupStart && api.groupEnd &&
             api.send && api.recv && api.getErrorString;
    });
    if (!ok) {
        fail(SS_ECUDA, "NCCL (libnccl.so.2) could not be loaded; set SS_NCCL_LIB");
        return nullptr;
    }
    return &api;
}

}  // namespace ss
