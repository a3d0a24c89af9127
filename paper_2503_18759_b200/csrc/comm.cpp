#include "comm.hpp"

#include <dlfcn.h>

#include <mutex>

namespace cpdb {

const Nccl& nccl() {
    static Nccl table;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            table.why = std::string("cannot load libnccl.so.2: ") + dlerror();
            return;
        }
        auto sym = [&](const char* name) { return dlsym(h, name); };
        table.GetUniqueId = reinterpret_cast<decltype(table.GetUniqueId)>(sym("ncclGetUniqueId"));
        table.CommInitRank = reinterpret_cast<decltype(table.CommInitRank)>(sym("ncclCommInitRank"));
        table.CommDestroy = reinterpret_cast<decltype(table.CommDestroy)>(sym("ncclCommDestroy"));
        table.AllReduce = reinterpret_cast<decltype(table.AllReduce)>(sym("ncclAllReduce"));
        table.AllGather = reinterpret_cast<decltype(table.AllGather)>(sym("ncclAllGather"));
        table.ReduceScatter =
            reinterpret_cast<decltype(table.ReduceScatter)>(sym("ncclReduceScatter"));
        table.GroupStart = reinterpret_cast<decltype(table.GroupStart)>(sym("ncclGroupStart"));
        table.GroupEnd = reinterpret_cast<decltype(table.GroupEnd)>(sym("ncclGroupEnd"));
        table.GetErrorString =
            reinterpret_cast<decltype(table.GetErrorString)>(sym("ncclGetErrorString"));
        table.ok = table.GetUniqueId && table.CommInitRank && table.CommDestroy &&
                   table.AllReduce && table.AllGather && table.ReduceScatter &&
                   table.GroupStart && table.GroupEnd && table.GetErrorString;
        if (!table.ok) table.why = "libnccl.so.2 lacks a required symbol";
    });
    return table;
}

}  // namespace cpdb
