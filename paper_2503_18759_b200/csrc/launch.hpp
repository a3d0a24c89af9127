// Host-side launch helper: programmatic dependent launch on one stream.
#pragma once

#include <cuda_runtime.h>

#include <cstdlib>

namespace cpdb {

// kernel<<<grid, block, smem, s>>>(args...) with programmatic stream
// serialisation, so its launch overlaps the previous kernel's tail (the
// kernel must begin with pdl_entry(), device.cuh).
inline bool pdl_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("CPDB_NO_PDL");
        return !(e && e[0] == '1');
    }();
    return on;
}

template <class... K, class... A>
cudaError_t launch_pdl(void (*kern)(K...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       A&&... args) {
    cudaLaunchConfig_t c{};
    c.gridDim = grid;
    c.blockDim = block;
    c.dynamicSmemBytes = smem;
    c.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    c.attrs = attr;
    c.numAttrs = pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelEx(&c, kern, static_cast<K>(args)...);
}

}  // namespace cpdb
