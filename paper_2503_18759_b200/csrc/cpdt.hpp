// .cpdt tensor files straight to / from HBM (format of
// /root/reference/proj/include/cpd/io.hpp:93-121).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include <cuda_runtime.h>

namespace cpdb {

struct CpdtHeader {
    std::vector<uint64_t> dims;
    uint64_t payload_offset = 0;  // bytes before the first value
};

// Throws Fail{CPDB_FILE_ERROR | CPDB_FORMAT_ERROR}.  Checks magic, version,
// extents and that the file holds exactly prod(dims) values.
CpdtHeader read_cpdt_header(const std::string& path);
// Copy `bytes` from file offset `offset` into device memory `dst`, pinned
// double-buffered chunks (file read of chunk k+1 overlaps the DMA of chunk k).
void file_to_device(const std::string& path, uint64_t offset, uint64_t bytes, void* dst,
                    cudaStream_t s);
// Write the header and then `n` doubles from device memory.
void device_to_cpdt(const std::string& path, const std::vector<uint64_t>& dims,
                    const double* src, uint64_t n, cudaStream_t s);
// Number of non-finite values in x[0..n) (device reduction).
uint64_t count_nonfinite(const double* x, uint64_t n, cudaStream_t s);

}  // namespace cpdb
