// .cpdt tensor files straight to / from HBM.  See cpdt.hpp.
#include "cpdt.hpp"

#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cerrno>
#include <cstring>

#include "cpdb.h"
#include "runtime.hpp"

namespace cpdb {
namespace {

constexpr uint64_t kChunk = 64ull << 20;  // bytes per staging buffer

struct Fd {
    int fd = -1;
    ~Fd() {
        if (fd >= 0) ::close(fd);
    }
};

void read_exact(int fd, void* dst, uint64_t bytes, uint64_t offset, const std::string& path) {
    auto* p = static_cast<unsigned char*>(dst);
    while (bytes > 0) {
        const ssize_t r = ::pread(fd, p, bytes, off_t(offset));
        if (r < 0) fail(CPDB_FILE_ERROR, "read failure on " + path);
        if (r == 0) fail(CPDB_FORMAT_ERROR, "truncated payload");
        p += r;
        bytes -= uint64_t(r);
        offset += uint64_t(r);
    }
}

void write_all(int fd, const void* src, uint64_t bytes, const std::string& path) {
    auto* p = static_cast<const unsigned char*>(src);
    while (bytes > 0) {
        const ssize_t r = ::write(fd, p, bytes);
        if (r <= 0) fail(CPDB_FILE_ERROR, "write failure on " + path);
        p += r;
        bytes -= uint64_t(r);
    }
}

// pinned staging pair + events, released on scope exit
struct Staging {
    void* buf[2] = {nullptr, nullptr};
    cudaEvent_t done[2] = {nullptr, nullptr};
    explicit Staging(uint64_t bytes) {
        for (int i = 0; i < 2; ++i) {
            CPDB_CK(cudaMallocHost(&buf[i], bytes));
            CPDB_CK(cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming));
        }
    }
    ~Staging() {
        for (int i = 0; i < 2; ++i) {
            if (done[i]) {
                cudaEventSynchronize(done[i]);
                cudaEventDestroy(done[i]);
            }
            if (buf[i]) cudaFreeHost(buf[i]);
        }
    }
};

}  // namespace

CpdtHeader read_cpdt_header(const std::string& path) {
    Fd f;
    f.fd = ::open(path.c_str(), O_RDONLY);
    if (f.fd < 0) fail(CPDB_FILE_ERROR, "cannot open " + path);
    struct stat st {};
    if (::fstat(f.fd, &st) != 0) fail(CPDB_FILE_ERROR, "cannot stat " + path);
    const uint64_t size = uint64_t(st.st_size);
    unsigned char head[6];
    if (size < 6) fail(CPDB_FORMAT_ERROR, "truncated payload");
    read_exact(f.fd, head, 6, 0, path);
    if (std::memcmp(head, "CPDT", 4) != 0) fail(CPDB_FORMAT_ERROR, "bad magic, expected CPDT");
    if (head[4] != 1) fail(CPDB_FORMAT_ERROR, "unsupported tensor file version");
    const uint32_t order = head[5];
    if (order == 0) fail(CPDB_FORMAT_ERROR, "tensor file order must be >= 1");
    CpdtHeader h;
    h.payload_offset = 6 + 8ull * order;
    if (size < h.payload_offset) fail(CPDB_FORMAT_ERROR, "truncated payload");
    std::vector<unsigned char> ext(8ull * order);
    read_exact(f.fd, ext.data(), ext.size(), 6, path);
    uint64_t n = 1;
    for (uint32_t k = 0; k < order; ++k) {
        uint64_t v = 0;
        for (int i = 0; i < 8; ++i) v |= uint64_t(ext[8 * k + i]) << (8 * i);  // little endian
        if (v == 0) fail(CPDB_FORMAT_ERROR, "tensor file extent must be >= 1");
        if (n > (UINT64_MAX / 8) / v) fail(CPDB_FORMAT_ERROR, "tensor file element count overflows");
        n *= v;
        h.dims.push_back(v);
    }
    const uint64_t need = h.payload_offset + 8 * n;
    if (size < need) fail(CPDB_FORMAT_ERROR, "truncated payload");
    if (size > need) fail(CPDB_FORMAT_ERROR, "trailing bytes after tensor payload");
    return h;
}

void file_to_device(const std::string& path, uint64_t offset, uint64_t bytes, void* dst,
                    cudaStream_t s) {
    Fd f;
    f.fd = ::open(path.c_str(), O_RDONLY);
    if (f.fd < 0) fail(CPDB_FILE_ERROR, "cannot open " + path);
    ::posix_fadvise(f.fd, off_t(offset), off_t(bytes), POSIX_FADV_SEQUENTIAL);
    Staging st(std::min(kChunk, std::max<uint64_t>(bytes, 8)));
    auto* d = static_cast<unsigned char*>(dst);
    uint64_t done = 0;
    for (int k = 0; done < bytes; ++k) {
        const int i = k & 1;
        const uint64_t len = std::min(kChunk, bytes - done);
        CPDB_CK(cudaEventSynchronize(st.done[i]));  // the DMA that last used buf[i]
        read_exact(f.fd, st.buf[i], len, offset + done, path);
        CPDB_CK(cudaMemcpyAsync(d + done, st.buf[i], len, cudaMemcpyHostToDevice, s));
        CPDB_CK(cudaEventRecord(st.done[i], s));
        done += len;
    }
    CPDB_CK(cudaStreamSynchronize(s));
}

void device_to_cpdt(const std::string& path, const std::vector<uint64_t>& dims,
                    const double* src, uint64_t n, cudaStream_t s) {
    Fd f;
    f.fd = ::open(path.c_str(), O_WRONLY | O_CREAT | O_TRUNC, 0644);
    if (f.fd < 0) fail(CPDB_FILE_ERROR, "cannot open " + path + " for writing");
    std::vector<unsigned char> head = {'C', 'P', 'D', 'T', 1, (unsigned char)dims.size()};
    for (uint64_t v : dims)
        for (int i = 0; i < 8; ++i) head.push_back(static_cast<unsigned char>(v >> (8 * i)));
    write_all(f.fd, head.data(), head.size(), path);
    const uint64_t bytes = 8 * n;
    Staging st(std::min(kChunk, std::max<uint64_t>(bytes, 8)));
    const auto* p = reinterpret_cast<const unsigned char*>(src);
    // D2H of chunk k+1 overlaps the file write of chunk k
    uint64_t issued = 0, written = 0;
    uint64_t len[2] = {0, 0};
    int k = 0;
    auto issue = [&](int i) {
        len[i] = std::min(kChunk, bytes - issued);
        CPDB_CK(cudaMemcpyAsync(st.buf[i], p + issued, len[i], cudaMemcpyDeviceToHost, s));
        CPDB_CK(cudaEventRecord(st.done[i], s));
        issued += len[i];
    };
    if (bytes > 0) issue(0);
    while (written < bytes) {
        const int i = k & 1;
        if (issued < bytes) issue(i ^ 1);
        CPDB_CK(cudaEventSynchronize(st.done[i]));
        write_all(f.fd, st.buf[i], len[i], path);
        written += len[i];
        ++k;
    }
    if (::fsync(f.fd) != 0 && errno != EINVAL) fail(CPDB_FILE_ERROR, "write failure on " + path);
}

}  // namespace cpdb
