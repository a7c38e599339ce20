// Bulk TSDG loader: the reference's byte format read unchanged, in one mmap'd
// sequential pass (replaces load_tsdg's per-field stream reads,
// diversify.cpp:274-306; format diversify.hpp:122-125):
//   "TSDG" | version u32 | n u64 | metric u8 | k u32 | alpha f32 | lambda0 u16 |
//   per node: degree u32, degree x (target u32, lambda u16, dist f32), all LE.
// Error messages follow the reference's wording (serialize.hpp:65,84-85;
// diversify.cpp:276-282).
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <cstdint>
#include <cstring>
#include <string>

#include "../../include/tsdg_gpu.h"

// The error slot lives in tsdg_gpu.cu (thread-local, read by tsdg_gpu_last_error).
void tsdg_set_error(const std::string& msg);

namespace {

struct Mapped {
    const unsigned char* p = nullptr;
    size_t size = 0;
    int fd = -1;
    ~Mapped() {
        if (p && size) munmap(const_cast<unsigned char*>(p), size);
        if (fd >= 0) close(fd);
    }
};

struct Reader {
    const std::string& path;
    const unsigned char* p;
    size_t size;
    size_t off = 0;
    bool ok = true;
    std::string err;

    bool need(size_t bytes) {
        if (off + bytes > size) {
            if (ok) err = path + ": truncated file at byte offset " + std::to_string(size);
            ok = false;
            return false;
        }
        return true;
    }
    template <class T>
    T le() {
        if (!need(sizeof(T))) return T{};
        T v = 0;
        for (size_t i = 0; i < sizeof(T); ++i) v = static_cast<T>(v | (static_cast<T>(p[off + i]) << (8 * i)));
        off += sizeof(T);
        return v;
    }
};

int open_map(const std::string& path, Mapped& m, std::string& err) {
    m.fd = open(path.c_str(), O_RDONLY);
    if (m.fd < 0) {
        err = path + ": cannot open for reading";
        return TSDG_ERUNTIME;
    }
    struct stat st {};
    if (fstat(m.fd, &st) != 0) {
        err = path + ": cannot stat";
        return TSDG_ERUNTIME;
    }
    m.size = static_cast<size_t>(st.st_size);
    if (m.size == 0) {
        err = path + ": truncated file at byte offset 0";
        return TSDG_ERUNTIME;
    }
    void* p = mmap(nullptr, m.size, PROT_READ, MAP_PRIVATE, m.fd, 0);
    if (p == MAP_FAILED) {
        err = path + ": mmap failed";
        m.size = 0;
        return TSDG_ERUNTIME;
    }
    madvise(p, m.size, MADV_SEQUENTIAL);
    m.p = static_cast<const unsigned char*>(p);
    return TSDG_OK;
}

int parse_header(Reader& r, tsdg_graph_header& h) {
    if (!r.need(4)) return TSDG_ERUNTIME;
    if (std::memcmp(r.p, "TSDG", 4) != 0) {
        r.err = r.path + ": not a TSDG file";
        return TSDG_ERUNTIME;
    }
    r.off = 4;
    const uint32_t version = r.le<uint32_t>();
    if (!r.ok) return TSDG_ERUNTIME;
    if (version != 1) {
        r.err = r.path + ": unsupported TSDG version " + std::to_string(version);
        return TSDG_ERUNTIME;
    }
    h.n = static_cast<uint32_t>(r.le<uint64_t>());
    h.metric = r.le<uint8_t>();
    h.k = r.le<uint32_t>();
    const uint32_t abits = r.le<uint32_t>();
    std::memcpy(&h.alpha, &abits, 4);
    h.lambda0 = r.le<uint16_t>();
    return r.ok ? TSDG_OK : TSDG_ERUNTIME;
}

}  // namespace

extern "C" int tsdg_read_tsdg_header(const char* path_c, tsdg_graph_header* out) {
    if (!path_c || !out) {
        tsdg_set_error("read_tsdg_header: null argument");
        return TSDG_EINVAL;
    }
    const std::string path(path_c);
    Mapped m;
    std::string err;
    if (int rc = open_map(path, m, err)) {
        tsdg_set_error(err);
        return rc;
    }
    Reader r{path, m.p, m.size};
    tsdg_graph_header h{};
    if (int rc = parse_header(r, h)) {
        tsdg_set_error(r.err);
        return rc;
    }
    uint64_t edges = 0;
    uint32_t maxdeg = 0;
    for (uint64_t u = 0; u < h.n; ++u) {
        const uint32_t deg = r.le<uint32_t>();
        if (!r.ok || !r.need(static_cast<size_t>(deg) * 10)) {
            tsdg_set_error(r.err);
            return TSDG_ERUNTIME;
        }
        r.off += static_cast<size_t>(deg) * 10;
        edges += deg;
        if (deg > maxdeg) maxdeg = deg;
    }
    h.num_edges = edges;
    h.max_degree = maxdeg;
    *out = h;
    return TSDG_OK;
}

extern "C" int tsdg_read_tsdg(const char* path_c, uint64_t* offsets, uint32_t* targets,
                              uint16_t* lambdas, float* dists) {
    if (!path_c) {
        tsdg_set_error("read_tsdg: null path");
        return TSDG_EINVAL;
    }
    const std::string path(path_c);
    Mapped m;
    std::string err;
    if (int rc = open_map(path, m, err)) {
        tsdg_set_error(err);
        return rc;
    }
    Reader r{path, m.p, m.size};
    tsdg_graph_header h{};
    if (int rc = parse_header(r, h)) {
        tsdg_set_error(r.err);
        return rc;
    }
    uint64_t total = 0;
    for (uint64_t u = 0; u < h.n; ++u) {
        if (offsets) offsets[u] = total;
        const uint32_t deg = r.le<uint32_t>();
        if (!r.ok || !r.need(static_cast<size_t>(deg) * 10)) {
            tsdg_set_error(r.err);
            return TSDG_ERUNTIME;
        }
        const unsigned char* e = r.p + r.off;
        for (uint32_t j = 0; j < deg; ++j, e += 10) {
            const uint64_t t = total + j;
            if (targets) targets[t] = uint32_t(e[0]) | uint32_t(e[1]) << 8 | uint32_t(e[2]) << 16 | uint32_t(e[3]) << 24;
            if (lambdas) lambdas[t] = static_cast<uint16_t>(e[4] | e[5] << 8);
            if (dists) {
                const uint32_t b = uint32_t(e[6]) | uint32_t(e[7]) << 8 | uint32_t(e[8]) << 16 | uint32_t(e[9]) << 24;
                std::memcpy(&dists[t], &b, 4);
            }
        }
        r.off += static_cast<size_t>(deg) * 10;
        total += deg;
    }
    if (offsets) offsets[h.n] = total;
    return TSDG_OK;
}
