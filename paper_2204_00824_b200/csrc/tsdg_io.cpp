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

#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

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
    // diversify.cpp:286 narrows the u64 count to the u32 NodeId range silently; a
    // count past that range cannot describe a valid graph (ids are u32), so it is
    // reported instead of truncated
    const uint64_t n64 = r.le<uint64_t>();
    if (r.ok && n64 > 0xFFFFFFFFull) {
        r.err = r.path + ": node count " + std::to_string(n64) + " exceeds the 32-bit id range";
        return TSDG_ERUNTIME;
    }
    h.n = static_cast<uint32_t>(n64);
    h.metric = r.le<uint8_t>();
    h.k = r.le<uint32_t>();
    const uint32_t abits = r.le<uint32_t>();
    std::memcpy(&h.alpha, &abits, 4);
    h.lambda0 = r.le<uint16_t>();
    return r.ok ? TSDG_OK : TSDG_ERUNTIME;
}

// open + mmap without the TSDG-specific size check (an empty vector file is the
// reference's "empty dataset", not a truncation)
int open_map_any(const std::string& path, Mapped& m, std::string& err) {
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
    if (m.size == 0) return TSDG_OK;
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

uint32_t le32(const unsigned char* p) {
    return uint32_t(p[0]) | uint32_t(p[1]) << 8 | uint32_t(p[2]) << 16 | uint32_t(p[3]) << 24;
}

// fvecs / bvecs record stream (io.cpp:58-121): (int32-LE d, d components) repeated.
// Walks the records in file order and reports the first error with the reference's
// wording and byte offsets (io.cpp:27-33 truncation, :58-80 dimension checks,
// :100-106 non-finite, :110 empty).  `out` (n x d floats) may be NULL; `n_out` /
// `d_out` receive the record count and dimension.
int parse_vector_records(const std::string& path, const unsigned char* p, size_t size,
                         uint32_t comp_bytes, float* out, uint32_t* n_out, uint32_t* d_out,
                         std::string& err) {
    uint64_t off = 0;
    uint32_t d = 0;
    uint64_t index = 0;
    while (off < size) {
        const uint64_t rec_off = off;
        if (size - off < 4) {
            err = path + ": truncated file while reading record dimension at byte offset " +
                  std::to_string(off);
            return TSDG_ERUNTIME;
        }
        const int32_t rd = static_cast<int32_t>(le32(p + off));
        off += 4;
        const std::string where = " at record " + std::to_string(index) + " (byte offset " +
                                  std::to_string(rec_off) + ")";
        if (rd > (1 << 24)) {
            err = path + ": implausible dimension " + std::to_string(rd) + where;
            return TSDG_ERUNTIME;
        }
        if (rd <= 0) {
            err = path + ": invalid dimension " + std::to_string(rd) + where;
            return TSDG_ERUNTIME;
        }
        if (d != 0 && static_cast<uint32_t>(rd) != d) {
            err = path + ": inconsistent dimension at record " + std::to_string(index) +
                  " (byte offset " + std::to_string(rec_off) + "): got " + std::to_string(rd) +
                  ", expected " + std::to_string(d);
            return TSDG_ERUNTIME;
        }
        if (d == 0) d = static_cast<uint32_t>(rd);
        const uint64_t body = static_cast<uint64_t>(comp_bytes) * d;
        if (size - off < body) {
            err = path + ": truncated file while reading record components at byte offset " +
                  std::to_string(off);
            return TSDG_ERUNTIME;
        }
        for (uint32_t j = 0; j < d; ++j) {
            float v;
            if (comp_bytes == 1) {
                v = static_cast<float>(p[off + j]);
            } else {
                const uint32_t b = le32(p + off + 4ull * j);
                std::memcpy(&v, &b, 4);
            }
            if (!std::isfinite(v)) {
                err = path + ": non-finite value at record " + std::to_string(index) +
                      " component " + std::to_string(j) + " (byte offset " +
                      std::to_string(rec_off + 4 + static_cast<uint64_t>(comp_bytes) * j) + ")";
                return TSDG_ERUNTIME;
            }
            if (out) out[index * d + j] = v;
        }
        off += body;
        ++index;
    }
    if (index == 0) {
        err = path + ": empty dataset";
        return TSDG_ERUNTIME;
    }
    if (n_out) *n_out = static_cast<uint32_t>(index);
    if (d_out) *d_out = d;
    return TSDG_OK;
}

bool ends_with(const std::string& s, const char* suf) {
    const size_t k = std::strlen(suf);
    return s.size() >= k && s.compare(s.size() - k, k, suf) == 0;
}

}  // namespace

// io.cpp:112-117: .bvecs -> uint8 components, anything else -> float32.
uint32_t tsdg_vector_component_bytes(const std::string& path) { return ends_with(path, ".bvecs") ? 1 : 4; }

// Shape of a vector file from its first record and its size: records are
// fixed-size once the first dimension is known.  Returns TSDG_OK and (n, d) when
// the size is an exact multiple of the record size and the first record's
// dimension is valid; otherwise runs the full parse so the error names the first
// bad record exactly as the reference does.  Record headers past the first and
// component values are NOT checked here (the device unpack checks them).
int tsdg_vector_file_shape(const std::string& path, uint32_t* n, uint32_t* d, std::string& err) {
    Mapped m;
    if (int rc = open_map_any(path, m, err)) return rc;
    const uint32_t cb = tsdg_vector_component_bytes(path);
    if (m.size >= 4) {
        const int32_t rd = static_cast<int32_t>(le32(m.p));
        if (rd > 0 && rd <= (1 << 24)) {
            const uint64_t rec = 4 + static_cast<uint64_t>(cb) * rd;
            if (m.size % rec == 0 && m.size / rec <= 0xFFFFFFFFull) {
                *n = static_cast<uint32_t>(m.size / rec);
                *d = static_cast<uint32_t>(rd);
                return TSDG_OK;
            }
        }
    }
    return parse_vector_records(path, m.p, m.size, cb, nullptr, n, d, err);
}

// Full host parse (the error path of the device loader; also the host loader).
int tsdg_parse_vector_file(const std::string& path, float* out, uint32_t* n, uint32_t* d,
                           std::string& err) {
    Mapped m;
    if (int rc = open_map_any(path, m, err)) return rc;
    return parse_vector_records(path, m.p, m.size, tsdg_vector_component_bytes(path), out, n, d,
                                err);
}

// TSDG header from its first bytes (the streaming loader reads the body itself).
int tsdg_parse_header_bytes(const std::string& path, const unsigned char* p, size_t size,
                            tsdg_graph_header* h, uint64_t* body_off, std::string& err) {
    Reader r{path, p, size};
    if (int rc = parse_header(r, *h)) {
        err = r.err;
        return rc;
    }
    *body_off = r.off;
    return TSDG_OK;
}

// The reference-worded truncation message of the bulk reader (for a TSDG whose
// node records run past the end of the file).
std::string tsdg_truncated_message(const std::string& path, uint64_t file_size) {
    return path + ": truncated file at byte offset " + std::to_string(file_size);
}

extern "C" int tsdg_read_vectors_shape(const char* path, uint32_t* n, uint32_t* d) {
    if (!path || !n || !d) {
        tsdg_set_error("read_vectors_shape: null argument");
        return TSDG_EINVAL;
    }
    std::string err;
    const int rc = tsdg_vector_file_shape(path, n, d, err);
    if (rc) tsdg_set_error(err);
    return rc;
}

extern "C" int tsdg_read_vectors(const char* path, float* out, uint32_t n, uint32_t d) {
    if (!path || !out) {
        tsdg_set_error("read_vectors: null argument");
        return TSDG_EINVAL;
    }
    std::string err;
    uint32_t fn = 0, fd = 0;
    int rc = tsdg_vector_file_shape(path, &fn, &fd, err);
    if (!rc && (fn != n || fd != d)) {
        tsdg_set_error(std::string(path) + ": file holds " + std::to_string(fn) + " x " +
                       std::to_string(fd) + " vectors, caller expects " + std::to_string(n) +
                       " x " + std::to_string(d));
        return TSDG_EINVAL;
    }
    if (!rc) rc = tsdg_parse_vector_file(path, out, &fn, &fd, err);
    if (rc) tsdg_set_error(err);
    return rc;
}

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
