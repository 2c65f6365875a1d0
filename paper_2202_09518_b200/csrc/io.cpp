// Matrix file formats of the reference's module boundary (include/oocnmf/io.hpp:28-66):
// the PDN1 binary container (header "PDNMF\0v1", u8 kind, u8 dtype, u64 rows, u64 cols, then a
// row-major dense payload or u64 nnz + u64 row_ptr + u64 col_idx + values) and Matrix Market
// (array / coordinate, real, general). Host code only — the GPU path consumes what these
// readers return.
//
// B200 extension: dtype 1 stores the values as f32 (the byte the reference reserves,
// src/io.cpp:78). The MU path computes in f32, so an f32 file halves the bytes read per
// window and lands directly in the f32 staging buffers (oocnmf_pdn1_read_dense_f32).
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <numeric>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "oocnmf_b200.h"

namespace ooc {
void set_last_error(const std::string& msg);
}

namespace {

constexpr char kPdnMagic[8] = {'P', 'D', 'N', 'M', 'F', '\0', 'v', '1'};

struct IoFail {
    int code;
    std::string msg;
};
[[noreturn]] void io_fail(const std::string& msg) { throw IoFail{OOCNMF_ERR_IO, msg}; }
[[noreturn]] void shape_fail(const std::string& msg) { throw IoFail{OOCNMF_ERR_SHAPE, msg}; }

template <class F>
int io_guard(F&& f) {
    try {
        f();
        return OOCNMF_OK;
    } catch (const IoFail& e) {
        ooc::set_last_error(e.msg);
        return e.code;
    } catch (const std::bad_alloc&) {
        ooc::set_last_error("host allocation failed");
        return OOCNMF_ERR_DEVICE;
    } catch (const std::exception& e) {
        ooc::set_last_error(e.what());
        return OOCNMF_ERR_IO;
    }
}

// ------------------------------------------------------------------------- PDN1
struct Pdn1 {
    std::ifstream in;
    std::string path;
    uint8_t kind = 0, dtype = 0;
    uint64_t rows = 0, cols = 0, nnz = 0;
    std::streamoff data = 0;  // dense payload, or the CSR row_ptr array

    size_t vbytes() const { return dtype == 1 ? 4 : 8; }

    explicit Pdn1(const std::string& p) : in(p, std::ios::binary), path(p) {
        if (!in) io_fail("cannot open: " + p);
        char magic[8];
        uint8_t kd[2];
        uint64_t rc[2];
        in.read(magic, 8);
        in.read(reinterpret_cast<char*>(kd), 2);
        in.read(reinterpret_cast<char*>(rc), 16);
        if (!in || std::memcmp(magic, kPdnMagic, 8) != 0) io_fail("bad PDN1 magic in " + p);
        kind = kd[0], dtype = kd[1], rows = rc[0], cols = rc[1];
        if (kind > 1) io_fail("unknown PDN1 kind " + std::to_string(kind) + " in " + p);
        if (dtype > 1) io_fail("unknown PDN1 dtype " + std::to_string(dtype) + " in " + p);
        if (kind == 1) {
            in.read(reinterpret_cast<char*>(&nnz), 8);
            if (!in) io_fail("PDN1: truncated read");
        }
        data = in.tellg();
    }

    void read_at(std::streamoff off, void* dst, size_t bytes) {
        in.seekg(off);
        in.read(static_cast<char*>(dst), std::streamsize(bytes));
        if (!in) io_fail("PDN1: truncated read");
    }
    // values [p0, p0 + count) of the stored value array (dense: flat index), widened / narrowed
    template <class T>
    void read_values(std::streamoff base, uint64_t p0, uint64_t count, T* out) {
        if (dtype == 1) {
            std::vector<float> tmp(count);
            read_at(base + std::streamoff(4 * p0), tmp.data(), 4 * count);
            for (uint64_t i = 0; i < count; ++i) out[i] = T(tmp[i]);
        } else {
            std::vector<double> tmp(count);
            read_at(base + std::streamoff(8 * p0), tmp.data(), 8 * count);
            for (uint64_t i = 0; i < count; ++i) out[i] = T(tmp[i]);
        }
    }
    template <class T>
    void dense_window(uint64_t r0, uint64_t r1, uint64_t c0, uint64_t c1, T* out) {
        if (kind != 0) io_fail("dense window read on CSR file " + path);
        if (r1 > rows || c1 > cols || r0 > r1 || c0 > c1) shape_fail("PDN1 window out of bounds");
        const uint64_t w = c1 - c0;
        if (c0 == 0 && c1 == cols) {  // contiguous rows: one read
            read_values(data, r0 * cols, (r1 - r0) * cols, out);
            return;
        }
        for (uint64_t i = r0; i < r1; ++i) read_values(data, i * cols + c0, w, out + (i - r0) * w);
    }
    std::streamoff col_off() const { return data + std::streamoff(8 * (rows + 1)); }
    std::streamoff val_off() const { return col_off() + std::streamoff(8 * nnz); }
    void row_bounds(uint64_t r0, uint64_t r1, uint64_t* p0, uint64_t* p1) {
        if (kind != 1) io_fail("CSR row read on dense file " + path);
        if (r1 > rows || r0 > r1) shape_fail("PDN1 row range out of bounds");
        read_at(data + std::streamoff(8 * r0), p0, 8);
        read_at(data + std::streamoff(8 * r1), p1, 8);
    }
};

void write_header(std::ofstream& out, uint8_t kind, uint8_t dtype, uint64_t rows, uint64_t cols) {
    out.write(kPdnMagic, 8);
    const uint8_t kd[2] = {kind, dtype};
    const uint64_t rc[2] = {rows, cols};
    out.write(reinterpret_cast<const char*>(kd), 2);
    out.write(reinterpret_cast<const char*>(rc), 16);
}

std::ofstream open_out(const char* path) {
    std::ofstream out(path, std::ios::binary | std::ios::trunc);
    if (!out) io_fail(std::string("cannot open for writing: ") + path);
    return out;
}

template <class T>
void write_values(std::ofstream& out, const T* v, uint64_t count, int dtype) {
    const uint64_t chunk = 1 << 20;
    if (dtype == 1) {
        std::vector<float> tmp;
        for (uint64_t p = 0; p < count; p += chunk) {
            const uint64_t n = std::min(chunk, count - p);
            tmp.assign(v + p, v + p + n);
            out.write(reinterpret_cast<const char*>(tmp.data()), std::streamsize(4 * n));
        }
    } else {
        std::vector<double> tmp;
        for (uint64_t p = 0; p < count; p += chunk) {
            const uint64_t n = std::min(chunk, count - p);
            tmp.assign(v + p, v + p + n);
            out.write(reinterpret_cast<const char*>(tmp.data()), std::streamsize(8 * n));
        }
    }
}

// ------------------------------------------------------------------------- Matrix Market
struct Mtx {
    bool dense = true;
    uint64_t rows = 0, cols = 0;
    std::vector<double> a;  // dense, row-major
    std::vector<uint64_t> rp, ci;
    std::vector<double> v;
};

Mtx read_mtx(const char* path) {
    std::ifstream in(path);
    if (!in) io_fail(std::string("cannot open: ") + path);
    std::string header, line;
    if (!std::getline(in, header) || header.rfind("%%MatrixMarket", 0) != 0)
        io_fail(std::string("not a Matrix Market file: ") + path);
    std::istringstream hs(header);
    std::string banner, object, format, field, symmetry;
    hs >> banner >> object >> format >> field >> symmetry;
    if (object != "matrix" || (field != "real" && field != "integer") || symmetry != "general")
        io_fail(std::string("unsupported Matrix Market flavor in ") + path + ": " + header);
    do {
        if (!std::getline(in, line)) io_fail(std::string("truncated Matrix Market file: ") + path);
    } while (!line.empty() && line[0] == '%');
    std::istringstream sizes(line);
    Mtx m;
    if (format == "array") {
        sizes >> m.rows >> m.cols;
        if (!sizes) io_fail(std::string("bad array size line in ") + path);
        m.a.assign(m.rows * m.cols, 0.0);
        for (uint64_t j = 0; j < m.cols; ++j)  // column-major payload
            for (uint64_t i = 0; i < m.rows; ++i)
                if (!(in >> m.a[i * m.cols + j])) io_fail(std::string("truncated array data in ") + path);
        return m;
    }
    if (format != "coordinate") io_fail(std::string("unsupported Matrix Market format in ") + path + ": " + format);
    uint64_t nnz = 0;
    sizes >> m.rows >> m.cols >> nnz;
    if (!sizes) io_fail(std::string("bad coordinate size line in ") + path);
    m.dense = false;
    std::vector<uint64_t> ii(nnz), jj(nnz);
    std::vector<double> vv(nnz);
    for (uint64_t e = 0; e < nnz; ++e) {
        if (!(in >> ii[e] >> jj[e] >> vv[e])) io_fail(std::string("truncated coordinate data in ") + path);
        if (ii[e] < 1 || ii[e] > m.rows || jj[e] < 1 || jj[e] > m.cols)
            io_fail(std::string("coordinate out of range in ") + path);
    }
    // CSR in (row, column) order; a repeated cell keeps its last value (file order)
    std::vector<uint64_t> ord(nnz);
    std::iota(ord.begin(), ord.end(), uint64_t(0));
    std::stable_sort(ord.begin(), ord.end(),
                     [&](uint64_t x, uint64_t y) { return ii[x] != ii[y] ? ii[x] < ii[y] : jj[x] < jj[y]; });
    m.rp.assign(m.rows + 1, 0);
    for (uint64_t q = 0; q < nnz; ++q) {
        const uint64_t e = ord[q];
        if (q + 1 < nnz && ii[ord[q + 1]] == ii[e] && jj[ord[q + 1]] == jj[e]) continue;  // a later duplicate wins
        m.ci.push_back(jj[e] - 1);
        m.v.push_back(vv[e]);
        ++m.rp[ii[e]];
    }
    for (uint64_t i = 0; i < m.rows; ++i) m.rp[i + 1] += m.rp[i];
    return m;
}

}  // namespace

extern "C" {

int oocnmf_pdn1_info(const char* path, int32_t* kind, int32_t* dtype, uint64_t* rows, uint64_t* cols,
                     uint64_t* nnz) {
    return io_guard([&] {
        Pdn1 f(path);
        *kind = f.kind, *dtype = f.dtype, *rows = f.rows, *cols = f.cols, *nnz = f.nnz;
    });
}

int oocnmf_pdn1_read_dense(const char* path, uint64_t r0, uint64_t r1, uint64_t c0, uint64_t c1, double* out) {
    return io_guard([&] {
        Pdn1 f(path);
        f.dense_window(r0, r1, c0, c1, out);
    });
}

int oocnmf_pdn1_read_dense_f32(const char* path, uint64_t r0, uint64_t r1, uint64_t c0, uint64_t c1, float* out) {
    return io_guard([&] {
        Pdn1 f(path);
        f.dense_window(r0, r1, c0, c1, out);
    });
}

int oocnmf_pdn1_csr_rows_nnz(const char* path, uint64_t r0, uint64_t r1, uint64_t* nnz) {
    return io_guard([&] {
        Pdn1 f(path);
        uint64_t p0 = 0, p1 = 0;
        f.row_bounds(r0, r1, &p0, &p1);
        *nnz = p1 - p0;
    });
}

int oocnmf_pdn1_read_csr_rows(const char* path, uint64_t r0, uint64_t r1, uint64_t* row_ptr, uint64_t* col_idx,
                              double* vals) {
    return io_guard([&] {
        Pdn1 f(path);
        uint64_t p0 = 0, p1 = 0;
        f.row_bounds(r0, r1, &p0, &p1);
        f.read_at(f.data + std::streamoff(8 * r0), row_ptr, 8 * (r1 - r0 + 1));
        for (uint64_t i = 0; i <= r1 - r0; ++i) row_ptr[i] -= p0;
        f.read_at(f.col_off() + std::streamoff(8 * p0), col_idx, 8 * (p1 - p0));
        f.read_values(f.val_off(), p0, p1 - p0, vals);
    });
}

int oocnmf_pdn1_write_dense(const char* path, const double* a, uint64_t rows, uint64_t cols, int32_t dtype) {
    return io_guard([&] {
        if (dtype < 0 || dtype > 1) shape_fail("PDN1 dtype must be 0 (f64) or 1 (f32)");
        auto out = open_out(path);
        write_header(out, 0, uint8_t(dtype), rows, cols);
        write_values(out, a, rows * cols, dtype);
        if (!out) io_fail(std::string("write failed: ") + path);
    });
}

int oocnmf_pdn1_write_dense_f32(const char* path, const float* a, uint64_t rows, uint64_t cols) {
    return io_guard([&] {
        auto out = open_out(path);
        write_header(out, 0, 1, rows, cols);
        out.write(reinterpret_cast<const char*>(a), std::streamsize(4 * rows * cols));
        if (!out) io_fail(std::string("write failed: ") + path);
    });
}

int oocnmf_pdn1_write_csr(const char* path, uint64_t rows, uint64_t cols, const uint64_t* row_ptr,
                          const uint64_t* col_idx, const double* vals, int32_t dtype) {
    return io_guard([&] {
        if (dtype < 0 || dtype > 1) shape_fail("PDN1 dtype must be 0 (f64) or 1 (f32)");
        auto out = open_out(path);
        write_header(out, 1, uint8_t(dtype), rows, cols);
        const uint64_t nnz = row_ptr[rows];
        out.write(reinterpret_cast<const char*>(&nnz), 8);
        out.write(reinterpret_cast<const char*>(row_ptr), std::streamsize(8 * (rows + 1)));
        out.write(reinterpret_cast<const char*>(col_idx), std::streamsize(8 * nnz));
        write_values(out, vals, nnz, dtype);
        if (!out) io_fail(std::string("write failed: ") + path);
    });
}

int oocnmf_mtx_info(const char* path, int32_t* kind, uint64_t* rows, uint64_t* cols, uint64_t* nnz) {
    return io_guard([&] {
        const Mtx m = read_mtx(path);
        *kind = m.dense ? 0 : 1, *rows = m.rows, *cols = m.cols, *nnz = m.dense ? 0 : m.v.size();
    });
}

int oocnmf_mtx_read(const char* path, double* dense_out, uint64_t* row_ptr, uint64_t* col_idx, double* vals) {
    return io_guard([&] {
        const Mtx m = read_mtx(path);
        if (m.dense) {
            if (!dense_out) shape_fail("mtx_read: dense file needs dense_out");
            std::copy(m.a.begin(), m.a.end(), dense_out);
        } else {
            if (!row_ptr || !col_idx || !vals) shape_fail("mtx_read: coordinate file needs CSR outputs");
            std::copy(m.rp.begin(), m.rp.end(), row_ptr);
            std::copy(m.ci.begin(), m.ci.end(), col_idx);
            std::copy(m.v.begin(), m.v.end(), vals);
        }
    });
}

int oocnmf_mtx_write_dense(const char* path, const double* a, uint64_t rows, uint64_t cols) {
    return io_guard([&] {
        FILE* f = std::fopen(path, "w");
        if (!f) io_fail(std::string("cannot open for writing: ") + path);
        std::fprintf(f, "%%%%MatrixMarket matrix array real general\n%llu %llu\n", (unsigned long long)rows,
                     (unsigned long long)cols);
        for (uint64_t j = 0; j < cols; ++j)
            for (uint64_t i = 0; i < rows; ++i) std::fprintf(f, "%.17g\n", a[i * cols + j]);
        if (std::fclose(f) != 0) io_fail(std::string("write failed: ") + path);
    });
}

int oocnmf_mtx_write_csr(const char* path, uint64_t rows, uint64_t cols, const uint64_t* row_ptr,
                         const uint64_t* col_idx, const double* vals) {
    return io_guard([&] {
        FILE* f = std::fopen(path, "w");
        if (!f) io_fail(std::string("cannot open for writing: ") + path);
        std::fprintf(f, "%%%%MatrixMarket matrix coordinate real general\n%llu %llu %llu\n",
                     (unsigned long long)rows, (unsigned long long)cols, (unsigned long long)row_ptr[rows]);
        for (uint64_t i = 0; i < rows; ++i)
            for (uint64_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p)
                std::fprintf(f, "%llu %llu %.17g\n", (unsigned long long)(i + 1),
                             (unsigned long long)(col_idx[p] + 1), vals[p]);
        if (std::fclose(f) != 0) io_fail(std::string("write failed: ") + path);
    });
}

}  // extern "C"
