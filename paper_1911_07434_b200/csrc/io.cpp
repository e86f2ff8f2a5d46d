// Frame I/O of the hot path's input format: FMCX binary matrices and the CSV writers.
//
// FMCX (R/include/fastmusic/io.hpp:17-21, R/src/io.cpp:66-109): little-endian "FMCX", u32 version = 1,
// u32 rows, u32 cols, then rows*cols complex64 (float32 re, float32 im) row-major. One M x N frame file
// therefore holds exactly one frame of the batched X layout (fm_batch_io.x), so the batch reader reads each
// payload straight into its slot of the (pinned) staging buffer that fm_estimate_batch_host copies from.
// Error behaviour follows the reference: open failure / bad magic / unsupported version / truncated payload
// -> FM_EIO (std::runtime_error in the facade), non-finite entries on write -> FM_EINVAL
// (ensure_finite, R/src/linalg.cpp:40-44).
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "fastmusic_b200.h"

fm_status fm_set_error(fm_status s, const std::string& msg);  // capi.cu (thread-local last error)

namespace {

constexpr char kMagic[4] = {'F', 'M', 'C', 'X'};
constexpr double kPi = 3.14159265358979323846;

struct File {
    FILE* f = nullptr;
    File(const char* path, const char* mode) : f(std::fopen(path, mode)) {}
    ~File() {
        if (f) std::fclose(f);
    }
};

// Host-side memory order is little-endian on every platform this library builds for (x86-64 / aarch64).
fm_status read_header(FILE* f, const std::string& path, uint32_t* rows, uint32_t* cols) {
    char magic[4];
    if (std::fread(magic, 1, 4, f) != 4 || std::memcmp(magic, kMagic, 4) != 0)
        return fm_set_error(FM_EIO, path + ": bad magic");
    uint32_t hdr[3] = {0, 0, 0};
    if (std::fread(hdr, 4, 3, f) != 3 || hdr[0] != 1) return fm_set_error(FM_EIO, path + ": unsupported version");
    *rows = hdr[1];
    *cols = hdr[2];
    return FM_OK;
}

fm_status write_c64(const char* path, int64_t rows, int64_t cols, const float* a) {
    if (!path || rows < 0 || cols < 0 || rows > UINT32_MAX || cols > UINT32_MAX || (rows * cols > 0 && !a))
        return fm_set_error(FM_EINVAL, "write_matrix_binary: bad arguments");
    const size_t n = static_cast<size_t>(rows) * cols * 2;
    for (size_t i = 0; i < n; ++i)
        if (!std::isfinite(a[i])) return fm_set_error(FM_EINVAL, "write_matrix_binary: non-finite entries");
    File f(path, "wb");
    if (!f.f) return fm_set_error(FM_EIO, std::string("cannot open for writing: ") + path);
    const uint32_t hdr[3] = {1u, static_cast<uint32_t>(rows), static_cast<uint32_t>(cols)};
    if (std::fwrite(kMagic, 1, 4, f.f) != 4 || std::fwrite(hdr, 4, 3, f.f) != 3 ||
        std::fwrite(a, sizeof(float), n, f.f) != n)
        return fm_set_error(FM_EIO, std::string("write failed: ") + path);
    return FM_OK;
}

fm_status read_c64(const char* path, int64_t rows, int64_t cols, float* a) {
    if (!path || rows < 0 || cols < 0 || (rows * cols > 0 && !a))
        return fm_set_error(FM_EINVAL, "read_matrix_binary: bad arguments");
    File f(path, "rb");
    if (!f.f) return fm_set_error(FM_EIO, std::string("cannot open for reading: ") + path);
    uint32_t r = 0, c = 0;
    fm_status st = read_header(f.f, path, &r, &c);
    if (st != FM_OK) return st;
    if (r != rows || c != cols)
        return fm_set_error(FM_EINVAL, std::string(path) + ": " + std::to_string(r) + "x" + std::to_string(c) +
                                           " matrix, expected " + std::to_string(rows) + "x" + std::to_string(cols));
    const size_t n = static_cast<size_t>(rows) * cols * 2;
    if (std::fread(a, sizeof(float), n, f.f) != n) return fm_set_error(FM_EIO, std::string(path) + ": truncated payload");
    return FM_OK;
}

template <typename F>
fm_status parallel_frames(int64_t frames, int32_t threads, F&& fn) {
    int nt = threads > 0 ? threads : static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
    nt = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(nt, frames)));
    std::atomic<int64_t> next{0};
    std::atomic<bool> failed{false};
    std::mutex mu;
    fm_status first = FM_OK;
    std::string msg;
    auto work = [&] {
        for (;;) {
            const int64_t i = next.fetch_add(1);
            if (i >= frames || failed.load()) return;
            const fm_status st = fn(i);
            if (st != FM_OK) {
                std::lock_guard<std::mutex> g(mu);
                if (!failed.exchange(true)) {
                    first = st;
                    msg = fm_last_error();  // thread-local: carry it to the caller's thread
                }
            }
        }
    };
    std::vector<std::thread> pool;
    for (int w = 1; w < nt; ++w) pool.emplace_back(work);
    work();
    for (auto& t : pool) t.join();
    return first == FM_OK ? FM_OK : fm_set_error(first, msg);
}

// %.17g is what std::ostream << std::setprecision(17) prints for a double (R/src/io.cpp:115,127).
void put17(std::string& s, double v) {
    char buf[40];
    std::snprintf(buf, sizeof buf, "%.17g", v);
    s += buf;
}

}  // namespace

extern "C" fm_status fm_fmcx_write(const char* path, int64_t rows, int64_t cols, const float* a) {
    return write_c64(path, rows, cols, a);
}

extern "C" fm_status fm_fmcx_read_header(const char* path, int64_t* rows, int64_t* cols) {
    if (!path || !rows || !cols) return fm_set_error(FM_EINVAL, "fm_fmcx_read_header: null argument");
    File f(path, "rb");
    if (!f.f) return fm_set_error(FM_EIO, std::string("cannot open for reading: ") + path);
    uint32_t r = 0, c = 0;
    const fm_status st = read_header(f.f, path, &r, &c);
    if (st != FM_OK) return st;
    *rows = r;
    *cols = c;
    return FM_OK;
}

extern "C" fm_status fm_fmcx_read(const char* path, int64_t rows, int64_t cols, float* a) {
    return read_c64(path, rows, cols, a);
}

extern "C" fm_status fm_z_fmcx_write(const char* path, int64_t rows, int64_t cols, const double* a) {
    // CxMat (column-major complex128) -> row-major complex64, static_cast<float> per part (io.cpp:78-85)
    if (!path || rows < 0 || cols < 0 || (rows * cols > 0 && !a))
        return fm_set_error(FM_EINVAL, "write_matrix_binary: bad arguments");
    const size_t n = static_cast<size_t>(rows) * cols;
    for (size_t i = 0; i < 2 * n; ++i)
        if (!std::isfinite(a[i])) return fm_set_error(FM_EINVAL, "write_matrix_binary: non-finite entries");
    std::vector<float> rm(2 * n);
    for (int64_t i = 0; i < rows; ++i)
        for (int64_t j = 0; j < cols; ++j) {
            const size_t s = (static_cast<size_t>(j) * rows + i) * 2, d = (static_cast<size_t>(i) * cols + j) * 2;
            rm[d] = static_cast<float>(a[s]);
            rm[d + 1] = static_cast<float>(a[s + 1]);
        }
    return write_c64(path, rows, cols, rm.data());
}

extern "C" fm_status fm_z_fmcx_read(const char* path, int64_t rows, int64_t cols, double* a) {
    std::vector<float> rm(static_cast<size_t>(rows > 0 && cols > 0 ? rows * cols * 2 : 0));
    const fm_status st = read_c64(path, rows, cols, rm.data());
    if (st != FM_OK) return st;
    for (int64_t i = 0; i < rows; ++i)
        for (int64_t j = 0; j < cols; ++j) {
            const size_t d = (static_cast<size_t>(j) * rows + i) * 2, s = (static_cast<size_t>(i) * cols + j) * 2;
            a[d] = rm[s];
            a[d + 1] = rm[s + 1];
        }
    return FM_OK;
}

extern "C" fm_status fm_fmcx_read_frames(const char* const* paths, int64_t frames, int64_t m, int64_t n, float* x,
                                         int32_t threads) {
    if (!paths || frames < 0 || m < 1 || n < 1 || (frames > 0 && !x))
        return fm_set_error(FM_EINVAL, "fm_fmcx_read_frames: bad arguments");
    const size_t per = static_cast<size_t>(m) * n * 2;
    return parallel_frames(frames, threads, [&](int64_t f) { return read_c64(paths[f], m, n, x + f * per); });
}

extern "C" fm_status fm_fmcx_write_frames(const char* const* paths, int64_t frames, int64_t m, int64_t n,
                                          const float* x, int32_t threads) {
    if (!paths || frames < 0 || m < 1 || n < 1 || (frames > 0 && !x))
        return fm_set_error(FM_EINVAL, "fm_fmcx_write_frames: bad arguments");
    const size_t per = static_cast<size_t>(m) * n * 2;
    return parallel_frames(frames, threads, [&](int64_t f) { return write_c64(paths[f], m, n, x + f * per); });
}

extern "C" fm_status fm_z_write_matrix_csv(const char* path, int64_t rows, int64_t cols, const double* a) {
    // R/src/io.cpp:111-122: "# rows=R cols=C re,im interleaved", then re,im per entry, %.17g
    if (!path || rows < 0 || cols < 0 || (rows * cols > 0 && !a))
        return fm_set_error(FM_EINVAL, "write_matrix_csv: bad arguments");
    File f(path, "w");
    if (!f.f) return fm_set_error(FM_EIO, std::string("cannot open for writing: ") + path);
    std::string s = "# rows=" + std::to_string(rows) + " cols=" + std::to_string(cols) + " re,im interleaved\n";
    for (int64_t i = 0; i < rows; ++i) {
        for (int64_t j = 0; j < cols; ++j) {
            const size_t o = (static_cast<size_t>(j) * rows + i) * 2;
            if (j > 0) s += ',';
            put17(s, a[o]);
            s += ',';
            put17(s, a[o + 1]);
        }
        s += '\n';
    }
    if (std::fwrite(s.data(), 1, s.size(), f.f) != s.size())
        return fm_set_error(FM_EIO, std::string("write failed: ") + path);
    return FM_OK;
}

extern "C" fm_status fm_write_spectrum_csv(const char* path, int64_t grid_size, double theta0, double theta1,
                                           const double* values) {
    // R/src/io.cpp:124-131: "theta_deg,value", theta_l * 180 / pi and the value, %.17g;
    // theta_l = theta0 + ((theta1 - theta0) * l) / (L - 1) (AngleGrid, R/src/spectrum.cpp:26-28)
    if (!path || grid_size < 2 || !values) return fm_set_error(FM_EINVAL, "write_spectrum_csv: bad arguments");
    File f(path, "w");
    if (!f.f) return fm_set_error(FM_EIO, std::string("cannot open for writing: ") + path);
    std::string s = "theta_deg,value\n";
    for (int64_t l = 0; l < grid_size; ++l) {
        const double th = theta0 + ((theta1 - theta0) * static_cast<double>(l)) / static_cast<double>(grid_size - 1);
        put17(s, th * 180.0 / kPi);
        s += ',';
        put17(s, values[l]);
        s += '\n';
    }
    if (std::fwrite(s.data(), 1, s.size(), f.f) != s.size())
        return fm_set_error(FM_EIO, std::string("write failed: ") + path);
    return FM_OK;
}
