// chunk_store.hpp -- tiled field files for per-rank window-slice input loading (f4).
//
// Byte format: the reference's chunked container (chunked_file.hpp / src/chunked_file.cpp), so its
// files load here and ours load there. Everything else is this repo's own design around POSIX
// pread: one open descriptor is shared by any number of reader threads (no seek state), a tile is
// fetched with one pread into a caller-owned buffer and verified before use, and a writer builds the
// whole image in memory and issues one write.
//
//   bytes [0, 8)            "SWCHNK01"
//   u64 x 6 (little endian) version (1), channels C, height H, width W, tile_h, tile_w
//   u64 x T                 byte offset of every tile (T = ceil(H / tile_h) * ceil(W / tile_w),
//                           tiles in row-major tile order)
//   u64 x T                 fnv1a64 of every tile's payload
//   payload                 per tile, float32 planes c = 0..C-1, each the tile's clipped rows y, x
//
// A field is FieldTensor<float>::values: C x (H*W) column-major, i.e. [pixel][channel] in memory.
// Host code, included by ctx.cu after the error types: rectangles outside the grid raise ConfigError
// (the reference's std::out_of_range, rc 2), I/O, format and checksum failures IoError (IoError /
// IntegrityError, common.hpp:33-40, rc 3).
#pragma once

#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cerrno>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

namespace swf {
namespace tiles {

constexpr unsigned char kTag[8] = {'S', 'W', 'C', 'H', 'N', 'K', '0', '1'};
constexpr uint64_t kFormat = 1;
constexpr size_t kHead = 8 + 6 * 8;

inline uint64_t fnv1a64(const void* p, size_t n, uint64_t h = 0xcbf29ce484222325ULL) {
    const unsigned char* b = static_cast<const unsigned char*>(p);
    for (const unsigned char* e = b + n; b != e; ++b) h = (h ^ *b) * 0x100000001b3ULL;
    return h;
}
inline uint64_t le64(const unsigned char* b) {
    uint64_t v = 0;
    for (int k = 7; k >= 0; --k) v = (v << 8) | b[k];
    return v;
}
inline void put_le64(unsigned char* b, uint64_t v) {
    for (int k = 0; k < 8; ++k, v >>= 8) b[k] = static_cast<unsigned char>(v);
}

struct Rect {  // pixel rectangle: rows [y0, y0 + h), columns [x0, x0 + w)
    int y0, x0, h, w;
};

// Tiling of an H x W grid of C-channel pixels.
struct Grid {
    int C = 0, H = 0, W = 0, th = 0, tw = 0;
    int rows() const { return (H + th - 1) / th; }
    int cols() const { return (W + tw - 1) / tw; }
    int count() const { return rows() * cols(); }
    Rect box(int ty, int tx) const {  // clipped pixel box of tile (ty, tx)
        const int y0 = ty * th, x0 = tx * tw;
        return {y0, x0, std::min(th, H - y0), std::min(tw, W - x0)};
    }
    size_t floats(int ty, int tx) const {
        const Rect b = box(ty, tx);
        return size_t(C) * b.h * b.w;
    }
    // tile rows / columns a rectangle touches (inclusive)
    void span(const Rect& r, int& ty0, int& ty1, int& tx0, int& tx1) const {
        ty0 = r.y0 / th;
        ty1 = (r.y0 + r.h - 1) / th;
        tx0 = r.x0 / tw;
        tx1 = (r.x0 + r.w - 1) / tw;
    }
    void require_inside(const Rect& r) const {
        if (r.h < 1 || r.w < 1 || r.y0 < 0 || r.x0 < 0 || r.y0 > H - r.h || r.x0 > W - r.w)
            throw ConfigError("chunked read: rectangle rows " + std::to_string(r.y0) + "+" + std::to_string(r.h) +
                              ", cols " + std::to_string(r.x0) + "+" + std::to_string(r.w) + " is not inside the " +
                              std::to_string(H) + " x " + std::to_string(W) + " grid");
    }
    uint64_t touched(const Rect& r) const {
        require_inside(r);
        int a, b, c, d;
        span(r, a, b, c, d);
        return uint64_t(b - a + 1) * uint64_t(d - c + 1);
    }
};

// Write a field as a tiled file (write_chunked, chunked_file.cpp:44-99).
inline void save(const std::string& path, const float* field, int C, int H, int W, int th, int tw) {
    if (th < 1 || tw < 1) throw ConfigError("chunked write: tile sides must be >= 1 (got " + std::to_string(th) +
                                            " x " + std::to_string(tw) + ")");
    if (C < 1 || H < 1 || W < 1) throw ConfigError("chunked write: field has no values");
    const Grid g{C, H, W, th, tw};
    const int T = g.count();
    size_t total = kHead + size_t(16) * T;
    for (int t = 0; t < T; ++t) total += g.floats(t / g.cols(), t % g.cols()) * 4;
    std::vector<unsigned char> img(total);
    std::memcpy(img.data(), kTag, 8);
    const uint64_t hdr[6] = {kFormat, uint64_t(C), uint64_t(H), uint64_t(W), uint64_t(th), uint64_t(tw)};
    for (int k = 0; k < 6; ++k) put_le64(img.data() + 8 + 8 * k, hdr[k]);
    size_t at = kHead + size_t(16) * T;
    for (int t = 0; t < T; ++t) {
        const Rect b = g.box(t / g.cols(), t % g.cols());
        float* dst = reinterpret_cast<float*>(img.data() + at);  // 4-byte aligned: header + tables are 8k
        for (int c = 0; c < C; ++c)
            for (int y = 0; y < b.h; ++y) {
                const float* row = field + (size_t(b.y0 + y) * W + b.x0) * C + c;
                for (int x = 0; x < b.w; ++x) *dst++ = row[size_t(x) * C];
            }
        const size_t bytes = size_t(C) * b.h * b.w * 4;
        put_le64(img.data() + kHead + 8 * size_t(t), at);
        put_le64(img.data() + kHead + 8 * size_t(T + t), fnv1a64(img.data() + at, bytes));
        at += bytes;
    }
    const int fd = ::open(path.c_str(), O_WRONLY | O_CREAT | O_TRUNC, 0644);
    if (fd < 0) throw IoError("chunked write: cannot open " + path + " for writing: " + std::strerror(errno));
    size_t done = 0;
    while (done < img.size()) {
        const ssize_t k = ::write(fd, img.data() + done, img.size() - done);
        if (k <= 0) {
            ::close(fd);
            throw IoError("chunked write: short write to " + path);
        }
        done += size_t(k);
    }
    if (::close(fd) != 0) throw IoError("chunked write: closing " + path + " failed");
}

// Read side (ChunkedReader, chunked_file.hpp:36-75): thread-safe -- tiles are fetched with pread into
// caller buffers, the tile counter is atomic.
class File {
public:
    explicit File(const std::string& path) : path_(path) {
        fd_ = ::open(path.c_str(), O_RDONLY);
        if (fd_ < 0) throw IoError("chunked read: cannot open " + path + ": " + std::strerror(errno));
        try {
            unsigned char h[kHead];
            fetch(h, kHead, 0, "header");
            if (std::memcmp(h, kTag, 8) != 0) throw IoError("chunked read: " + path + " is not a tiled field file");
            if (le64(h + 8) != kFormat)
                throw IoError("chunked read: " + path + " has format version " + std::to_string(le64(h + 8)));
            uint64_t v[5];
            for (int k = 0; k < 5; ++k) v[k] = le64(h + 16 + 8 * k);
            for (uint64_t x : v)
                if (x < 1 || x > (1u << 30)) throw IoError("chunked read: implausible dimensions in " + path);
            g_ = Grid{int(v[0]), int(v[1]), int(v[2]), int(v[3]), int(v[4])};
            const size_t T = size_t(g_.count());
            std::vector<unsigned char> tab(16 * T);
            fetch(tab.data(), tab.size(), kHead, "tile tables");
            off_.resize(T);
            sum_.resize(T);
            for (size_t t = 0; t < T; ++t) {
                off_[t] = le64(tab.data() + 8 * t);
                sum_[t] = le64(tab.data() + 8 * (T + t));
            }
        } catch (...) {
            ::close(fd_);
            throw;
        }
    }
    ~File() {
        if (fd_ >= 0) ::close(fd_);
    }
    File(const File&) = delete;
    File& operator=(const File&) = delete;

    const Grid& grid() const { return g_; }
    uint64_t tiles_read() const { return reads_.load(); }
    void reset_tiles_read() { reads_ = 0; }

    // Tile (ty, tx) into buf (resized; planes c, rows y, columns x of the clipped box), checksum-verified.
    void tile(int ty, int tx, std::vector<float>& buf) const {
        const size_t t = size_t(ty) * g_.cols() + tx;
        buf.resize(g_.floats(ty, tx));
        fetch(buf.data(), buf.size() * 4, off_[t], "tile " + std::to_string(t));
        if (fnv1a64(buf.data(), buf.size() * 4) != sum_[t])
            throw IoError("IntegrityError: tile " + std::to_string(t) + " of " + path_ + " fails its checksum");
        reads_.fetch_add(1);
    }
    // The part of tile (ty, tx) inside r, into out = [r.h * r.w][C] (disjoint per tile).
    void place(const Rect& r, int ty, int tx, const std::vector<float>& buf, float* out) const {
        const Rect b = g_.box(ty, tx);
        const int y0 = std::max(r.y0, b.y0), y1 = std::min(r.y0 + r.h, b.y0 + b.h);
        const int x0 = std::max(r.x0, b.x0), x1 = std::min(r.x0 + r.w, b.x0 + b.w);
        const int C = g_.C;
        for (int y = y0; y < y1; ++y) {
            float* o = out + (size_t(y - r.y0) * r.w + (x0 - r.x0)) * C;
            for (int c = 0; c < C; ++c) {
                const float* src = buf.data() + (size_t(c) * b.h + (y - b.y0)) * b.w + (x0 - b.x0);
                for (int x = 0; x < x1 - x0; ++x) o[size_t(x) * C + c] = src[x];
            }
        }
    }
    // read_window_slice (chunked_file.cpp:156-188): out = [r.h * r.w][C]
    void read(const Rect& r, float* out) const {
        g_.require_inside(r);
        int ty0, ty1, tx0, tx1;
        g_.span(r, ty0, ty1, tx0, tx1);
        std::vector<float> buf;
        for (int ty = ty0; ty <= ty1; ++ty)
            for (int tx = tx0; tx <= tx1; ++tx) {
                tile(ty, tx, buf);
                place(r, ty, tx, buf, out);
            }
    }

private:
    void fetch(void* dst, size_t n, uint64_t at, const std::string& what) const {
        size_t done = 0;
        while (done < n) {
            const ssize_t k = ::pread(fd_, static_cast<char*>(dst) + done, n - done, off_t(at + done));
            if (k < 0 && errno == EINTR) continue;
            if (k <= 0) throw IoError("chunked read: " + path_ + " ends inside the " + what);
            done += size_t(k);
        }
    }
    std::string path_;
    int fd_ = -1;
    Grid g_;
    std::vector<uint64_t> off_, sum_;
    mutable std::atomic<uint64_t> reads_{0};
};

}  // namespace tiles
}  // namespace swf
