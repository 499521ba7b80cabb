// chunked.hpp -- the reference's chunked field container (chunked_file.hpp, src/chunked_file.cpp),
// byte-compatible, for per-rank window-slice input loading. Host code; included by ctx.cu after the
// error types (ConfigError for rects outside the grid -- the reference's std::out_of_range --,
// IoError for I/O, format and checksum failures -- IoError / IntegrityError, common.hpp:33-40).
//
// Layout (all integers little-endian u64, payload f32):
//   magic "SWCHNK01" | version=1 | channels H W | chunk_h chunk_w
//   | chunk offset table | chunk checksum table (fnv1a64 of the payload bytes)
//   | chunks in row-major chunk order, each (c, y, x) row-major over its clipped tile
// Fields are FieldTensor values: C x (H*W) column-major, i.e. [pixel][channel] in memory.
#pragma once

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <string>
#include <vector>

namespace swf {
namespace chunked {

constexpr char kMagic[8] = {'S', 'W', 'C', 'H', 'N', 'K', '0', '1'};
constexpr uint64_t kVersion = 1;

inline uint64_t fnv1a(const void* data, size_t n, uint64_t h = 0xcbf29ce484222325ULL) {
    const auto* p = static_cast<const unsigned char*>(data);
    for (size_t i = 0; i < n; ++i) {
        h ^= p[i];
        h *= 0x100000001b3ULL;
    }
    return h;
}

struct Rect {
    int y0, x0, h, w;
};

inline void put_u64(std::ofstream& out, uint64_t v) {
    unsigned char b[8];
    for (int i = 0; i < 8; ++i) b[i] = static_cast<unsigned char>((v >> (8 * i)) & 0xff);
    out.write(reinterpret_cast<const char*>(b), 8);
}
inline uint64_t get_u64(std::ifstream& in) {
    unsigned char b[8] = {0};
    in.read(reinterpret_cast<char*>(b), 8);
    uint64_t v = 0;
    for (int i = 0; i < 8; ++i) v |= uint64_t(b[i]) << (8 * i);
    return v;
}
inline int cdiv(int a, int b) { return (a + b - 1) / b; }

// write_chunked (chunked_file.cpp:44-99): field = [H*W][C]
inline void write(const std::string& path, const float* field, int C, int H, int W, int ch, int cw) {
    if (ch <= 0 || cw <= 0) throw ConfigError("chunked write: chunk dims must be positive");
    if (C <= 0 || H <= 0 || W <= 0) throw ConfigError("chunked write: empty field");
    const int ny = cdiv(H, ch), nx = cdiv(W, cw), n = ny * nx;
    std::ofstream out(path, std::ios::binary);
    if (!out) throw IoError("cannot create container: " + path);
    out.write(kMagic, 8);
    for (uint64_t v : {kVersion, uint64_t(C), uint64_t(H), uint64_t(W), uint64_t(ch), uint64_t(cw)}) put_u64(out, v);
    std::vector<uint64_t> off(n), sum(n);
    uint64_t pos = 8 + 6 * 8 + 2 * 8 * uint64_t(n);
    std::vector<std::vector<float>> bufs(n);
    for (int cy = 0; cy < ny; ++cy)
        for (int cx = 0; cx < nx; ++cx) {
            const int idx = cy * nx + cx, y0 = cy * ch, x0 = cx * cw;
            const int hh = std::min(ch, H - y0), ww = std::min(cw, W - x0);
            std::vector<float>& b = bufs[idx];
            b.resize(size_t(C) * hh * ww);
            size_t k = 0;
            for (int c = 0; c < C; ++c)
                for (int y = y0; y < y0 + hh; ++y)
                    for (int x = x0; x < x0 + ww; ++x) b[k++] = field[(size_t(y) * W + x) * C + c];
            off[idx] = pos;
            sum[idx] = fnv1a(b.data(), b.size() * 4);
            pos += b.size() * 4;
        }
    for (uint64_t v : off) put_u64(out, v);
    for (uint64_t v : sum) put_u64(out, v);
    for (const auto& b : bufs) out.write(reinterpret_cast<const char*>(b.data()), std::streamsize(b.size() * 4));
    if (!out) throw IoError("write failed: " + path);
}

// ChunkedReader (chunked_file.cpp:101-188). Not thread-safe: one reader per thread.
class Reader {
public:
    explicit Reader(const std::string& path) : path_(path), in_(path, std::ios::binary) {
        if (!in_) throw IoError("cannot open container: " + path);
        char magic[8];
        in_.read(magic, 8);
        if (!in_ || std::memcmp(magic, kMagic, 8) != 0) throw IoError("bad container magic: " + path);
        if (get_u64(in_) != kVersion) throw IoError("unsupported container version in " + path);
        C_ = int(get_u64(in_));
        H_ = int(get_u64(in_));
        W_ = int(get_u64(in_));
        ch_ = int(get_u64(in_));
        cw_ = int(get_u64(in_));
        if (!in_ || C_ <= 0 || H_ <= 0 || W_ <= 0 || ch_ <= 0 || cw_ <= 0)
            throw IoError("truncated or invalid container header: " + path);
        ny_ = cdiv(H_, ch_);
        nx_ = cdiv(W_, cw_);
        const int n = ny_ * nx_;
        off_.resize(n);
        sum_.resize(n);
        for (auto& v : off_) v = get_u64(in_);
        for (auto& v : sum_) v = get_u64(in_);
        if (!in_) throw IoError("truncated container header: " + path);
    }
    int channels() const { return C_; }
    int height() const { return H_; }
    int width() const { return W_; }
    int chunk_h() const { return ch_; }
    int chunk_w() const { return cw_; }
    uint64_t chunk_reads() const { return reads_; }
    void reset_chunk_reads() { reads_ = 0; }

    void check(const Rect& r) const {  // check_rect (chunked_file.cpp:124-131)
        if (r.h <= 0 || r.w <= 0 || r.y0 < 0 || r.x0 < 0 || r.y0 + r.h > H_ || r.x0 + r.w > W_)
            throw ConfigError("window rect [" + std::to_string(r.y0) + "," + std::to_string(r.x0) + " " +
                              std::to_string(r.h) + "x" + std::to_string(r.w) + "] outside " + std::to_string(H_) +
                              "x" + std::to_string(W_) + " grid");
    }
    uint64_t cover(const Rect& r) const {  // chunk_cover (chunked_file.cpp:133-138)
        check(r);
        return uint64_t((r.y0 + r.h - 1) / ch_ - r.y0 / ch_ + 1) * uint64_t((r.x0 + r.w - 1) / cw_ - r.x0 / cw_ + 1);
    }
    // read_window_slice (chunked_file.cpp:156-188): out = [h*w][C] (FieldTensor of the rect)
    void read(const Rect& r, float* out) {
        check(r);
        int cy0, cy1, cx0, cx1;
        chunk_range(r, cy0, cy1, cx0, cx1);
        for (int cy = cy0; cy <= cy1; ++cy)
            for (int cx = cx0; cx <= cx1; ++cx) read_chunk(r, cy, cx, out);
    }
    // chunk rows / columns covering a (checked) rect
    void chunk_range(const Rect& r, int& cy0, int& cy1, int& cx0, int& cx1) const {
        cy0 = r.y0 / ch_, cy1 = (r.y0 + r.h - 1) / ch_;
        cx0 = r.x0 / cw_, cx1 = (r.x0 + r.w - 1) / cw_;
    }
    // one chunk's part of read(): load + verify chunk (cy, cx), copy its intersection with r into out
    // (disjoint from every other chunk's part, so readers on separate handles may fill one out)
    void read_chunk(const Rect& r, int cy, int cx, float* out) {
        const int y0 = cy * ch_, x0 = cx * cw_;
        const int hh = std::min(ch_, H_ - y0), ww = std::min(cw_, W_ - x0);
        load(cy, cx, hh, ww);
        const int ys = std::max(r.y0, y0), ye = std::min(r.y0 + r.h, y0 + hh);
        const int xs = std::max(r.x0, x0), xe = std::min(r.x0 + r.w, x0 + ww);
        for (int c = 0; c < C_; ++c)
            for (int y = ys; y < ye; ++y) {
                const float* src = buf_.data() + (size_t(c) * hh + (y - y0)) * ww;
                float* dst = out + (size_t(y - r.y0) * r.w) * C_ + c;
                for (int x = xs; x < xe; ++x) dst[size_t(x - r.x0) * C_] = src[x - x0];
            }
    }

private:
    void load(int cy, int cx, int hh, int ww) {  // load_chunk (chunked_file.cpp:140-154)
        const int idx = cy * nx_ + cx;
        buf_.resize(size_t(C_) * hh * ww);
        in_.clear();
        in_.seekg(std::streamoff(off_[idx]));
        in_.read(reinterpret_cast<char*>(buf_.data()), std::streamsize(buf_.size() * 4));
        if (!in_) throw IoError("truncated chunk " + std::to_string(idx) + " in " + path_);
        if (fnv1a(buf_.data(), buf_.size() * 4) != sum_[idx])
            throw IoError("checksum mismatch in chunk " + std::to_string(idx) + " of " + path_);
        ++reads_;
    }

    std::string path_;
    std::ifstream in_;
    int C_ = 0, H_ = 0, W_ = 0, ch_ = 0, cw_ = 0, ny_ = 0, nx_ = 0;
    std::vector<uint64_t> off_, sum_;
    std::vector<float> buf_;
    uint64_t reads_ = 0;
};

}  // namespace chunked
}  // namespace swf
