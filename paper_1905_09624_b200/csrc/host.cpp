// Host C++ core: params, sizing math, FORMAT.md reader/writer.
// See host.hpp.  Citations are to /root/reference/proj.
#include "host.hpp"

#include <algorithm>
#include <cerrno>
#include <cmath>
#include <memory>
#include <numeric>

#include <fcntl.h>
#include <unistd.h>

namespace cobsg {

void Params::validate() const { // params.hpp:26-35
    if (q < 1) throw UsageError("params: q must be >= 1");
    if (k < 1) throw UsageError("params: k must be >= 1");
    if (!(p > 0.0 && p < 1.0)) throw UsageError("params: p must be in (0,1)");
    if (block_size < 1) throw UsageError("params: block size must be >= 1");
    if (hash_scheme != 0) throw UsageError("params: unknown hash scheme");
}

namespace bloom {

// The libm calls and their order are those of bloom.cpp so the widths (and
// therefore the files) are bit-identical.  Built without -march/-ffast-math.
double fpr_approx(uint64_t w, uint32_t k, uint64_t v) { // bloom.cpp:42-48
    if (w < 1) throw UsageError("bloom: w must be >= 1");
    if (k < 1) throw UsageError("bloom: k must be >= 1");
    if (v == 0) return 0.0;
    double a = -double(k) * double(v) / double(w);
    double miss = -std::expm1(a);
    return std::exp(double(k) * std::log(miss));
}

uint64_t size_filter(uint64_t v, double p, uint32_t k) { // bloom.cpp:50-66
    if (!(p > 0.0 && p < 1.0))
        throw UsageError("bloom: p must be in (0,1), got " + std::to_string(p));
    if (k < 1) throw UsageError("bloom: k must be >= 1");
    if (v == 0) return 1;
    double root = std::pow(p, 1.0 / double(k));
    if (root >= 1.0)
        throw UsageError("bloom: p too close to 1 for sizing with k=" + std::to_string(k));
    double denom = -std::log1p(-root);
    auto w = static_cast<uint64_t>(std::ceil(double(k) * double(v) / denom));
    if (w < 1) w = 1;
    while (w > 1 && fpr_approx(w - 1, k, v) <= p) --w;
    while (fpr_approx(w, k, v) > p) ++w;
    return w;
}

uint64_t score_threshold(uint64_t ell, double K) { // bloom.cpp:120-123
    auto t = static_cast<uint64_t>(std::ceil(K * double(ell) - 1e-9));
    return std::max<uint64_t>(t, 1);
}

} // namespace bloom

namespace {
constexpr uint64_t P1 = 0x9E3779B185EBCA87ULL, P2 = 0xC2B2AE3D27D4EB4FULL,
                   P3 = 0x165667B19E3779F9ULL, P4 = 0x85EBCA77C2B2AE63ULL,
                   P5 = 0x27D4EB2F165667C5ULL;
inline uint64_t rotl(uint64_t x, int r) { return (x << r) | (x >> (64 - r)); }
inline uint64_t le64(const uint8_t* p) {
    uint64_t v;
    std::memcpy(&v, p, 8);
    return v;
}
inline uint32_t le32(const uint8_t* p) {
    uint32_t v;
    std::memcpy(&v, p, 4);
    return v;
}
inline uint64_t rnd(uint64_t acc, uint64_t lane) { return rotl(acc + lane * P2, 31) * P1; }
} // namespace

uint64_t xxh64(const void* data, size_t len, uint64_t seed) {
    const uint8_t* p = static_cast<const uint8_t*>(data);
    const uint8_t* end = p + len;
    uint64_t h;
    if (len >= 32) {
        uint64_t v1 = seed + P1 + P2, v2 = seed + P2, v3 = seed, v4 = seed - P1;
        do {
            v1 = rnd(v1, le64(p));
            v2 = rnd(v2, le64(p + 8));
            v3 = rnd(v3, le64(p + 16));
            v4 = rnd(v4, le64(p + 24));
            p += 32;
        } while (p + 32 <= end);
        h = rotl(v1, 1) + rotl(v2, 7) + rotl(v3, 12) + rotl(v4, 18);
        for (uint64_t v : {v1, v2, v3, v4}) h = (h ^ rnd(0, v)) * P1 + P4;
    } else {
        h = seed + P5;
    }
    h += len;
    for (; p + 8 <= end; p += 8) h = rotl(h ^ rnd(0, le64(p)), 27) * P1 + P4;
    if (p + 4 <= end) {
        h = rotl(h ^ (uint64_t(le32(p)) * P1), 23) * P2 + P3;
        p += 4;
    }
    for (; p < end; ++p) h = rotl(h ^ (uint64_t(*p) * P5), 11) * P1;
    h ^= h >> 33;
    h *= P2;
    h ^= h >> 29;
    h *= P3;
    h ^= h >> 32;
    return h;
}

// ---- name ranks --------------------------------------------------------

std::vector<uint32_t> IndexMeta::name_ranks() const {
    std::vector<uint32_t> order(docs.size());
    std::iota(order.begin(), order.end(), 0u);
    std::sort(order.begin(), order.end(),
              [&](uint32_t a, uint32_t b) { return docs[a].name < docs[b].name; });
    std::vector<uint32_t> rank(docs.size());
    for (uint32_t r = 0; r < order.size(); ++r) rank[order[r]] = r;
    return rank;
}

// ---- writer: storage.cpp:345-380 (head, tables, offsets) ---------------

namespace {
void put(std::vector<uint8_t>& out, uint64_t v, int bytes) { // storage.cpp:28-43
    for (int i = 0; i < bytes; ++i) out.push_back(static_cast<uint8_t>(v >> (8 * i)));
}
constexpr char kMagic[8] = {'C', 'O', 'B', 'S', 'I', 'D', 'X', '1'};
constexpr size_t kFixedHead = 52;
} // namespace

void IndexMeta::layout() {
    uint64_t base = 0, pos = kFixedHead;
    for (BlockMeta& b : blocks) {
        b.doc_base = base;
        pos += 16;
        for (uint64_t i = 0; i < b.doc_count; ++i) pos += 10 + docs[base + i].name.size();
        base += b.doc_count;
    }
    pos += 8 * blocks.size();
    payload_start = pos;
    for (BlockMeta& b : blocks) {
        b.offset = pos;
        pos += b.payload_bytes();
    }
    file_size = pos;
}

std::vector<uint8_t> IndexMeta::header_bytes() const {
    std::vector<uint8_t> h;
    h.insert(h.end(), kMagic, kMagic + 8);
    put(h, 1, 1);
    put(h, kind, 1);
    put(h, params.hash_scheme, 1);
    put(h, params.canonical ? 1 : 0, 1);
    put(h, params.q, 4);
    put(h, params.k, 4);
    uint64_t pbits;
    std::memcpy(&pbits, &params.p, 8);
    put(h, pbits, 8);
    put(h, params.block_size, 8);
    put(h, blocks.size(), 8);
    put(h, docs.size(), 8);
    uint64_t base = 0;
    for (const BlockMeta& b : blocks) {
        put(h, b.doc_count, 8);
        put(h, b.w, 8);
        for (uint64_t i = 0; i < b.doc_count; ++i) {
            const DocEntry& d = docs[base + i];
            if (d.name.size() > UINT16_MAX) // storage.cpp:368-369
                throw DataError("document name too long to store: " + d.name);
            put(h, d.name.size(), 2);
            h.insert(h.end(), d.name.begin(), d.name.end());
            put(h, d.term_count, 8);
        }
        base += b.doc_count;
    }
    uint64_t off = h.size() + 8 * blocks.size(); // storage.cpp:376-380
    for (const BlockMeta& b : blocks) {
        put(h, off, 8);
        off += b.payload_bytes();
    }
    return h;
}

// ---- reader: storage.cpp:67-280 ----------------------------------------

ByteSource file_source(const std::string& path) {
    int fd = ::open(path.c_str(), O_RDONLY);
    if (fd < 0)
        throw DataError("cannot open index file " + path + ": " + std::strerror(errno));
    off_t size = ::lseek(fd, 0, SEEK_END);
    if (size < 0) {
        ::close(fd);
        throw DataError("cannot stat index file " + path);
    }
    auto shared_fd = std::shared_ptr<int>(new int(fd), [](int* f) {
        ::close(*f);
        delete f;
    });
    ByteSource s;
    s.size = static_cast<uint64_t>(size);
    s.path = path;
    s.read_at = [shared_fd, path](uint64_t off, void* dst, uint64_t len) {
        uint8_t* p = static_cast<uint8_t*>(dst);
        while (len > 0) {
            ssize_t got = ::pread(*shared_fd, p, len, static_cast<off_t>(off));
            if (got < 0) {
                if (errno == EINTR) continue;
                throw DataError("read error in " + path + ": " + std::strerror(errno));
            }
            if (got == 0) throw DataError("unexpected end of file in " + path);
            p += got;
            off += static_cast<uint64_t>(got);
            len -= static_cast<uint64_t>(got);
        }
    };
    return s;
}

ByteSource memory_source(const uint8_t* data, uint64_t len, const std::string& path) {
    ByteSource s;
    s.size = len;
    s.path = path;
    s.read_at = [data, len, path](uint64_t off, void* dst, uint64_t n) {
        if (off > len || n > len - off) throw DataError("unexpected end of file in " + path);
        std::memcpy(dst, data + off, n);
    };
    return s;
}

namespace {

// Buffered sequential header reader (storage.cpp:112-176).
class Cursor {
public:
    explicit Cursor(const ByteSource& s) : s_(s) {}
    uint64_t pos() const { return pos_; }
    uint64_t remaining() const { return s_.size - pos_; }
    void read(void* dst, uint64_t len) {
        if (len > s_.size - pos_) throw DataError("index file " + s_.path + " is truncated");
        uint8_t* p = static_cast<uint8_t*>(dst);
        while (len > 0) {
            if (pos_ < buf_start_ || pos_ >= buf_start_ + buf_.size()) refill();
            uint64_t avail = buf_start_ + buf_.size() - pos_;
            uint64_t take = std::min(avail, len);
            std::memcpy(p, buf_.data() + (pos_ - buf_start_), take);
            p += take;
            pos_ += take;
            len -= take;
        }
    }
    uint64_t le(int n) {
        uint8_t b[8];
        read(b, n);
        uint64_t v = 0;
        for (int i = n - 1; i >= 0; --i) v = (v << 8) | b[i];
        return v;
    }

private:
    void refill() {
        uint64_t take = std::min<uint64_t>(1 << 20, s_.size - pos_);
        buf_.resize(take);
        s_.read_at(pos_, buf_.data(), take);
        buf_start_ = pos_;
    }
    const ByteSource& s_;
    uint64_t pos_ = 0, buf_start_ = 0;
    std::vector<uint8_t> buf_;
};

} // namespace

IndexMeta parse_index(const ByteSource& src) {
    auto bad = [&](const std::string& what) -> DataError {
        return DataError("index file " + src.path + ": " + what);
    };
    IndexMeta out;
    out.file_size = src.size;
    if (src.size < kFixedHead) throw bad("too small to be an index file"); // :185
    Cursor cur(src);
    char magic[8];
    cur.read(magic, 8);
    if (std::memcmp(magic, kMagic, 8) != 0) throw bad("bad magic");
    uint64_t version = cur.le(1);
    if (version != 1) throw bad("unsupported format version " + std::to_string(version));
    out.kind = static_cast<uint8_t>(cur.le(1));
    if (out.kind != kKindClassic && out.kind != kKindCompact)
        throw bad("unknown index kind " + std::to_string(out.kind));
    out.params.hash_scheme = static_cast<uint8_t>(cur.le(1));
    if (out.params.hash_scheme != 0)
        throw bad("unknown hash scheme " + std::to_string(out.params.hash_scheme));
    uint64_t canonical = cur.le(1);
    if (canonical > 1) throw bad("bad canonical flag");
    out.params.canonical = canonical != 0;
    out.params.q = static_cast<uint32_t>(cur.le(4));
    out.params.k = static_cast<uint32_t>(cur.le(4));
    uint64_t pbits = cur.le(8);
    std::memcpy(&out.params.p, &pbits, 8);
    out.params.block_size = cur.le(8);
    uint64_t num_blocks = cur.le(8);
    uint64_t num_docs = cur.le(8);
    if (out.params.q < 1 || out.params.k < 1) throw bad("bad q/k parameters"); // :209-214
    if (!(out.params.p > 0.0 && out.params.p < 1.0)) throw bad("target FPR out of range");
    if (out.params.block_size < 1) throw bad("bad block size");
    if (num_blocks < 1) throw bad("no blocks");
    if (out.kind == kKindClassic && num_blocks != 1)
        throw bad("classic index must have exactly one block");
    if (num_blocks > src.size / 17) throw bad("block count exceeds file size"); // :218

    out.blocks.resize(num_blocks);
    uint64_t seen = 0;
    for (BlockMeta& b : out.blocks) { // :222-237
        b.doc_count = cur.le(8);
        b.w = cur.le(8);
        if (b.doc_count < 1) throw bad("empty block");
        if (b.w < 1) throw bad("zero block width");
        if (b.doc_count > cur.remaining() / 10) throw bad("document table exceeds file size");
        b.doc_base = seen;
        for (uint64_t i = 0; i < b.doc_count; ++i) {
            DocEntry d;
            uint64_t len = cur.le(2);
            d.name.resize(len);
            cur.read(d.name.data(), len);
            d.term_count = cur.le(8);
            out.docs.push_back(std::move(d));
        }
        seen += b.doc_count;
    }
    if (seen != num_docs) throw bad("document count mismatch"); // :238

    for (BlockMeta& b : out.blocks) b.offset = cur.le(8); // :240-250
    out.payload_start = cur.pos();
    uint64_t expected = out.payload_start;
    for (const BlockMeta& b : out.blocks) {
        if (b.offset != expected) throw bad("payload offsets not contiguous");
        if (b.payload_bytes() > src.size - expected) throw bad("payload exceeds file size");
        expected += b.payload_bytes();
    }
    if (expected != src.size) throw bad("trailing bytes after payload");

    if (out.kind == kKindCompact) { // :253-265
        uint64_t prev_w = 0, prev_tc = 0, g = 0;
        for (const BlockMeta& b : out.blocks) {
            if (b.w < prev_w) throw bad("block widths decrease");
            prev_w = b.w;
            for (uint64_t i = 0; i < b.doc_count; ++i, ++g) {
                if (out.docs[g].term_count < prev_tc) throw bad("document term counts not sorted");
                prev_tc = out.docs[g].term_count;
            }
        }
    }

    std::vector<const std::string*> names; // :267-277
    names.reserve(out.docs.size());
    for (const DocEntry& d : out.docs) names.push_back(&d.name);
    std::sort(names.begin(), names.end(),
              [](const std::string* a, const std::string* b) { return *a < *b; });
    auto dup = std::adjacent_find(names.begin(), names.end(),
                                  [](const std::string* a, const std::string* b) { return *a == *b; });
    if (dup != names.end()) throw bad("duplicate document name " + **dup);
    return out;
}

} // namespace cobsg
