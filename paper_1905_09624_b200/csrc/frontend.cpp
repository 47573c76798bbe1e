// File front ends of the path: the FASTA batch
// query with the CLI's TSV output, and document ingestion for builds.
//
// Files are read once, in 1 MiB chunks, through a byte-level record scanner
// that writes sequence bytes straight to where the device path wants them
// -- a pinned host buffer sized by the file (the query batch's H2D source)
// or the build's packed corpus -- with one offset per record; no per-record
// strings, no second copy of the file.  The scanner keeps the reference
// reader's observable semantics (termizer.cpp:48-88,139-172, cli.cpp:60-82):
//   * lines end at '\n'; a '\r' right before a '\n' is not part of the line
//     (a final line with no '\n' keeps a trailing '\r');
//   * empty lines are ignored; a line starting with '>' opens a record named
//     by the rest of the line; any other line is sequence, uppercased (a-z)
//     and appended to the open record -- one with an empty name is opened if
//     sequence comes before any header;
//   * query names are cut at the first ' ' or '\t', empty ones become
//     "query_<record index>" (termizer.cpp:150-162);
//   * text-format documents are the file's raw bytes as one string.
#include "frontend.hpp"

#include <algorithm>
#include <cerrno>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <sys/stat.h>

#include <cuda_runtime.h>

#include "build.hpp"
#include "dev.cuh"
#include "index.hpp"

namespace cobsg {

namespace fs = std::filesystem;

namespace {

constexpr size_t kChunk = 1u << 20;

// Reads a file in chunks; f(bytes, n) per chunk.  DataError on open/read
// failure with the reference reader's messages (termizer.cpp:32-39).
template <typename F>
void for_each_chunk(const std::string& path, F&& f) {
    std::FILE* fp = std::fopen(path.c_str(), "rb");
    if (!fp) throw DataError("cannot open input file: " + path);
    std::vector<uint8_t> buf(kChunk);
    for (;;) {
        const size_t n = std::fread(buf.data(), 1, buf.size(), fp);
        if (n) f(buf.data(), n);
        if (n < buf.size()) {
            const bool bad = std::ferror(fp) != 0;
            std::fclose(fp);
            if (bad) throw DataError("error reading input file: " + path);
            return;
        }
    }
}

uint64_t file_size(const std::string& path) {
    struct stat st;
    if (::stat(path.c_str(), &st) != 0) throw DataError("cannot open input file: " + path);
    return static_cast<uint64_t>(st.st_size);
}

inline uint8_t upper(uint8_t c) { return (c >= 'a' && c <= 'z') ? static_cast<uint8_t>(c - 32) : c; }

// Byte-level FASTA record scanner.  Sink must provide
//   void open(std::string&& name)          a record starts (header text, or "")
//   void put(const uint8_t* p, size_t n)   uppercased sequence bytes of it
class FastaScanner {
  public:
    template <typename Sink>
    void feed(const uint8_t* p, size_t n, Sink& sink) {
        size_t i = 0;
        while (i < n) {
            const uint8_t c = p[i];
            if (cr_) { // a '\r' waiting to learn whether it ends the line
                cr_ = false;
                if (c == '\n') {
                    end_line(sink);
                    ++i;
                    continue;
                }
                content(static_cast<uint8_t>('\r'), sink);
            }
            if (c == '\n') {
                end_line(sink);
                ++i;
            } else if (c == '\r') {
                cr_ = true;
                ++i;
            } else if (state_ == kSeq) { // a run of sequence bytes up to the next line break
                size_t j = i;
                while (j < n && p[j] != '\n' && p[j] != '\r') ++j;
                put_upper(p + i, j - i, sink);
                i = j;
            } else {
                content(c, sink);
                ++i;
            }
        }
    }
    template <typename Sink>
    void finish(Sink& sink) {
        if (cr_) content(static_cast<uint8_t>('\r'), sink); // last line had no '\n': keeps its '\r'
        cr_ = false;
        end_line(sink);
    }

  private:
    enum State { kLineStart, kHeader, kSeq };
    State state_ = kLineStart;
    bool open_ = false, cr_ = false;
    std::string name_;
    uint8_t up_[256];

    template <typename Sink>
    void content(uint8_t c, Sink& sink) {
        if (state_ == kLineStart) {
            if (c == '>') {
                state_ = kHeader;
                name_.clear();
                return;
            }
            state_ = kSeq;
            if (!open_) { // sequence before any header: an unnamed record
                sink.open(std::string());
                open_ = true;
            }
        }
        if (state_ == kHeader)
            name_.push_back(static_cast<char>(c));
        else
            put_upper(&c, 1, sink);
    }
    template <typename Sink>
    void put_upper(const uint8_t* p, size_t n, Sink& sink) {
        while (n) {
            const size_t m = std::min(n, sizeof up_);
            for (size_t k = 0; k < m; ++k) up_[k] = upper(p[k]);
            sink.put(up_, m);
            p += m;
            n -= m;
        }
    }
    template <typename Sink>
    void end_line(Sink& sink) {
        if (state_ == kHeader) {
            sink.open(std::move(name_));
            name_ = std::string();
            open_ = true;
        }
        state_ = kLineStart;
    }
};

bool fasta_by_extension(const std::string& path) { // termizer.cpp:41-46
    const std::string ext = fs::path(path).extension().string();
    static const char* const kExt[] = {".fa", ".fasta", ".fna"};
    for (const char* e : kExt)
        if (ext.size() == std::strlen(e) &&
            std::equal(ext.begin(), ext.end(), e, [](char a, char b) { return std::tolower((unsigned char)a) == b; }))
            return true;
    return false;
}

// Pinned host buffer of a fixed capacity (the query batch's H2D source).
struct PinnedBytes {
    uint8_t* p = nullptr;
    uint64_t n = 0, cap = 0;
    explicit PinnedBytes(uint64_t c) : cap(c) { COBS_CUDA(cudaMallocHost(&p, std::max<uint64_t>(c, 1))); }
    ~PinnedBytes() {
        if (p) cudaFreeHost(p);
    }
    PinnedBytes(const PinnedBytes&) = delete;
    PinnedBytes& operator=(const PinnedBytes&) = delete;
};

// Query records: names (cut at a blank, "query_<i>" if empty) and packed
// sequences in a pinned buffer that can hold the whole file.
struct QuerySink {
    PinnedBytes& bytes;
    std::vector<uint64_t>& off;
    std::vector<std::string>& names;
    void open(std::string&& name) {
        if (!names.empty()) off.push_back(bytes.n);
        const size_t blank = name.find_first_of(" \t");
        if (blank != std::string::npos) name.resize(blank);
        if (name.empty()) name = "query_" + std::to_string(names.size());
        names.push_back(std::move(name));
    }
    void put(const uint8_t* p, size_t n) {
        std::memcpy(bytes.p + bytes.n, p, n);
        bytes.n += n;
    }
};

// Build documents: every record (or the whole text file) is one content
// string of the current document, appended to the packed corpus.
struct CorpusSink {
    std::string& seqs;
    std::vector<uint64_t>& seg_off;
    bool any = false;
    void open(std::string&&) {
        if (any) seg_off.push_back(seqs.size());
        any = true;
    }
    void put(const uint8_t* p, size_t n) { seqs.append(reinterpret_cast<const char*>(p), n); }
    void close() {
        if (any) seg_off.push_back(seqs.size());
    }
};

} // namespace

std::vector<std::string> expand_inputs(const std::vector<std::string>& inputs) { // cli.cpp:60-82
    std::vector<std::string> out;
    for (const std::string& in : inputs) {
        std::error_code ec;
        const fs::file_status st = fs::status(in, ec);
        if (fs::is_directory(st)) { // every regular file below, in path-string order
            std::vector<std::string> below;
            for (fs::recursive_directory_iterator it(in), end; it != end; ++it)
                if (it->is_regular_file()) below.push_back(it->path().string());
            std::sort(below.begin(), below.end());
            out.insert(out.end(), below.begin(), below.end());
            continue;
        }
        if (!fs::is_regular_file(st)) throw DataError("input not found: " + in);
        out.push_back(in);
    }
    if (out.empty()) throw DataError("no input files");
    return out;
}

std::string doc_name_from_path(const std::string& path) { return fs::path(path).stem().string(); } // termizer.cpp:164-166

std::string query_fasta_tsv(DeviceIndex& ix, const std::string& fasta_path, double K, uint64_t top_t) {
    if (!(K > 0.0 && K <= 1.0)) throw UsageError("K must be in (0,1]"); // cli.cpp:194-195
    PinnedBytes bytes(file_size(fasta_path));
    std::vector<uint64_t> off{0};
    std::vector<std::string> names;
    QuerySink sink{bytes, off, names};
    FastaScanner scan;
    uint64_t read = 0;
    for_each_chunk(fasta_path, [&](const uint8_t* p, size_t n) {
        read += n; // sequence bytes <= bytes read <= the buffer (unless the file grew meanwhile)
        if (read > bytes.cap) throw DataError("error reading input file: " + fasta_path);
        scan.feed(p, n, sink);
    });
    scan.finish(sink);
    if (!names.empty()) off.push_back(bytes.n);
    const uint64_t nq = names.size();
    QueryResults R;
    query_batch(ix, bytes.p, off.data(), nq, K, top_t, 1u /* COBS_Q_HITS */, R);
    // the CLI's batch output in input order (cli.cpp:187-190,205-221)
    std::string out;
    for (uint64_t i = 0; i < nq; ++i) {
        out.push_back('*');
        out += names[i];
        if (R.status[i]) {
            out += "\tERR\t";
            out += R.message[i];
            out.push_back('\n');
            continue;
        }
        out.push_back('\t');
        out += std::to_string(R.hit_n[i]);
        out.push_back('\n');
        const std::string tail = '\t' + std::to_string(R.ell[i]) + '\n';
        for (uint64_t h = R.hit_off[i], e = h + R.hit_n[i]; h < e; ++h) {
            out += ix.meta.docs[R.doc[h]].name;
            out.push_back('\t');
            out += std::to_string(R.score[h]);
            out += tail;
        }
    }
    return out;
}

std::vector<uint8_t> build_from_files(const std::vector<std::string>& inputs, const Params& params,
                                      uint8_t kind, int format, int device) {
    params.validate(); // cmd_build: cli.cpp:113
    const std::vector<std::string> files = expand_inputs(inputs);
    std::string seqs;
    std::vector<uint64_t> seg_off{0}, doc_segs{0};
    std::vector<std::string> names;
    for (const std::string& f : files) { // load_document: termizer.cpp:168-172
        const bool fasta = format == kFormatFasta || (format == kFormatAuto && fasta_by_extension(f));
        if (fasta) {
            CorpusSink sink{seqs, seg_off};
            FastaScanner scan;
            for_each_chunk(f, [&](const uint8_t* p, size_t n) { scan.feed(p, n, sink); });
            scan.finish(sink);
            sink.close();
        } else { // text: the raw file bytes are the document's one string
            for_each_chunk(f, [&](const uint8_t* p, size_t n) { seqs.append(reinterpret_cast<const char*>(p), n); });
            seg_off.push_back(seqs.size());
        }
        doc_segs.push_back(seg_off.size() - 1);
        names.push_back(doc_name_from_path(f));
    }
    return build_index(reinterpret_cast<const uint8_t*>(seqs.data()), seg_off.data(), seg_off.size() - 1,
                       doc_segs.data(), names, params, kind, 0, device);
}

} // namespace cobsg
