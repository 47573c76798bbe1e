// File front ends of the path: the FASTA batch
// query with the CLI's TSV output, and document ingestion for builds.  Own
// implementation of the reference's reader semantics (SPEC.md "termizer",
// proj/src/termizer.cpp:32-88,139-172) and output format
// (proj/src/cli.cpp:60-82,187-221).
#include "frontend.hpp"

#include <algorithm>
#include <cctype>
#include <filesystem>
#include <fstream>
#include <sstream>

#include "build.hpp"
#include "index.hpp"

namespace cobsg {

namespace fs = std::filesystem;

std::string read_file_bytes(const std::string& path) { // termizer.cpp:32-39
    std::ifstream in(path, std::ios::binary);
    if (!in) throw DataError("cannot open input file: " + path);
    std::ostringstream buf;
    buf << in.rdbuf();
    if (in.bad()) throw DataError("error reading input file: " + path);
    return std::move(buf).str();
}

namespace {

bool fasta_extension(const fs::path& path) { // termizer.cpp:41-46
    std::string ext = path.extension().string();
    std::transform(ext.begin(), ext.end(), ext.begin(),
                   [](unsigned char c) { return static_cast<char>(std::tolower(c)); });
    return ext == ".fa" || ext == ".fasta" || ext == ".fna";
}

} // namespace

std::vector<FastaRecord> parse_fasta(const std::string& text) { // termizer.cpp:48-88
    std::vector<FastaRecord> records;
    bool open = false;
    size_t pos = 0;
    while (pos <= text.size()) {
        size_t nl = text.find('\n', pos);
        std::string_view line;
        if (nl == std::string::npos) {
            if (pos >= text.size()) break;
            line = std::string_view(text).substr(pos);
            pos = text.size() + 1;
        } else {
            line = std::string_view(text).substr(pos, nl - pos);
            if (!line.empty() && line.back() == '\r') line.remove_suffix(1); // \r\n
            pos = nl + 1;
        }
        if (!line.empty() && line.front() == '>') {
            records.push_back({std::string(line.substr(1)), std::string()});
            open = true;
        } else if (line.empty()) {
            continue;
        } else {
            if (!open) { // a headerless leading sequence still forms a record
                records.push_back({std::string(), std::string()});
                open = true;
            }
            std::string& seq = records.back().seq;
            for (char c : line) seq.push_back(static_cast<char>(std::toupper(static_cast<unsigned char>(c))));
        }
    }
    return records;
}

std::vector<FastaRecord> read_fasta_named(const std::string& path) { // termizer.cpp:150-162
    std::vector<FastaRecord> records = parse_fasta(read_file_bytes(path));
    size_t n = 0;
    for (FastaRecord& r : records) {
        size_t space = r.name.find_first_of(" \t");
        if (space != std::string::npos) r.name.resize(space);
        if (r.name.empty()) r.name = "query_" + std::to_string(n);
        ++n;
    }
    return records;
}

std::vector<std::string> read_input(const std::string& path, int format) { // termizer.cpp:139-148
    if (format == kFormatAuto) format = fasta_extension(path) ? kFormatFasta : kFormatText;
    std::string bytes = read_file_bytes(path);
    if (format == kFormatText) return {std::move(bytes)};
    std::vector<std::string> out;
    for (FastaRecord& r : parse_fasta(bytes)) out.push_back(std::move(r.seq));
    return out;
}

std::vector<std::string> expand_inputs(const std::vector<std::string>& inputs) { // cli.cpp:60-82
    std::vector<std::string> files;
    for (const std::string& input : inputs) {
        fs::path path(input);
        std::error_code ec;
        if (fs::is_directory(path, ec)) {
            std::vector<fs::path> found;
            for (const auto& entry : fs::recursive_directory_iterator(path))
                if (entry.is_regular_file()) found.push_back(entry.path());
            std::sort(found.begin(), found.end(),
                      [](const fs::path& a, const fs::path& b) { return a.string() < b.string(); });
            for (const fs::path& p : found) files.push_back(p.string());
        } else if (fs::is_regular_file(path, ec)) {
            files.push_back(path.string());
        } else {
            throw DataError("input not found: " + input);
        }
    }
    if (files.empty()) throw DataError("no input files");
    return files;
}

std::string doc_name_from_path(const std::string& path) { // termizer.cpp:164-166
    return fs::path(path).stem().string();
}

std::string query_fasta_tsv(DeviceIndex& ix, const std::string& fasta_path, double K, uint64_t top_t) {
    if (!(K > 0.0 && K <= 1.0)) throw UsageError("K must be in (0,1]"); // cli.cpp:194-195
    std::vector<FastaRecord> queries = read_fasta_named(fasta_path);
    std::string bytes;
    std::vector<uint64_t> off{0};
    for (const FastaRecord& r : queries) {
        bytes += r.seq;
        off.push_back(bytes.size());
    }
    QueryResults R;
    query_batch(ix, reinterpret_cast<const uint8_t*>(bytes.data()), off.data(), queries.size(), K, top_t,
                1u /* COBS_Q_HITS */, R);
    // output in input order (cli.cpp:205-221; print_hits :187-190)
    std::string out;
    for (uint64_t i = 0; i < queries.size(); ++i) {
        const std::string& name = queries[i].name;
        if (R.status[i]) {
            out += '*' + name + "\tERR\t" + R.message[i] + '\n';
            continue;
        }
        out += '*' + name + '\t' + std::to_string(R.hit_n[i]) + '\n';
        const std::string ell = std::to_string(R.ell[i]);
        for (uint64_t h = 0; h < R.hit_n[i]; ++h) {
            const uint32_t d = R.doc[R.hit_off[i] + h];
            out += ix.meta.docs[d].name + '\t' + std::to_string(R.score[R.hit_off[i] + h]) + '\t' + ell + '\n';
        }
    }
    return out;
}

std::vector<uint8_t> build_from_files(const std::vector<std::string>& inputs, const Params& params,
                                      uint8_t kind, int format, int device) {
    params.validate(); // cmd_build: cli.cpp:113
    std::vector<std::string> files = expand_inputs(inputs);
    std::string seqs;
    std::vector<uint64_t> seg_off{0}, doc_segs{0};
    std::vector<std::string> names;
    for (const std::string& f : files) { // load_document: termizer.cpp:168-172
        for (std::string& s : read_input(f, format)) {
            seqs += s;
            seg_off.push_back(seqs.size());
        }
        doc_segs.push_back(seg_off.size() - 1);
        names.push_back(doc_name_from_path(f));
    }
    return build_index(reinterpret_cast<const uint8_t*>(seqs.data()), seg_off.data(), seg_off.size() - 1,
                       doc_segs.data(), names, params, kind, 0, device);
}

} // namespace cobsg
