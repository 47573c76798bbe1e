// ORACLE SHIM — TEST INFRASTRUCTURE ONLY.
//
// extern "C" wrappers over the UNMODIFIED reference library (the 7 non-CLI
// sources of /root/reference/proj/src, compiled by oracle/Makefile into
// oracle/_ref/libcobs_ref.so).  Used by tests/ as the reference-itself oracle
// and by `bench.py --impl reference` as the reference's CPU path.  Nothing in
// the product links this.
//
// Reference API used: cobs::extract_terms (termizer.hpp:37), cobs::xxh64
// (xxhash64.hpp:45), cobs::bloom::{size_filter,score_threshold}
// (bloom.hpp:25,48), cobs::build_classic / build_compact
// (classic_index.hpp:37, compact_index.hpp:26), cobs::write_index /
// open_resident (storage.hpp:14-19), cobs::query (query.hpp:46) and the
// cobs::IndexView interface (index_view.hpp:18-47), which the config-5
// procedural/in-memory views below implement.
#include <algorithm>
#include <filesystem>
#include <sstream>
#include <atomic>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "cobs/bloom.hpp"
#include "cobs/classic_index.hpp"
#include "cobs/compact_index.hpp"
#include "cobs/error.hpp"
#include "cobs/index_view.hpp"
#include "cobs/query.hpp"
#include "cobs/storage.hpp"
#include "cobs/termizer.hpp"
#include "cobs/xxhash64.hpp"

#include "../paper_1905_09624_b200/csrc/synth.h"

namespace {

void set_err(char* err, size_t errlen, const char* msg) {
    if (err && errlen) std::snprintf(err, errlen, "%s", msg);
}

// Map exceptions to the CLI's codes (proj/src/cli.cpp:448-454).
template <typename F>
int guarded(char* err, size_t errlen, F&& f) {
    try {
        f();
        return 0;
    } catch (const cobs::DataError& e) {
        set_err(err, errlen, e.what());
        return 2;
    } catch (const std::invalid_argument& e) {
        set_err(err, errlen, e.what());
        return 1;
    } catch (const std::exception& e) {
        set_err(err, errlen, e.what());
        return 3;
    }
}

// Config-5 index: header from synth.h + reference sizing, rows either
// regenerated per call (procedural) or materialised once in host RAM.
class C5View final : public cobs::IndexView {
public:
    C5View(uint64_t seed, uint64_t n, uint64_t B, double median, double sigma, double p,
           bool materialise, int threads)
        : seed_(seed) {
        params_.q = 31;
        params_.k = 1;
        params_.p = p;
        params_.canonical = false;
        params_.block_size = B;
        std::vector<uint64_t> tc(n);
        syn_c5_term_counts(seed, n, median, sigma, tc.data());
        std::vector<std::pair<uint64_t, std::string>> docs(n);
        for (uint64_t i = 0; i < n; ++i) {
            char nm[24];
            int l = syn_c5_name(i, nm);
            docs[i] = {tc[i], std::string(nm, size_t(l))};
        }
        std::sort(docs.begin(), docs.end()); // (term_count, name): compact_index.cpp:27-30
        uint64_t nb = (n + B - 1) / B;
        blocks_.resize(nb);
        for (uint64_t b = 0; b < nb; ++b) {
            uint64_t lo = b * B, hi = std::min(n, lo + B), mx = 0;
            for (uint64_t i = lo; i < hi; ++i) {
                blocks_[b].docs.push_back({docs[i].second, docs[i].first});
                mx = std::max(mx, docs[i].first);
            }
            blocks_[b].w = cobs::bloom::size_filter(mx, p, 1); // classic_index.cpp:61
            blocks_[b].thr = syn_c5_thr16(blocks_[b].w, mx);
        }
        if (materialise) {
            uint64_t total = 0;
            for (auto& blk : blocks_) {
                blk.off = total;
                total += blk.w * ((blk.docs.size() + 7) / 8);
            }
            payload_.reset(new uint8_t[total]);
            std::atomic<uint64_t> next{0};
            auto work = [&] {
                for (;;) {
                    uint64_t t = next.fetch_add(1);
                    // task = (block, chunk of 65536 rows)
                    uint64_t acc = 0, b = 0;
                    for (; b < blocks_.size(); ++b) {
                        uint64_t chunks = (blocks_[b].w + 65535) / 65536;
                        if (t < acc + chunks) break;
                        acc += chunks;
                    }
                    if (b >= blocks_.size()) return;
                    const Block& blk = blocks_[b];
                    uint64_t rb = (blk.docs.size() + 7) / 8;
                    uint64_t r0 = (t - acc) * 65536, r1 = std::min(blk.w, r0 + 65536);
                    for (uint64_t r = r0; r < r1; ++r)
                        for (uint64_t j = 0; j < rb; ++j)
                            payload_[blk.off + r * rb + j] =
                                syn_c5_byte(seed_, b, r, j, blk.thr, blk.docs.size());
                }
            };
            std::vector<std::thread> th;
            for (int i = 0; i < std::max(1, threads); ++i) th.emplace_back(work);
            for (auto& x : th) x.join();
        }
    }

    const cobs::IndexParams& params() const override { return params_; }
    uint8_t kind() const override { return cobs::kKindCompact; }
    size_t block_count() const override { return blocks_.size(); }
    uint64_t doc_count(size_t b) const override { return blocks_[b].docs.size(); }
    uint64_t width(size_t b) const override { return blocks_[b].w; }
    const cobs::DocEntry& doc(size_t b, uint64_t i) const override { return blocks_[b].docs[i]; }
    const uint8_t* row_data(size_t b, uint64_t r, size_t lo, size_t hi,
                            uint8_t* scratch) const override {
        const Block& blk = blocks_[b];
        if (payload_) return payload_.get() + blk.off + r * row_bytes(b) + lo;
        for (size_t j = lo; j < hi; ++j)
            scratch[j - lo] = syn_c5_byte(seed_, b, r, j, blk.thr, blk.docs.size());
        return scratch;
    }

private:
    struct Block {
        std::vector<cobs::DocEntry> docs;
        uint64_t w = 0, off = 0;
        uint32_t thr = 0;
    };
    uint64_t seed_;
    cobs::IndexParams params_;
    std::vector<Block> blocks_;
    std::unique_ptr<uint8_t[]> payload_;
};

struct Handle {
    std::unique_ptr<cobs::IndexView> view;
    std::unordered_map<std::string, uint64_t> global; // name -> global column
};

void index_names(Handle* h) {
    uint64_t g = 0;
    for (size_t b = 0; b < h->view->block_count(); ++b)
        for (uint64_t i = 0; i < h->view->doc_count(b); ++i) h->global[h->view->doc(b, i).name] = g++;
}

} // namespace

extern "C" {

uint64_t ref_xxh64(const void* data, size_t len, uint64_t seed) {
    return cobs::xxh64(data, len, seed);
}

int ref_size_filter(uint64_t v, double p, uint32_t k, uint64_t* w) {
    return guarded(nullptr, 0, [&] { *w = cobs::bloom::size_filter(v, p, k); });
}

double ref_fpr_approx(uint64_t w, uint32_t k, uint64_t v) {
    return cobs::bloom::fpr_approx(w, k, v);
}

uint64_t ref_score_threshold(uint64_t ell, double K) { return cobs::bloom::score_threshold(ell, K); }

// extract_terms over nseg content strings; terms (ell*q bytes) malloc'd.
int ref_extract_terms(const uint8_t* const* segs, const uint64_t* lens, size_t nseg, uint32_t q,
                      int canonical, uint8_t** terms, uint64_t* ell, uint64_t* skipped,
                      uint64_t* occ) {
    return guarded(nullptr, 0, [&] {
        std::vector<std::string> content;
        for (size_t i = 0; i < nseg; ++i)
            content.emplace_back(reinterpret_cast<const char*>(segs[i]), lens[i]);
        cobs::TermSet ts = cobs::extract_terms("", content, q, canonical != 0);
        *ell = ts.term_count();
        *skipped = ts.skipped;
        *occ = ts.occurrences;
        *terms = static_cast<uint8_t*>(std::malloc(ts.terms.size() * q + 1));
        for (size_t t = 0; t < ts.terms.size(); ++t) std::memcpy(*terms + t * q, ts.terms[t].data(), q);
    });
}

void ref_free(void* p) { std::free(p); }

// Build classic (kind 0) or compact (kind 1) through the reference API and
// write it with the reference writer.
int ref_build_write(const uint8_t* const* segs, const uint64_t* lens, const uint64_t* doc_seg,
                    const char* const* names, size_t n_docs, uint32_t q, uint32_t k, double p,
                    int canonical, uint64_t block_size, int kind, uint64_t forced_w,
                    uint32_t workers, const char* path, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        cobs::IndexParams params;
        params.q = q;
        params.k = k;
        params.p = p;
        params.canonical = canonical != 0;
        params.block_size = block_size;
        std::vector<cobs::TermSet> docs(n_docs);
        std::vector<std::thread> th;
        std::atomic<size_t> next{0};
        auto work = [&] {
            for (size_t d = next.fetch_add(1); d < n_docs; d = next.fetch_add(1)) {
                std::vector<std::string> content;
                for (uint64_t s = doc_seg[d]; s < doc_seg[d + 1]; ++s)
                    content.emplace_back(reinterpret_cast<const char*>(segs[s]), lens[s]);
                docs[d] = cobs::extract_terms(names[d], content, q, canonical != 0);
            }
        };
        for (uint32_t i = 0; i < std::max(1u, workers); ++i) th.emplace_back(work);
        for (auto& x : th) x.join();
        if (kind == 0)
            cobs::write_index(cobs::build_classic(docs, params, workers, forced_w), path);
        else
            cobs::write_index(cobs::build_compact(docs, params, workers), path);
    });
}

// build_classic / build_compact over TermSets given directly (each segment
// is one term, kept as given: no sort, no dedup), + write_index.
int ref_build_terms_write(const uint8_t* const* segs, const uint64_t* lens, const uint64_t* doc_seg,
                          const char* const* names, size_t n_docs, uint32_t q, uint32_t k, double p,
                          int canonical, uint64_t block_size, int kind, uint64_t forced_w,
                          uint32_t workers, const char* path, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        cobs::IndexParams params;
        params.q = q;
        params.k = k;
        params.p = p;
        params.canonical = canonical != 0;
        params.block_size = block_size;
        std::vector<cobs::TermSet> docs(n_docs);
        for (size_t d = 0; d < n_docs; ++d) {
            docs[d].name = names[d];
            for (uint64_t s = doc_seg[d]; s < doc_seg[d + 1]; ++s)
                docs[d].terms.emplace_back(reinterpret_cast<const char*>(segs[s]), lens[s]);
            docs[d].occurrences = docs[d].terms.size();
        }
        if (kind == 0)
            cobs::write_index(cobs::build_classic(docs, params, workers, forced_w), path);
        else
            cobs::write_index(cobs::build_compact(docs, params, workers), path);
    });
}

// build_classic over docs [0, split) and [split, n) with a common forced
// width, merge_classic, write_index (acceptance.cpp criterion 9 shape).
int ref_merge_write(const uint8_t* const* segs, const uint64_t* lens, const uint64_t* doc_seg,
                    const char* const* names, size_t n_docs, size_t split, uint32_t q, uint32_t k,
                    double p, int canonical, uint64_t forced_w, const char* path, char* err,
                    size_t errlen) {
    return guarded(err, errlen, [&] {
        cobs::IndexParams params;
        params.q = q;
        params.k = k;
        params.p = p;
        params.canonical = canonical != 0;
        std::vector<cobs::TermSet> left, right;
        for (size_t d = 0; d < n_docs; ++d) {
            std::vector<std::string> content;
            for (uint64_t s = doc_seg[d]; s < doc_seg[d + 1]; ++s)
                content.emplace_back(reinterpret_cast<const char*>(segs[s]), lens[s]);
            (d < split ? left : right).push_back(cobs::extract_terms(names[d], content, q, canonical != 0));
        }
        cobs::ClassicIndex a = cobs::build_classic(left, params, 1, forced_w);
        cobs::ClassicIndex b = cobs::build_classic(right, params, 1, forced_w);
        cobs::write_index(cobs::merge_classic(a, b), path);
    });
}

int ref_open(const char* path, void** out, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        auto h = std::make_unique<Handle>();
        h->view = cobs::open_resident(path);
        index_names(h.get());
        *out = h.release();
    });
}

// cobs::open_random_access (storage.cpp:320-341): rows pread on demand,
// bytes_read() counts them (the reference's own traffic accounting).
int ref_open_random_access(const char* path, void** out, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        auto h = std::make_unique<Handle>();
        h->view = cobs::open_random_access(path);
        index_names(h.get());
        *out = h.release();
    });
}

uint64_t ref_bytes_read(void* h) { return static_cast<Handle*>(h)->view->bytes_read(); }

int ref_c5_open(uint64_t seed, uint64_t n, uint64_t B, double median, double sigma, double p,
                int materialise, int threads, void** out, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        auto h = std::make_unique<Handle>();
        h->view = std::make_unique<C5View>(seed, n, B, median, sigma, p, materialise != 0, threads);
        index_names(h.get());
        *out = h.release();
    });
}

void ref_close(void* h) { delete static_cast<Handle*>(h); }

uint64_t ref_total_docs(void* h) { return static_cast<Handle*>(h)->view->total_docs(); }

int ref_write(void* h, const char* path, char* err, size_t errlen) {
    return guarded(err, errlen, [&] { cobs::write_index(*static_cast<Handle*>(h)->view, path); });
}

// One query through cobs::query; hits returned as (global column, score)
// in the reference's order.  doc/score arrays malloc'd.
int ref_query(void* hv, const uint8_t* pat, uint64_t len, double K, uint64_t top_t,
              uint32_t workers, uint64_t* ell, uint64_t* skipped, uint64_t** docs,
              uint64_t** scores, uint64_t* n_hits, char* err, size_t errlen) {
    Handle* h = static_cast<Handle*>(hv);
    *docs = nullptr;
    *scores = nullptr;
    *n_hits = 0;
    return guarded(err, errlen, [&] {
        cobs::QueryOptions opts;
        opts.K = K;
        opts.top_t = top_t;
        opts.workers = workers;
        cobs::QueryResult r =
            cobs::query(*h->view, std::string_view(reinterpret_cast<const char*>(pat), len), opts);
        *ell = r.ell;
        *skipped = r.skipped;
        *n_hits = r.hits.size();
        *docs = static_cast<uint64_t*>(std::malloc(sizeof(uint64_t) * (r.hits.size() + 1)));
        *scores = static_cast<uint64_t*>(std::malloc(sizeof(uint64_t) * (r.hits.size() + 1)));
        for (size_t i = 0; i < r.hits.size(); ++i) {
            (*docs)[i] = h->global.at(r.hits[i].doc_name);
            (*scores)[i] = r.hits[i].score;
        }
    });
}

// Batch of queries, one std::thread per core pulling queries with
// workers = 1 (the CLI batch mode, proj/src/cli.cpp:205-221).  When
// `scores` is non-null the per-document score matrix (n x total_docs) is
// filled through the K = 1e-12 export (tau = 1; absent documents score 0)
// and K is ignored.  Returns total hits through n_hits[i].
int ref_query_batch(void* hv, const uint8_t* pats, const uint64_t* off, size_t n, double K,
                    int threads, uint64_t* ell, uint64_t* skipped, int* status, uint64_t* n_hits,
                    uint32_t* scores) {
    Handle* h = static_cast<Handle*>(hv);
    uint64_t D = h->view->total_docs();
    std::atomic<size_t> next{0};
    auto work = [&] {
        for (size_t i = next.fetch_add(1); i < n; i = next.fetch_add(1)) {
            status[i] = guarded(nullptr, 0, [&] {
                cobs::QueryOptions opts;
                opts.K = scores ? 1e-12 : K;
                opts.workers = 1;
                cobs::QueryResult r = cobs::query(
                    *h->view,
                    std::string_view(reinterpret_cast<const char*>(pats + off[i]), off[i + 1] - off[i]),
                    opts);
                ell[i] = r.ell;
                skipped[i] = r.skipped;
                n_hits[i] = r.hits.size();
                if (scores) {
                    uint32_t* row = scores + i * D;
                    std::memset(row, 0, sizeof(uint32_t) * D);
                    for (const auto& hit : r.hits) row[h->global.at(hit.doc_name)] = uint32_t(hit.score);
                }
            });
        }
    };
    std::vector<std::thread> th;
    for (int i = 0; i < std::max(1, threads); ++i) th.emplace_back(work);
    for (auto& x : th) x.join();
    return 0;
}

// `cobs query idx -F file` batch output (cli.cpp:192-223, print_hits
// :187-190), restated here because cli.cpp itself cannot be compiled (its
// CLI11 dependency is absent): the reference's read_fasta_named + query()
// per record, the CLI's exact formatting.  *out malloc'd.
int ref_query_fasta_tsv(void* hv, const char* path, double K, uint64_t top_t, char** out, char* err,
                        size_t errlen) {
    Handle* h = static_cast<Handle*>(hv);
    *out = nullptr;
    return guarded(err, errlen, [&] {
        if (!(K > 0.0 && K <= 1.0)) throw std::invalid_argument("K must be in (0,1]");
        auto queries = cobs::read_fasta_named(path);
        std::ostringstream o;
        for (const auto& [name, sequence] : queries) {
            try {
                cobs::QueryOptions opts;
                opts.K = K;
                opts.top_t = top_t;
                cobs::QueryResult r = cobs::query(*h->view, sequence, opts);
                o << '*' << name << '\t' << r.hits.size() << '\n';
                for (const auto& hit : r.hits) o << hit.doc_name << '\t' << hit.score << '\t' << r.ell << '\n';
            } catch (const cobs::DataError& e) {
                o << '*' << name << "\tERR\t" << e.what() << '\n';
            }
        }
        std::string s = o.str();
        *out = static_cast<char*>(std::malloc(s.size() + 1));
        std::memcpy(*out, s.c_str(), s.size() + 1);
    });
}

// `cobs build inputs... --mode M --format F` (cli.cpp:112-166) with the
// reference's load_document / build_* / write_index; expand_inputs
// (cli.cpp:60-82) restated for the same reason as above.
int ref_build_files(const char* const* inputs, size_t n, uint32_t q, uint32_t k, double p, int canonical,
                    uint64_t block_size, int kind, int format, const char* out_path, char* err,
                    size_t errlen) {
    namespace fs = std::filesystem;
    return guarded(err, errlen, [&] {
        cobs::IndexParams params;
        params.q = q;
        params.k = k;
        params.p = p;
        params.canonical = canonical != 0;
        params.block_size = block_size;
        params.validate();
        std::vector<fs::path> files;
        for (size_t i = 0; i < n; ++i) {
            fs::path path(inputs[i]);
            std::error_code ec;
            if (fs::is_directory(path, ec)) {
                std::vector<fs::path> found;
                for (const auto& e : fs::recursive_directory_iterator(path))
                    if (e.is_regular_file()) found.push_back(e.path());
                std::sort(found.begin(), found.end(),
                          [](const fs::path& a, const fs::path& b) { return a.string() < b.string(); });
                files.insert(files.end(), found.begin(), found.end());
            } else if (fs::is_regular_file(path, ec)) {
                files.push_back(path);
            } else {
                throw cobs::DataError(std::string("input not found: ") + inputs[i]);
            }
        }
        if (files.empty()) throw cobs::DataError("no input files");
        cobs::InputFormat fmt = format == 1   ? cobs::InputFormat::fasta
                                : format == 2 ? cobs::InputFormat::text
                                              : cobs::InputFormat::autodetect;
        std::vector<cobs::TermSet> docs;
        for (const auto& f : files) docs.push_back(cobs::load_document(f, q, canonical != 0, fmt));
        if (kind == 0)
            cobs::write_index(cobs::build_classic(docs, params, 1), out_path);
        else
            cobs::write_index(cobs::build_compact(docs, params, 1), out_path);
    });
}

} // extern "C"
