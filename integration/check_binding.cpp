// check_binding.cpp -- runs the reference's own callers over the B200 path
// through cobs_gpu_binding.hpp (test infrastructure: built against the
// reference sources by integration/Makefile into integration/_build/, run on
// a GPU box by tests/test_gpu_binding.py).  One "[PASS] name" / "[FAIL] name:
// detail" line per check; exit status 1 iff a check failed.
//
// What is exercised, reference side unchanged:
//   cobs::write_index(IndexView&)      over a DeviceIndexView (storage.cpp:345-397)
//   cobs::query(IndexView&, ...)       the reference engine reading rows from HBM
//   cobs::run_validation(...)          the reference's three validation suites
//   cobs::oracle_query(...)            the reference's replay oracle
//   cobs::open_resident / DataError    the reader's rejection messages
// against the device engine (cobs::gpu::query / query_batch) and the device
// build from TermSets (cobs::gpu::build_classic / build_compact).
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <iterator>
#include <random>
#include <sstream>
#include <unistd.h>
#include <string>
#include <vector>

#include "cobs/classic_index.hpp"
#include "cobs/compact_index.hpp"
#include "cobs/storage.hpp"
#include "cobs/validate.hpp"
#include "cobs_gpu_binding.hpp"

namespace fs = std::filesystem;

namespace {

int g_fail = 0;

void report(const std::string& name, bool ok, const std::string& detail = "") {
    std::printf("[%s] %s%s%s\n", ok ? "PASS" : "FAIL", name.c_str(), ok ? "" : ": ", ok ? "" : detail.c_str());
    std::fflush(stdout);
    if (!ok) ++g_fail;
}

std::string read_file(const fs::path& p) {
    std::ifstream in(p, std::ios::binary);
    return std::string(std::istreambuf_iterator<char>(in), {});
}

std::string dna(std::mt19937_64& rng, size_t n, double n_rate = 0.0) {
    static const char kAcgt[] = "ACGT";
    std::uniform_real_distribution<double> u(0.0, 1.0);
    std::string s(n, 'A');
    for (char& c : s) c = (n_rate > 0 && u(rng) < n_rate) ? 'N' : kAcgt[rng() & 3];
    return s;
}

struct Corpus {
    std::vector<cobs::CorpusDoc> docs;
    std::vector<cobs::TermSet> terms;
};

Corpus make_corpus(std::mt19937_64& rng, size_t n, const cobs::IndexParams& P) {
    Corpus c;
    std::uniform_int_distribution<size_t> len(0, 4000), nrec(1, 3);
    for (size_t i = 0; i < n; ++i) {
        cobs::CorpusDoc d;
        const size_t r = nrec(rng);
        for (size_t j = 0; j < r; ++j) d.records.push_back(dna(rng, len(rng) / r, i % 7 == 0 ? 0.01 : 0.0));
        char name[32];
        std::snprintf(name, sizeof name, "doc_%04zu", (i * 7919) % n);
        d.terms = cobs::extract_terms(name, d.records, P.q, P.canonical);
        c.terms.push_back(d.terms);
        c.docs.push_back(std::move(d));
    }
    return c;
}

std::vector<std::string> make_patterns(std::mt19937_64& rng, const Corpus& c, size_t n) {
    std::vector<std::string> pats;
    for (size_t i = 0; i < n; ++i) {
        const auto& recs = c.docs[rng() % c.docs.size()].records;
        const std::string& src = recs[rng() % recs.size()];
        if (i % 3 == 2 || src.size() < 200) {
            pats.push_back(dna(rng, 100 + rng() % 900));
            continue;
        }
        const size_t lo = rng() % (src.size() - 150);
        std::string p = src.substr(lo, std::min<size_t>(src.size() - lo, 150 + rng() % 850));
        for (size_t m = 0; m < p.size() / 50; ++m) p[rng() % p.size()] = "ACGT"[rng() & 3];
        pats.push_back(std::move(p));
    }
    pats.push_back("ACGT");       // shorter than q: DataError
    pats.push_back(std::string(40, 'N')); // all skipped when canonical
    return pats;
}

bool same(const cobs::QueryResult& a, const cobs::QueryResult& b) {
    return a.ell == b.ell && a.skipped == b.skipped && a.hits == b.hits;
}

// reference query (any view) vs device query, including the error path
std::string compare_queries(const cobs::IndexView& ref_view, const cobs::IndexView& ref_over_dev,
                            const cobs::gpu::DeviceIndexView& dev, const std::vector<std::string>& pats,
                            const cobs::QueryOptions& opts, bool via_rows) {
    std::vector<std::string> errors;
    std::vector<cobs::QueryResult> batch = cobs::gpu::query_batch(dev, pats, opts, &errors);
    for (size_t i = 0; i < pats.size(); ++i) {
        std::string want_err;
        cobs::QueryResult want;
        try {
            want = cobs::query(ref_view, pats[i], opts);
        } catch (const cobs::DataError& e) {
            want_err = e.what();
        }
        if (want_err != errors[i]) return "error mismatch at pattern " + std::to_string(i) + ": '" + want_err + "' vs '" + errors[i] + "'";
        if (!want_err.empty()) continue;
        if (!same(want, batch[i])) return "device result differs at pattern " + std::to_string(i);
        if (via_rows && i % 8 == 0 && !same(want, cobs::query(ref_over_dev, pats[i], opts)))
            return "reference engine over HBM rows differs at pattern " + std::to_string(i);
    }
    return "";
}

} // namespace

int main(int argc, char** argv) {
    const int device = argc > 1 ? std::atoi(argv[1]) : 0;
    const fs::path dir = fs::temp_directory_path() / ("cobs_binding_" + std::to_string(::getpid()));
    fs::create_directories(dir);
    std::mt19937_64 rng(20261019);

    struct Cfg {
        const char* name;
        uint32_t q, k;
        bool canonical;
        uint64_t block_size;
        bool compact;
    };
    const Cfg cfgs[] = {{"classic_q31_k1", 31, 1, false, 1024, false},
                        {"compact_q31_k1_canonical_B64", 31, 1, true, 64, true},
                        {"compact_q20_k3_B100", 20, 3, false, 100, true}};

    for (const Cfg& cfg : cfgs) {
        cobs::IndexParams P;
        P.q = cfg.q;
        P.k = cfg.k;
        P.canonical = cfg.canonical;
        P.block_size = cfg.block_size;
        const std::string tag = cfg.name;
        Corpus corpus = make_corpus(rng, 300, P);
        const fs::path ref_path = dir / (tag + "_ref.cobs");
        if (cfg.compact)
            cobs::write_index(cobs::build_compact(corpus.terms, P, 4), ref_path);
        else
            cobs::write_index(cobs::build_classic(corpus.terms, P, 4), ref_path);
        const std::string ref_bytes = read_file(ref_path);

        // device build from the reference's TermSets; the reference writer
        // over the DeviceIndexView (row_data = D2H) reproduces the file
        auto built = cfg.compact ? cobs::gpu::build_compact(corpus.terms, P, 1, device)
                                 : cobs::gpu::build_classic(corpus.terms, P, 1, 0, device);
        const fs::path dev_path = dir / (tag + "_dev.cobs");
        cobs::write_index(*built, dev_path);
        report(tag + ": reference write_index over device-built view == reference build", read_file(dev_path) == ref_bytes);

        // the reference's validation suites over the device-built index
        // (rows served from a host mirror of the HBM payload)
        built->mirror();
        cobs::ValidationReport rep = cobs::run_validation(*built, corpus.docs, 100000, 7); // CLI default trials (cli.cpp:337)
        report(tag + ": run_validation over device-built view",
               rep.all_ok(),
               rep.no_false_negatives.detail + " | " + rep.fpr_measurement.detail + " | " + rep.oracle_equivalence.detail);

        // open the reference's file on the device; queries: device engine ==
        // reference engine (resident file) == reference engine over HBM rows
        auto dev = cobs::gpu::open_resident(ref_path.string(), device);
        auto ref_view = cobs::open_resident(ref_path);
        std::vector<std::string> pats = make_patterns(rng, corpus, 120);
        for (double K : {0.3, 0.8, 1.0}) {
            for (uint64_t top_t : {uint64_t(0), uint64_t(5)}) {
                cobs::QueryOptions o;
                o.K = K;
                o.top_t = top_t;
                std::string err = compare_queries(*ref_view, *dev, *dev, pats, o, K == 0.8 && top_t == 0);
                std::ostringstream n;
                n << tag << ": query K=" << K << " top_t=" << top_t;
                report(n.str(), err.empty(), err);
            }
        }
        // oracle_query (replay from the corpus) == device query
        {
            std::string err;
            for (size_t i = 0; i < 10 && err.empty(); ++i) {
                cobs::QueryOptions o;
                o.K = 0.5;
                cobs::QueryResult a = cobs::gpu::query(*dev, pats[i], o);
                cobs::QueryResult b = cobs::oracle_query(*dev, corpus.docs, pats[i], o);
                if (!same(a, b)) err = "pattern " + std::to_string(i);
            }
            report(tag + ": oracle_query == device query", err.empty(), err);
        }
        // mirrored row_data serves the same bytes
        {
            dev->mirror();
            const fs::path mir_path = dir / (tag + "_mirror.cobs");
            cobs::write_index(*dev, mir_path);
            report(tag + ": write_index over mirrored view == file", read_file(mir_path) == ref_bytes);
        }
        // exceptions: K outside (0,1], l = 0 (query.cpp:125-138)
        {
            std::string want, got;
            cobs::QueryOptions bad;
            bad.K = 0.0;
            try { cobs::query(*ref_view, "ACGTACGT", bad); } catch (const std::invalid_argument& e) { want = e.what(); }
            try { cobs::gpu::query(*dev, "ACGTACGT", bad); } catch (const std::invalid_argument& e) { got = e.what(); }
            report(tag + ": invalid_argument for K = 0", !want.empty() && want == got, want + " vs " + got);
            want.clear();
            got.clear();
            try { cobs::query(*ref_view, "ACG", {}); } catch (const cobs::DataError& e) { want = e.what(); }
            try { cobs::gpu::query(*dev, "ACG", {}); } catch (const cobs::DataError& e) { got = e.what(); }
            report(tag + ": DataError for a short pattern", !want.empty() && want == got, want + " vs " + got);
        }
    }

    // reader rejection: truncated and bad-magic files give the same DataError
    {
        cobs::IndexParams P;
        Corpus corpus = make_corpus(rng, 20, P);
        const fs::path good = dir / "small.cobs";
        cobs::write_index(cobs::build_classic(corpus.terms, P), good);
        std::string bytes = read_file(good);
        std::string err;
        for (int variant = 0; variant < 3 && err.empty(); ++variant) {
            std::string b = bytes;
            if (variant == 0) b.resize(b.size() - 3);
            if (variant == 1) b[0] = 'X';
            if (variant == 2) b.resize(40);
            const fs::path bad = dir / ("bad" + std::to_string(variant) + ".cobs");
            std::ofstream(bad, std::ios::binary).write(b.data(), b.size());
            std::string want, got;
            try { cobs::open_resident(bad); } catch (const cobs::DataError& e) { want = e.what(); }
            try { cobs::gpu::open_resident(bad.string(), device); } catch (const cobs::DataError& e) { got = e.what(); }
            if (want.empty() || want != got) err = "variant " + std::to_string(variant) + ": " + want + " vs " + got;
        }
        report("open_resident rejection messages", err.empty(), err);
    }

    // merge_classic of two device builds == the reference's merge
    {
        cobs::IndexParams P;
        Corpus a = make_corpus(rng, 50, P), b = make_corpus(rng, 40, P);
        for (auto& t : b.terms) t.name = "b_" + t.name;
        const uint64_t w = 50000;
        auto da = cobs::gpu::build_classic(a.terms, P, 1, w, device);
        auto db = cobs::gpu::build_classic(b.terms, P, 1, w, device);
        auto dm = cobs::gpu::merge_classic(*da, *db, device);
        const fs::path want_path = dir / "merge_ref.cobs", got_path = dir / "merge_dev.cobs";
        cobs::write_index(cobs::merge_classic(cobs::build_classic(a.terms, P, 1, w), cobs::build_classic(b.terms, P, 1, w)),
                          want_path);
        cobs::write_index(*dm, got_path);
        report("merge_classic == reference merge", read_file(want_path) == read_file(got_path));
    }

    fs::remove_all(dir);
    std::printf("%d failed\n", g_fail);
    return g_fail ? 1 : 0;
}
