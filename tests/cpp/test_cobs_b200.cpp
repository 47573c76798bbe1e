// C++ parity tests of the host API (include/cobs_b200.hpp) on the device,
// shaped like the reference's own doctest suites (proj/tests/test_query.cpp,
// test_storage.cpp, test_index.cpp) and checked against the CPU oracle
// (oracle/cobs_oracle.h, test infrastructure) and the reference's golden
// vectors.  Build: `make cpptest`; run: tests/cpp/test_cobs_b200.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <functional>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include "cobs_b200.hpp"
#include "cobs_oracle.h"

using namespace cobs_b200;

// ---- a minimal doctest-like harness ---------------------------------------
static int g_fail = 0, g_checks = 0;
static std::vector<std::pair<const char*, std::function<void()>>>& registry() {
    static std::vector<std::pair<const char*, std::function<void()>>> r;
    return r;
}
struct Reg {
    Reg(const char* n, std::function<void()> f) { registry().emplace_back(n, std::move(f)); }
};
#define TEST_CASE(name)                       \
    static void name();                       \
    static Reg reg_##name(#name, name);       \
    static void name()
#define CHECK(x)                                                             \
    do {                                                                     \
        ++g_checks;                                                          \
        if (!(x)) {                                                          \
            ++g_fail;                                                        \
            std::fprintf(stderr, "%s:%d: CHECK(%s) failed\n", __FILE__, __LINE__, #x); \
        }                                                                    \
    } while (0)
#define CHECK_THROWS_AS(expr, T)                                             \
    do {                                                                     \
        ++g_checks;                                                          \
        bool ok_ = false;                                                    \
        try {                                                                \
            (void)(expr);                                                    \
        } catch (const T&) {                                                 \
            ok_ = true;                                                      \
        } catch (...) {                                                      \
        }                                                                    \
        if (!ok_) {                                                          \
            ++g_fail;                                                        \
            std::fprintf(stderr, "%s:%d: %s did not throw %s\n", __FILE__, __LINE__, #expr, #T); \
        }                                                                    \
    } while (0)

// ---- fixtures ----------------------------------------------------------------
static std::string random_dna(std::mt19937_64& rng, size_t n) {
    static const char b[4] = {'A', 'C', 'G', 'T'};
    std::uniform_int_distribution<int> d(0, 3);
    std::string s(n, 0);
    for (char& c : s) c = b[d(rng)];
    return s;
}
static std::vector<Document> gen_docs(std::mt19937_64& rng, size_t n, size_t lo, size_t hi) {
    std::uniform_real_distribution<double> ll(std::log(double(lo)), std::log(double(hi)));
    std::vector<Document> docs(n);
    for (size_t i = 0; i < n; ++i) {
        char nm[16];
        std::snprintf(nm, sizeof nm, "doc%04zu", i);
        docs[i].name = nm;
        docs[i].content = {random_dna(rng, std::max<size_t>(31, size_t(std::exp(ll(rng)))))};
    }
    return docs;
}
static std::string tmp_path(const char* name) { return std::string("/tmp/cobs_cpptest_") + name; }
static std::string read_file(const std::string& p) {
    std::ifstream in(p, std::ios::binary);
    std::ostringstream s;
    s << in.rdbuf();
    return s.str();
}
static void write_file(const std::string& p, const std::string& d) {
    std::ofstream(p, std::ios::binary) << d;
}

// The oracle's view of a file image.
struct Oracle {
    std::string img;
    orc_index x{};
    explicit Oracle(const std::string& image) : img(image) {
        char err[256];
        if (orc_parse(reinterpret_cast<const uint8_t*>(img.data()), img.size(), "t", &x, err, sizeof err))
            throw std::runtime_error(err);
    }
    ~Oracle() { orc_index_free(&x); }
    // hits (name, score), ell, skipped; code 0/1/2
    int query(const std::string& pat, double K, uint64_t top, QueryResult& out) const {
        orc_hit* hits = nullptr;
        uint64_t nh = 0;
        char err[256];
        int rc = orc_query(&x, reinterpret_cast<const uint8_t*>(pat.data()), pat.size(), K, top, nullptr, &out.ell,
                           &out.skipped, &hits, &nh, err, sizeof err);
        out.hits.clear();
        for (uint64_t i = 0; i < nh; ++i)
            out.hits.push_back({std::string(reinterpret_cast<const char*>(x.names[hits[i].doc]),
                                            x.name_len[hits[i].doc]),
                                hits[i].score});
        orc_free(hits);
        return rc;
    }
};

// ---- tests ---------------------------------------------------------------------
TEST_CASE(golden_layout_of_a_minimal_classic_index) { // test_storage.cpp:61-91 / FORMAT.md
    auto idx = build_classic({{"d", {std::string(31, 'A')}}}, IndexParams{});
    write_index(*idx, tmp_path("tiny.cobs"));
    static const unsigned char want[90] = {
        0x43, 0x4f, 0x42, 0x53, 0x49, 0x44, 0x58, 0x31, 1, 0, 0, 0, 0x1f, 0, 0, 0, 1, 0, 0, 0,
        0x33, 0x33, 0x33, 0x33, 0x33, 0x33, 0xd3, 0x3f, 0, 4, 0, 0, 0, 0, 0, 0, 1, 0, 0, 0, 0, 0, 0, 0,
        1, 0, 0, 0, 0, 0, 0, 0, 1, 0, 0, 0, 0, 0, 0, 0, 3, 0, 0, 0, 0, 0, 0, 0, 1, 0, 0x64,
        1, 0, 0, 0, 0, 0, 0, 0, 0x57, 0, 0, 0, 0, 0, 0, 0, 0, 1, 0};
    std::string got = read_file(tmp_path("tiny.cobs"));
    CHECK(got.size() == 90);
    CHECK(std::memcmp(got.data(), want, 90) == 0);
    CHECK(idx->width(0) == 3 && idx->doc(0, 0) == (DocEntry{"d", 1}));
}

TEST_CASE(ties_rank_by_name_ascending_after_score_descending) { // test_query.cpp:90-115
    std::mt19937_64 rng(11);
    std::string dna = random_dna(rng, 400);
    std::vector<Document> docs;
    for (const char* n : {"zebra", "apple", "mango"}) docs.push_back({n, {dna}});
    docs.push_back({"other", {random_dna(rng, 400)}});
    auto idx = build_classic(docs, IndexParams{});
    QueryResult r = query(*idx, dna.substr(0, 200), {1.0, 0, 1});
    CHECK(r.hits.size() >= 3);
    CHECK(r.hits[0].doc_name == "apple" && r.hits[1].doc_name == "mango" && r.hits[2].doc_name == "zebra");
    CHECK(r.hits[0].score == r.ell && r.hits[2].score == r.ell);
    QueryResult capped = query(*idx, dna.substr(0, 200), {1.0, 2, 1});
    CHECK(capped.hits.size() == 2 && capped.hits[0] == r.hits[0] && capped.hits[1] == r.hits[1]);
}

TEST_CASE(patterns_without_usable_terms_are_rejected) { // test_query.cpp:117-130
    std::mt19937_64 rng(13);
    auto plain = build_classic(gen_docs(rng, 4, 100, 200), IndexParams{});
    CHECK_THROWS_AS(query(*plain, "ACGT"), DataError);
    CHECK_THROWS_AS(query(*plain, std::string(40, 'A'), {0.0, 0, 1}), std::invalid_argument);
    CHECK_THROWS_AS(query(*plain, std::string(40, 'A'), {1.5, 0, 1}), std::invalid_argument);
    IndexParams cp;
    cp.canonical = true;
    auto canon = build_classic(gen_docs(rng, 4, 100, 200), cp);
    CHECK_THROWS_AS(query(*canon, std::string(40, 'N')), DataError);
}

TEST_CASE(canonical_queries_report_skipped_grams) { // test_query.cpp:132-148
    std::mt19937_64 rng(17);
    IndexParams p;
    p.canonical = true;
    auto docs = gen_docs(rng, 6, 200, 2000);
    auto idx = build_classic(docs, p);
    const std::string& c = docs[0].content[0];
    QueryResult r = query(*idx, c.substr(0, 60) + "N" + c.substr(60, 60), {1.0, 0, 1});
    CHECK(r.skipped == 31);
}

TEST_CASE(query_matches_the_oracle_across_kinds_and_k) { // test_query.cpp:150-186
    std::mt19937_64 rng(19);
    for (int trial = 0; trial < 8; ++trial) {
        IndexParams p;
        p.k = 1 + trial % 3;
        p.canonical = trial % 2 == 1;
        p.block_size = 4;
        auto docs = gen_docs(rng, 6 + trial * 3, 60, 2500);
        for (int kind = 0; kind < 2; ++kind) {
            auto idx = kind == 0 ? build_classic(docs, p) : build_compact(docs, p);
            write_index(*idx, tmp_path("q.cobs"));
            Oracle o(read_file(tmp_path("q.cobs")));
            for (int pat = 0; pat < 12; ++pat) {
                std::string pattern;
                if (pat % 3 == 0) {
                    pattern = random_dna(rng, 150);
                } else {
                    const std::string& src = docs[pat % docs.size()].content[0];
                    size_t len = std::min<size_t>(src.size(), 100 + pat * 40);
                    pattern = src.substr(rng() % (src.size() - len + 1), len);
                }
                QueryOptions opts{pat % 2 == 0 ? 1.0 : 0.5, 0, 1};
                QueryResult want;
                int rc = o.query(pattern, opts.K, 0, want);
                if (rc) {
                    CHECK_THROWS_AS(query(*idx, pattern, opts), DataError);
                    continue;
                }
                QueryResult got = query(*idx, pattern, opts);
                CHECK(got.ell == want.ell && got.skipped == want.skipped);
                CHECK(got.hits == want.hits);
            }
        }
    }
}

TEST_CASE(scores_above_65535_use_wide_counters) { // test_query.cpp:207-234
    std::mt19937_64 rng(29);
    std::string big = random_dna(rng, 70000);
    auto idx = build_classic({{"big", {big}}, {"small", {random_dna(rng, 500)}}}, IndexParams{});
    QueryResult r = query(*idx, big, {1.0, 0, 1});
    CHECK(r.ell > 65535);
    CHECK(!r.hits.empty() && r.hits[0].doc_name == "big" && r.hits[0].score == r.ell);
    write_index(*idx, tmp_path("w.cobs"));
    Oracle o(read_file(tmp_path("w.cobs")));
    QueryResult want;
    o.query(big.substr(1000, 40000), 0.9, 0, want);
    CHECK(query(*idx, big.substr(1000, 40000), {0.9, 0, 3}).hits == want.hits);
}

TEST_CASE(write_read_write_round_trips_byte_identically) { // test_storage.cpp:93-120
    std::mt19937_64 rng(43);
    IndexParams p;
    p.k = 2;
    p.block_size = 5;
    auto docs = gen_docs(rng, 17, 50, 3000);
    for (int kind = 0; kind < 2; ++kind) {
        auto idx = kind == 0 ? build_classic(docs, p) : build_compact(docs, p);
        write_index(*idx, tmp_path("o.cobs"));
        std::string original = read_file(tmp_path("o.cobs"));
        auto res = open_resident(tmp_path("o.cobs"));
        write_index(*res, tmp_path("c.cobs"));
        CHECK(read_file(tmp_path("c.cobs")) == original);
        auto ra = open_random_access(tmp_path("o.cobs"), 1ull << 20); // host-resident, streamed
        write_index(*ra, tmp_path("r.cobs"));
        CHECK(read_file(tmp_path("r.cobs")) == original);
        CHECK(res->params() == p && res->kind() == kind);
        QueryResult a = query(*res, docs[3].content[0].substr(0, 200), {0.5, 0, 1});
        QueryResult b = query(*ra, docs[3].content[0].substr(0, 200), {0.5, 0, 1});
        CHECK(a.hits == b.hits && a.ell == b.ell);
    }
}

TEST_CASE(corrupt_files_are_rejected) { // test_storage.cpp:192-235
    auto idx = build_classic({{"d", {std::string(31, 'A')}}}, IndexParams{});
    write_index(*idx, tmp_path("g.cobs"));
    std::string bytes = read_file(tmp_path("g.cobs"));
    for (auto [off, val] : std::vector<std::pair<size_t, int>>{
             {0, 'X'}, {8, 2}, {9, 7}, {10, 1}, {11, 2}, {12, 0}, {16, 0}, {36, 2}, {44, 9}, {60, 9}, {79, 12}}) {
        std::string m = bytes;
        m[off] = char(val);
        write_file(tmp_path("m.cobs"), m);
        CHECK_THROWS_AS(open_resident(tmp_path("m.cobs")), DataError);
    }
    for (size_t cut : {0u, 7u, 51u, 70u, 86u, 89u}) {
        write_file(tmp_path("m.cobs"), bytes.substr(0, cut));
        CHECK_THROWS_AS(open_resident(tmp_path("m.cobs")), DataError);
    }
    write_file(tmp_path("m.cobs"), bytes + "Z");
    CHECK_THROWS_AS(open_resident(tmp_path("m.cobs")), DataError);
    CHECK(open_resident(tmp_path("g.cobs"))->total_docs() == 1);
}

TEST_CASE(merge_equals_a_single_forced_width_build) { // acceptance.cpp criterion 9
    std::mt19937_64 rng(4444);
    auto all = gen_docs(rng, 60, 100, 8000);
    std::vector<Document> left(all.begin(), all.begin() + 35), right(all.begin() + 35, all.end());
    auto whole = build_classic(all, IndexParams{});
    auto a = build_classic(left, IndexParams{}, whole->width(0));
    auto b = build_classic(right, IndexParams{}, whole->width(0));
    auto merged = merge_classic(*a, *b);
    write_index(*merged, tmp_path("m1.cobs"));
    write_index(*whole, tmp_path("m2.cobs"));
    CHECK(read_file(tmp_path("m1.cobs")) == read_file(tmp_path("m2.cobs")));
    auto narrow = build_classic(right, IndexParams{}, whole->width(0) + 1);
    CHECK_THROWS_AS(merge_classic(*a, *narrow), DataError);
}

TEST_CASE(device_build_equals_the_oracle_build) { // byte-identical files
    std::mt19937_64 rng(91);
    for (int trial = 0; trial < 6; ++trial) {
        IndexParams p;
        p.k = 1 + trial % 3;
        p.canonical = trial % 2 == 0;
        p.block_size = 3 + trial;
        auto docs = gen_docs(rng, 20 + trial, 31, 3000);
        std::vector<const uint8_t*> segs;
        std::vector<uint64_t> lens, doc_seg{0};
        std::vector<const char*> names;
        for (const Document& d : docs) {
            segs.push_back(reinterpret_cast<const uint8_t*>(d.content[0].data()));
            lens.push_back(d.content[0].size());
            doc_seg.push_back(segs.size());
            names.push_back(d.name.c_str());
        }
        orc_params op{p.q, p.k, p.p, p.canonical ? 1 : 0, p.block_size, 0};
        for (int kind = 0; kind < 2; ++kind) {
            uint8_t* img = nullptr;
            uint64_t n = 0;
            char err[256];
            CHECK(orc_build_image(segs.data(), lens.data(), doc_seg.data(), names.data(), docs.size(), &op,
                                  kind, 0, &img, &n, err, sizeof err) == 0);
            auto idx = kind == 0 ? build_classic(docs, p) : build_compact(docs, p);
            write_index(*idx, tmp_path("b.cobs"));
            std::string got = read_file(tmp_path("b.cobs"));
            CHECK(got.size() == n && std::memcmp(got.data(), img, n) == 0);
            orc_free(img);
        }
    }
}

TEST_CASE(block_shards_merge_to_the_whole_index) {
    std::mt19937_64 rng(2024);
    auto docs = gen_docs(rng, 50, 200, 4000);
    IndexParams p;
    p.block_size = 6;
    auto built = build_compact(docs, p);
    write_index(*built, tmp_path("s.cobs"));
    auto whole = open_resident(tmp_path("s.cobs"));
    const uint64_t nb = whole->block_count();
    auto s0 = open_blocks(tmp_path("s.cobs"), 0, nb / 2);
    auto s1 = open_blocks(tmp_path("s.cobs"), nb / 2, nb);
    CHECK(column_offset(*s0) == 0 && column_offset(*s1) == s0->total_docs());
    std::vector<std::string> pats;
    for (int i = 0; i < 8; ++i) pats.push_back(docs[(i * 7) % docs.size()].content[0].substr(0, 300));
    for (uint64_t top_t : {uint64_t(0), uint64_t(3)}) {
        QueryOptions o;
        o.K = 0.3;
        o.top_t = top_t;
        auto w = query_batch(*whole, pats, o, nullptr);
        auto a = query_batch(*s0, pats, o, nullptr);
        auto b = query_batch(*s1, pats, o, nullptr);
        for (size_t i = 0; i < pats.size(); ++i) {
            std::vector<ScoredHit> m = a[i].hits;
            m.insert(m.end(), b[i].hits.begin(), b[i].hits.end());
            std::sort(m.begin(), m.end(), [](const ScoredHit& x, const ScoredHit& y) {
                return x.score != y.score ? x.score > y.score : x.doc_name < y.doc_name;
            });
            if (top_t && m.size() > top_t) m.resize(top_t);
            CHECK(m == w[i].hits);
            CHECK(a[i].ell == w[i].ell && b[i].ell == w[i].ell);
        }
    }
    CHECK_THROWS_AS(open_blocks(tmp_path("s.cobs"), 1, 1), std::invalid_argument);
}

TEST_CASE(file_backed_streaming_equals_resident) { // storage.hpp:23 from the file
    std::mt19937_64 rng(77);
    auto docs = gen_docs(rng, 40, 500, 6000);
    IndexParams p;
    p.block_size = 5;
    auto built = build_compact(docs, p);
    write_index(*built, tmp_path("f.cobs"));
    auto res = open_resident(tmp_path("f.cobs"));
    uint64_t biggest = 0;
    for (size_t b = 0; b < res->block_count(); ++b)
        biggest = std::max<uint64_t>(biggest, res->width(b) * ((res->row_bytes(b) + 31) / 32 * 32));
    auto fb = open_random_access(tmp_path("f.cobs"), 2 * biggest + 4096, 0, /*from_file=*/true);
    CHECK(fb->streaming() && !res->streaming());
    std::vector<std::string> pats;
    for (int i = 0; i < 6; ++i) pats.push_back(docs[i * 5].content[0].substr(100, 400));
    QueryOptions o;
    o.K = 0.4;
    auto x = query_batch(*res, pats, o, nullptr);
    auto y = query_batch(*fb, pats, o, nullptr);
    for (size_t i = 0; i < pats.size(); ++i) CHECK(x[i].hits == y[i].hits && x[i].ell == y[i].ell);
    write_index(*fb, tmp_path("f2.cobs"));
    CHECK(read_file(tmp_path("f.cobs")) == read_file(tmp_path("f2.cobs")));
}

int main() {
    for (auto& [name, fn] : registry()) {
        int before = g_fail;
        try {
            fn();
        } catch (const std::exception& e) {
            ++g_fail;
            std::fprintf(stderr, "%s: unexpected exception: %s\n", name, e.what());
        }
        std::printf("[%s] %s\n", g_fail == before ? "PASS" : "FAIL", name);
    }
    std::printf("%d checks, %d failed\n", g_checks, g_fail);
    return g_fail ? 1 : 0;
}
