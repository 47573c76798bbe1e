/* Host-side synthetic workload generator (C ABI over synth.h) used by the
 * bench and the tests to build documents and query batches.  Not part of the
 * COBS path. Multi-threaded with pthreads for the large configs. */
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#include "../paper_1905_09624_b200/csrc/synth.h"

void syn_c_doc_lengths(uint64_t seed, uint64_t n, int dist, double a, double b, uint64_t minlen,
                       uint64_t* out) {
    syn_doc_lengths(seed, n, dist, a, b, minlen, out);
}

void syn_c_c5_term_counts(uint64_t seed, uint64_t n, double median, double sigma, uint64_t* out) {
    syn_c5_term_counts(seed, n, median, sigma, out);
}

uint32_t syn_c_c5_thr16(uint64_t w, uint64_t n) { return syn_c5_thr16(w, n); }

void syn_c_c5_row(uint64_t seed, uint64_t block, uint64_t row, uint64_t rb, uint32_t thr16,
                  uint64_t dc, uint8_t* out) {
    uint64_t key = syn_c5_key(seed, block);
    for (uint64_t j = 0; j < rb; ++j) out[j] = syn_c5_byte_k(key, row, j, thr16, dc);
}

typedef struct job {
    uint64_t seed;
    int alpha;
    const uint64_t* doc_ids;
    const uint64_t* out_off;
    uint64_t n;
    char* out;
    const syn_query_spec* qs;
    const uint64_t* doc_len;
    uint64_t n_docs;
    uint64_t next;
    pthread_mutex_t mu;
} job;

static void* doc_worker(void* arg) {
    job* j = (job*)arg;
    for (;;) {
        pthread_mutex_lock(&j->mu);
        uint64_t i = j->next++;
        pthread_mutex_unlock(&j->mu);
        if (i >= j->n) return NULL;
        uint64_t len = j->out_off[i + 1] - j->out_off[i];
        syn_doc_bytes(j->seed, j->alpha, j->doc_ids[i], 0, len, j->out + j->out_off[i]);
    }
}

/* Documents doc_ids[i] with lengths out_off[i+1]-out_off[i] into out. */
void syn_c_docs(uint64_t seed, int alpha, const uint64_t* doc_ids, const uint64_t* out_off,
                uint64_t n, char* out, int threads) {
    job j;
    memset(&j, 0, sizeof j);
    j.seed = seed;
    j.alpha = alpha;
    j.doc_ids = doc_ids;
    j.out_off = out_off;
    j.n = n;
    j.out = out;
    pthread_mutex_init(&j.mu, NULL);
    if (threads < 1) threads = 1;
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
    for (int t = 0; t < threads; ++t) pthread_create(&th[t], NULL, doc_worker, &j);
    for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
    free(th);
}

static void* query_worker(void* arg) {
    job* j = (job*)arg;
    for (;;) {
        pthread_mutex_lock(&j->mu);
        uint64_t i = j->next;
        j->next += 64;
        pthread_mutex_unlock(&j->mu);
        if (i >= j->n) return NULL;
        uint64_t e = i + 64 < j->n ? i + 64 : j->n;
        for (; i < e; ++i)
            syn_query(j->qs, j->doc_len, j->n_docs, j->doc_ids[i], j->out + j->qs->qlen * (i));
    }
}

/* Queries ids[0..n) of a batch, each qlen bytes, packed into out[n*qlen]. */
void syn_c_queries(const syn_query_spec* qs, const uint64_t* doc_len, uint64_t n_docs,
                   const uint64_t* ids, uint64_t n, char* out, int threads) {
    job j;
    memset(&j, 0, sizeof j);
    j.qs = qs;
    j.doc_len = doc_len;
    j.n_docs = n_docs;
    j.doc_ids = ids;
    j.n = n;
    j.out = out;
    pthread_mutex_init(&j.mu, NULL);
    if (threads < 1) threads = 1;
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
    for (int t = 0; t < threads; ++t) pthread_create(&th[t], NULL, query_worker, &j);
    for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
    free(th);
}
