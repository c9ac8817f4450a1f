/*
 * oracle.c — CPU restatement of the reference hot path. TEST INFRASTRUCTURE ONLY
 * (see oracle.h). Plain C11 + pthreads; every function cites the reference
 * file:line (under /root/reference/proj) whose algorithm it restates.
 */
#define _GNU_SOURCE
#include "oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

/* ------------------------------------------------------------------ PRF */

static inline uint64_t rotl64(uint64_t x, unsigned r) {
    return r == 0 ? x : (x << r) | (x >> (64 - r));
}

/* prf.cpp:47-76: Threefish-256 rotation schedule, 20 rounds, key-schedule parity
 * word 0x1BD11BDAA9FC1A22, subkey injection before round 0 and after every 4th round,
 * x1 <-> x3 swap after every round. */
void or_threefry(const uint64_t key[4], const uint64_t ctr[4], uint64_t out[4]) {
    static const unsigned rot[8][2] = {{14, 16}, {52, 57}, {23, 40}, {5, 37},
                                       {25, 33}, {46, 12}, {58, 22}, {32, 32}};
    uint64_t ks[5];
    ks[0] = key[0];
    ks[1] = key[1];
    ks[2] = key[2];
    ks[3] = key[3];
    ks[4] = 0x1BD11BDAA9FC1A22ull ^ key[0] ^ key[1] ^ key[2] ^ key[3];
    uint64_t x0 = ctr[0] + ks[0], x1 = ctr[1] + ks[1], x2 = ctr[2] + ks[2], x3 = ctr[3] + ks[3];
    for (unsigned d = 0; d < 20; ++d) {
        x0 += x1;
        x1 = rotl64(x1, rot[d & 7][0]) ^ x0;
        x2 += x3;
        x3 = rotl64(x3, rot[d & 7][1]) ^ x2;
        uint64_t t = x1;
        x1 = x3;
        x3 = t;
        if ((d & 3) == 3) {
            const uint64_t s = d / 4 + 1;
            x0 += ks[s % 5];
            x1 += ks[(s + 1) % 5];
            x2 += ks[(s + 2) % 5];
            x3 += ks[(s + 3) % 5] + s;
        }
    }
    out[0] = x0;
    out[1] = x1;
    out[2] = x2;
    out[3] = x3;
}

/* prf.hpp:29-37 */
uint64_t or_tag(const char* name) {
    uint64_t h = 0xcbf29ce484222325ull;
    for (const unsigned char* p = (const unsigned char*)name; *p; ++p) {
        h ^= *p;
        h *= 0x100000001b3ull;
    }
    return h;
}

/* prf.cpp:80-82 */
uint64_t or_stream_word(const uint64_t key[4], uint64_t tag, uint64_t sub, uint64_t index) {
    const uint64_t ctr[4] = {tag, sub, index, 0};
    uint64_t o[4];
    or_threefry(key, ctr, o);
    return o[0];
}

/* prf.cpp:84-94 */
uint64_t or_uniform_below(const uint64_t key[4], uint64_t tag, uint64_t sub, uint64_t bound,
                          uint64_t index) {
    if (bound == 0) return UINT64_MAX;
    if ((bound & (bound - 1)) == 0) return or_stream_word(key, tag, sub, index) & (bound - 1);
    const uint64_t limit = ~0ull - (~0ull % bound + 1) % bound;
    for (uint64_t attempt = 0;; ++attempt) {
        const uint64_t ctr[4] = {tag, sub, index, attempt};
        uint64_t o[4];
        or_threefry(key, ctr, o);
        if (o[0] <= limit) return o[0] % bound;
    }
}

/* prf.cpp:96-102 */
int or_bernoulli(const uint64_t key[4], uint64_t tag, uint64_t sub, double p, uint64_t index) {
    if (p < 0.0 || p > 1.0) return -1;
    const uint64_t r = or_stream_word(key, tag, sub, index);
    const double u = (double)(r >> 11) * 0x1.0p-53;
    return u < p;
}

/* prf.cpp:104-115: word w = block({tag, sub, w/4, 1})[w%4], tail masked. */
void or_stream_bits(const uint64_t key[4], uint64_t tag, uint64_t sub, uint64_t nbits,
                    uint64_t* out) {
    const uint64_t nwords = (nbits + 63) / 64;
    for (uint64_t w = 0; w < nwords; w += 4) {
        const uint64_t ctr[4] = {tag, sub, w / 4, 1};
        uint64_t o[4];
        or_threefry(key, ctr, o);
        for (unsigned i = 0; i < 4 && w + i < nwords; ++i) out[w + i] = o[i];
    }
    if (nbits & 63) out[nwords - 1] &= (1ull << (nbits & 63)) - 1;
}

/* ------------------------------------------------------------- threads */

static int resolve_threads(int nthreads) {
    if (nthreads > 0) return nthreads;
    long c = sysconf(_SC_NPROCESSORS_ONLN);
    return c > 0 ? (int)c : 1;
}

typedef void (*range_fn)(void* ctx, uint64_t lo, uint64_t hi, int tid);
typedef struct {
    range_fn fn;
    void* ctx;
    uint64_t lo, hi;
    int tid;
} range_job;

static void* range_thread(void* p) {
    range_job* j = (range_job*)p;
    j->fn(j->ctx, j->lo, j->hi, j->tid);
    return NULL;
}

/* Split [0, n) into nthreads contiguous ranges, aligned to `align` elements. */
static void parallel_ranges(uint64_t n, uint64_t align, int nthreads, range_fn fn, void* ctx) {
    nthreads = resolve_threads(nthreads);
    if (nthreads == 1 || n < 2 * align) {
        fn(ctx, 0, n, 0);
        return;
    }
    uint64_t per = (n + nthreads - 1) / nthreads;
    per = (per + align - 1) / align * align;
    pthread_t th[512];
    range_job jobs[512];
    if (nthreads > 512) nthreads = 512;
    int started = 0;
    for (int t = 0; t < nthreads; ++t) {
        const uint64_t lo = (uint64_t)t * per;
        if (lo >= n) break;
        const uint64_t hi = lo + per < n ? lo + per : n;
        jobs[t] = (range_job){fn, ctx, lo, hi, t};
        pthread_create(&th[t], NULL, range_thread, &jobs[t]);
        ++started;
    }
    for (int t = 0; t < started; ++t) pthread_join(th[t], NULL);
}

/* --------------------------------------------------------- input maker */

typedef struct {
    const uint64_t* key;
    double p;
    uint64_t nbits;
    uint64_t* out;
    uint64_t tag;
} input_ctx;

static void input_range(void* vc, uint64_t lo, uint64_t hi, int tid) {
    (void)tid;
    input_ctx* c = (input_ctx*)vc;
    /* lo/hi are word indices, multiples of 4 */
    const uint64_t nwords = (c->nbits + 63) / 64;
    if (c->p == 0.5) {
        for (uint64_t w = lo; w < hi; w += 4) {
            const uint64_t ctr[4] = {c->tag, 0, w / 4, 1};
            uint64_t o[4];
            or_threefry(c->key, ctr, o);
            for (unsigned i = 0; i < 4 && w + i < nwords; ++i) c->out[w + i] = o[i];
        }
    } else {
        for (uint64_t w = lo; w < hi && w < nwords; ++w) {
            uint64_t v = 0;
            for (unsigned b = 0; b < 64; ++b) {
                const uint64_t i = w * 64 + b;
                if (i >= c->nbits) break;
                if (or_bernoulli(c->key, c->tag, 0, c->p, i) == 1) v |= 1ull << b;
            }
            c->out[w] = v;
        }
    }
}

void or_make_input(const uint64_t key[4], double p, uint64_t nbits, uint64_t* out,
                   int nthreads) {
    const uint64_t nwords = (nbits + 63) / 64;
    if (nwords == 0) return;
    input_ctx c = {key, p, nbits, out, or_tag("input")};
    parallel_ranges((nwords + 3) / 4 * 4, 4, nthreads, input_range, &c);
    if (nbits & 63) out[nwords - 1] &= (1ull << (nbits & 63)) - 1;
}

/* ------------------------------------------------------------- sampler */

typedef struct {
    uint64_t n;
    uint32_t s;
    const uint64_t* key;
    uint64_t tag;
    uint32_t* assignment;
    uint64_t* counts; /* nthreads x s */
} assign_ctx;

static void assign_range(void* vc, uint64_t lo, uint64_t hi, int tid) {
    assign_ctx* c = (assign_ctx*)vc;
    uint64_t* cnt = c->counts + (uint64_t)tid * c->s;
    for (uint64_t i = lo; i < hi; ++i) {
        const uint32_t v = (uint32_t)or_uniform_below(c->key, c->tag, 0, c->s, i) + 1;
        c->assignment[i] = v;
        ++cnt[v - 1];
    }
}

/* sampling.cpp:10-25: V_i = uniform_below(s, i) + 1 from KeyedStream(seed, "sampling"). */
int or_assign_subblocks(uint64_t n, uint32_t s, const uint64_t key[4], uint32_t* assignment,
                        uint64_t* raw_counts, int nthreads) {
    if (s == 0) return -1;
    nthreads = resolve_threads(nthreads);
    if (nthreads > 512) nthreads = 512;
    uint64_t* counts = (uint64_t*)calloc((size_t)nthreads * s, sizeof(uint64_t));
    assign_ctx c = {n, s, key, or_tag("sampling"), assignment, counts};
    parallel_ranges(n, 64, nthreads, assign_range, &c);
    for (uint32_t j = 0; j < s; ++j) {
        uint64_t t = 0;
        for (int q = 0; q < nthreads; ++q) t += counts[(uint64_t)q * s + j];
        raw_counts[j] = t;
    }
    free(counts);
    return 0;
}

/* sampling.cpp:27-39 (stable: round order inside every block). */
void or_sift_partition(const uint8_t* keep, uint64_t n, const uint32_t* assignment, uint32_t s,
                       uint64_t* offsets, uint64_t* indices) {
    memset(offsets, 0, sizeof(uint64_t) * ((size_t)s + 1));
    for (uint64_t i = 0; i < n; ++i)
        if (keep[i]) ++offsets[assignment[i]];
    for (uint32_t j = 0; j < s; ++j) offsets[j + 1] += offsets[j];
    uint64_t* fill = (uint64_t*)malloc(sizeof(uint64_t) * ((size_t)s + 1));
    memcpy(fill, offsets, sizeof(uint64_t) * ((size_t)s + 1));
    for (uint64_t i = 0; i < n; ++i)
        if (keep[i]) indices[fill[assignment[i] - 1]++] = i;
    free(fill);
}

/* ------------------------------------------------------------ toeplitz */

/* bitstring.cpp:91-127: head / whole-word body / tail; reads past src yield 0. */
void or_xor_bit_range(uint64_t* dst, uint64_t dst_words, uint64_t dst_off, const uint64_t* src,
                      uint64_t src_words, uint64_t src_off, uint64_t nbits) {
    (void)dst_words;
    if (nbits == 0) return;
#define RD(bit)                                                                          \
    ({                                                                                   \
        const uint64_t q_ = (bit) >> 6;                                                  \
        const unsigned r_ = (unsigned)((bit) & 63);                                      \
        uint64_t lo_ = q_ < src_words ? src[q_] : 0;                                     \
        uint64_t v_ = lo_;                                                               \
        if (r_) {                                                                        \
            uint64_t hi_ = q_ + 1 < src_words ? src[q_ + 1] : 0;                         \
            v_ = (lo_ >> r_) | (hi_ << (64 - r_));                                       \
        }                                                                                \
        v_;                                                                              \
    })
    uint64_t done = 0;
    const unsigned dhead = (unsigned)(dst_off & 63);
    if (dhead) {
        const uint64_t take = 64 - dhead < nbits ? 64 - dhead : nbits;
        const uint64_t mask = take == 64 ? ~0ull : ((1ull << take) - 1);
        dst[dst_off >> 6] ^= (RD(src_off) & mask) << dhead;
        done = take;
    }
    uint64_t dw = (dst_off + done) >> 6;
    while (nbits - done >= 64) {
        dst[dw++] ^= RD(src_off + done);
        done += 64;
    }
    if (done < nbits) {
        const uint64_t take = nbits - done;
        dst[dw] ^= RD(src_off + done) & ((1ull << take) - 1);
    }
#undef RD
}

/* toeplitz.cpp:34-52: column j of T is the seed slice starting at bit n-1-j; XOR it into
 * the output for every set input bit (seed padded by one zero word, toeplitz.cpp:25-30). */
void or_toeplitz_hash(const uint64_t* seed, uint64_t m, uint64_t n, const uint64_t* input,
                      uint64_t* out) {
    const uint64_t sw = (m + n - 1 + 63) / 64;
    const uint64_t ow = (m + 63) / 64;
    memset(out, 0, ow * 8);
    const uint64_t iw = (n + 63) / 64;
    for (uint64_t w = 0; w < iw; ++w) {
        uint64_t word = input[w];
        while (word) {
            const uint64_t j = w * 64 + (uint64_t)__builtin_ctzll(word);
            or_xor_bit_range(out, ow, 0, seed, sw, n - 1 - j, m);
            word &= word - 1;
        }
    }
}

static inline int get_bit(const uint64_t* w, uint64_t i) { return (int)((w[i >> 6] >> (i & 63)) & 1); }

/* toeplitz.cpp:54-76 */
void or_blocked_toeplitz_hash(const uint64_t* seed, uint64_t m, uint64_t n,
                              const uint64_t* input, uint64_t m_prime, uint64_t n_prime,
                              uint64_t* out) {
    const uint64_t sw = (m + n - 1 + 63) / 64;
    const uint64_t ow = (m + 63) / 64;
    memset(out, 0, ow * 8);
    for (uint64_t r0 = 0; r0 < m; r0 += m_prime) {
        const uint64_t rows = m_prime < m - r0 ? m_prime : m - r0;
        for (uint64_t c0 = 0; c0 < n; c0 += n_prime) {
            const uint64_t cols = n_prime < n - c0 ? n_prime : n - c0;
            for (uint64_t j = c0; j < c0 + cols; ++j) {
                if (!get_bit(input, j)) continue;
                or_xor_bit_range(out, ow, r0, seed, sw, n - 1 - j + r0, rows);
            }
        }
    }
}

/* tests/oracle_gf2.hpp:38-48 */
void or_dense_toeplitz(const uint64_t* seed, uint64_t m, uint64_t n, const uint64_t* input,
                       uint64_t* out) {
    memset(out, 0, ((m + 63) / 64) * 8);
    for (uint64_t i = 0; i < m; ++i) {
        int acc = 0;
        for (uint64_t j = 0; j < n; ++j) acc ^= get_bit(seed, n - 1 + i - j) & get_bit(input, j);
        if (acc) out[i >> 6] |= 1ull << (i & 63);
    }
}

void or_reverse_bits(const uint64_t* x, uint64_t n, uint64_t* y) {
    memset(y, 0, ((n + 63) / 64) * 8);
    for (uint64_t c = 0; c < n; ++c)
        if (get_bit(x, n - 1 - c)) y[c >> 6] |= 1ull << (c & 63);
}

/* K[i] = parity(sum_c seed[i+c] & y[c]) with y[c] = x[n-1-c] — the same bit as
 * toeplitz.hpp:11-17's T[i][j] = seed[n-1+i-j] applied to x[j]. Word-parallel. */
void or_toeplitz_rows(const uint64_t* seed, uint64_t n, const uint64_t* y_rev,
                      const uint64_t* rows, uint64_t nrows, uint8_t* bits_out) {
    const uint64_t yw = (n + 63) / 64;
    for (uint64_t q = 0; q < nrows; ++q) {
        const uint64_t i = rows[q];
        uint64_t acc = 0;
        for (uint64_t c = 0; c < yw; ++c) {
            const uint64_t bit = i + 64 * c;
            const uint64_t qw = bit >> 6;
            const unsigned r = (unsigned)(bit & 63);
            /* window of 64 seed bits starting at `bit`; caller guarantees the seed buffer
             * holds ceil((i + 64*yw)/64)+1 words (bits past the seed only meet zero y bits) */
            uint64_t win = seed[qw] >> r;
            if (r) win |= seed[qw + 1] << (64 - r);
            acc ^= win & y_rev[c];
        }
        bits_out[q] = (uint8_t)(__builtin_popcountll(acc) & 1);
    }
}

/* ------------------------------------------------------ abort threshold */

/* sampling.cpp:41-49 */
double or_relative_entropy(double x, double p) {
    if (!(p > 0.0 && p < 1.0)) return NAN;
    if (!(x >= 0.0 && x <= 1.0)) return NAN;
    if (x == 0.0) return log(1.0 / (1.0 - p));
    if (x == 1.0) return log(1.0 / p);
    return x * log(x / p) + (1.0 - x) * log((1.0 - x) / (1.0 - p));
}

/* sampling.cpp:51-56 */
double or_binomial_tail_bound(uint64_t n, uint64_t limit, double p) {
    const double x = (double)limit / (double)n;
    const double arg = sqrt(2.0 * (double)n * or_relative_entropy(x, p));
    return 0.5 * erfc(arg / sqrt(2.0));
}

/* sampling.cpp:58-90 */
uint64_t or_block_limit(uint64_t n, double p, double eps, uint64_t m_blocks, int* err) {
    *err = 0;
    if (n == 0 || !(p > 0.0 && p < 1.0) || !(eps > 0.0 && eps < 1.0) || m_blocks == 0) {
        *err = 1;
        return 0;
    }
    const double threshold = eps / (double)m_blocks;
    if (threshold < 1e-300) {
        *err = 2;
        return 0;
    }
    const uint64_t lo0 = (uint64_t)ceil((double)n * p);
    if (or_binomial_tail_bound(n, n, p) > threshold) {
        *err = 2;
        return 0;
    }
    if (or_binomial_tail_bound(n, lo0, p) <= threshold) return lo0;
    uint64_t lo = lo0, hi = n;
    while (hi - lo > 1) {
        const uint64_t mid = lo + (hi - lo) / 2;
        if (or_binomial_tail_bound(n, mid, p) <= threshold)
            hi = mid;
        else
            lo = mid;
    }
    return hi;
}

/* toeplitz.cpp:78-89 */
uint64_t or_cycle_estimate(uint64_t input_len, uint64_t output_len, uint64_t m_prime, int* err) {
    *err = 0;
    if (m_prime == 0) {
        *err = 1;
        return 0;
    }
    const uint64_t passes = (output_len + m_prime - 1) / m_prime;
    const unsigned __int128 total = (unsigned __int128)input_len + output_len +
                                    (unsigned __int128)(input_len + m_prime) * passes;
    if (total > (unsigned __int128)~0ull) {
        *err = 3;
        return 0;
    }
    return (uint64_t)total;
}

/* ---------------------------------------------------------- extraction */

typedef struct {
    const uint64_t* input;
    uint32_t s;
    const uint64_t* hash_key;
    int per_block;
    uint64_t k;
    const uint64_t* offsets;
    const uint64_t* indices;
    uint64_t* out_blocks; /* s x ceil(k/64) */
    uint64_t tag;
    const uint32_t* which; /* NULL: identity */
} hash_ctx;

static void hash_one(hash_ctx* c, uint32_t j, const uint64_t* idx, uint64_t nj, uint64_t* out) {
    /* gather (ssbh_main.cpp:329-331) */
    uint64_t* x = (uint64_t*)calloc((nj + 63) / 64 + 1, 8);
    for (uint64_t q = 0; q < nj; ++q)
        if (get_bit(c->input, idx[q])) x[q >> 6] |= 1ull << (q & 63);
    /* seed (ssbh_main.cpp:332-334) */
    const uint64_t sb = c->k + nj - 1;
    uint64_t* seed = (uint64_t*)calloc((sb + 63) / 64 + 1, 8);
    or_stream_bits(c->hash_key, c->tag, c->per_block ? j : 0, sb, seed);
    or_toeplitz_hash(seed, c->k, nj, x, out);
    free(seed);
    free(x);
}

static void hash_range(void* vc, uint64_t lo, uint64_t hi, int tid) {
    (void)tid;
    hash_ctx* c = (hash_ctx*)vc;
    const uint64_t kw = (c->k + 63) / 64;
    for (uint64_t q = lo; q < hi; ++q) {
        const uint32_t j = c->which ? c->which[q] : (uint32_t)q;
        const uint64_t slot = c->which ? q : j;
        hash_one(c, j, c->indices + c->offsets[slot], c->offsets[slot + 1] - c->offsets[slot],
                 c->out_blocks + slot * kw);
    }
}

/* concatenation (bitstring.cpp:42-47) of s blocks of k bits each */
static void concat_blocks(const uint64_t* blocks, uint32_t s, uint64_t k, uint64_t* out_key) {
    const uint64_t kw = (k + 63) / 64;
    const uint64_t total_words = ((uint64_t)s * k + 63) / 64;
    memset(out_key, 0, total_words * 8);
    for (uint32_t j = 0; j < s; ++j)
        or_xor_bit_range(out_key, total_words, (uint64_t)j * k, blocks + (uint64_t)j * kw, kw, 0, k);
}

int or_extract(const uint64_t* input, uint64_t n, uint32_t s, const uint64_t samp_key[4],
               const uint64_t hash_key[4], int per_block_seed, uint64_t k, uint64_t* out_key,
               uint64_t* out_nj, int nthreads) {
    return or_extract_sifted(input, NULL, n, s, samp_key, hash_key, per_block_seed, k, out_key,
                             out_nj, nthreads);
}

/* run_extraction's sift + hash loop (pipeline.cpp:109-136): keep_in (1 byte per round,
 * NULL = all kept) selects the rounds that join their sub-block. */
int or_extract_sifted(const uint64_t* input, const uint8_t* keep_in, uint64_t n, uint32_t s,
                      const uint64_t samp_key[4], const uint64_t hash_key[4], int per_block_seed,
                      uint64_t k, uint64_t* out_key, uint64_t* out_nj, int nthreads) {
    if (s == 0 || k == 0) return -1;
    uint32_t* assignment = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
    uint64_t* raw = (uint64_t*)malloc(sizeof(uint64_t) * s);
    or_assign_subblocks(n, s, samp_key, assignment, raw, nthreads);
    uint8_t* keep = (uint8_t*)malloc(n ? n : 1);
    if (keep_in)
        memcpy(keep, keep_in, n);
    else
        memset(keep, 1, n);
    uint64_t* offsets = (uint64_t*)malloc(sizeof(uint64_t) * ((size_t)s + 1));
    uint64_t* indices = (uint64_t*)malloc(sizeof(uint64_t) * (n ? n : 1));
    or_sift_partition(keep, n, assignment, s, offsets, indices);
    free(keep);
    free(assignment);
    int rc = 0;
    for (uint32_t j = 0; j < s; ++j) {
        out_nj[j] = offsets[j + 1] - offsets[j];
        if (out_nj[j] == 0) rc = -1;
    }
    if (rc == 0) {
        const uint64_t kw = (k + 63) / 64;
        uint64_t* blocks = (uint64_t*)calloc((size_t)s * kw, 8);
        hash_ctx c = {input, s, hash_key, per_block_seed, k, offsets, indices, blocks,
                      or_tag("hash-seed"), NULL};
        parallel_ranges(s, 1, nthreads, hash_range, &c);
        concat_blocks(blocks, s, k, out_key);
        free(blocks);
    }
    free(raw);
    free(offsets);
    free(indices);
    return rc;
}

/* ------------------------------------------------ streaming extraction */

typedef struct {
    uint64_t n;
    uint32_t s;
    const uint64_t* key;
    uint64_t tag;
    const int32_t* slot_of; /* s entries: -1 or slot in `which` */
    uint64_t* counts;       /* nthreads x s */
    uint64_t** lists;       /* nthreads x nwhich growable index lists */
    uint64_t* lens;         /* nthreads x nwhich */
    uint64_t* caps;
    uint32_t nwhich;
} scan_ctx;

static void scan_range(void* vc, uint64_t lo, uint64_t hi, int tid) {
    scan_ctx* c = (scan_ctx*)vc;
    uint64_t* cnt = c->counts + (uint64_t)tid * c->s;
    for (uint64_t i = lo; i < hi; ++i) {
        const uint32_t v = (uint32_t)or_uniform_below(c->key, c->tag, 0, c->s, i);
        ++cnt[v];
        const int32_t slot = c->slot_of[v];
        if (slot >= 0) {
            const uint64_t li = (uint64_t)tid * c->nwhich + (uint64_t)slot;
            if (c->lens[li] == c->caps[li]) {
                c->caps[li] = c->caps[li] ? c->caps[li] * 2 : 1024;
                c->lists[li] = (uint64_t*)realloc(c->lists[li], c->caps[li] * 8);
            }
            c->lists[li][c->lens[li]++] = i;
        }
    }
}

int or_extract_selected(const uint64_t* input, uint64_t n, uint32_t s,
                        const uint64_t samp_key[4], const uint64_t hash_key[4],
                        int per_block_seed, uint64_t k, const uint32_t* which, uint32_t nwhich,
                        uint64_t* out_keys, uint64_t* out_nj, int nthreads) {
    if (s == 0 || k == 0) return -1;
    nthreads = resolve_threads(nthreads);
    if (nthreads > 512) nthreads = 512;
    int32_t* slot_of = (int32_t*)malloc(sizeof(int32_t) * s);
    for (uint32_t j = 0; j < s; ++j) slot_of[j] = -1;
    for (uint32_t q = 0; q < nwhich; ++q) slot_of[which[q]] = (int32_t)q;
    const size_t nl = (size_t)nthreads * nwhich;
    scan_ctx c = {n, s, samp_key, or_tag("sampling"), slot_of,
                  (uint64_t*)calloc((size_t)nthreads * s, 8),
                  (uint64_t**)calloc(nl ? nl : 1, sizeof(uint64_t*)),
                  (uint64_t*)calloc(nl ? nl : 1, 8), (uint64_t*)calloc(nl ? nl : 1, 8), nwhich};
    /* contiguous per-thread ranges in thread order => concatenation keeps round order */
    parallel_ranges(n, 64, nthreads, scan_range, &c);
    for (uint32_t j = 0; j < s; ++j) {
        uint64_t t = 0;
        for (int q = 0; q < nthreads; ++q) t += c.counts[(uint64_t)q * s + j];
        out_nj[j] = t;
    }
    uint64_t* offsets = (uint64_t*)malloc(8 * ((size_t)nwhich + 1));
    offsets[0] = 0;
    for (uint32_t q = 0; q < nwhich; ++q) offsets[q + 1] = offsets[q] + out_nj[which[q]];
    uint64_t* indices = (uint64_t*)malloc(8 * (offsets[nwhich] ? offsets[nwhich] : 1));
    for (uint32_t q = 0; q < nwhich; ++q) {
        uint64_t pos = offsets[q];
        for (int t = 0; t < nthreads; ++t) {
            const uint64_t li = (uint64_t)t * nwhich + q;
            if (c.lens[li]) memcpy(indices + pos, c.lists[li], c.lens[li] * 8);
            pos += c.lens[li];
            free(c.lists[li]);
        }
    }
    int rc = 0;
    for (uint32_t q = 0; q < nwhich; ++q)
        if (out_nj[which[q]] == 0) rc = -1;
    if (rc == 0) {
        hash_ctx h = {input, s, hash_key, per_block_seed, k, offsets, indices, out_keys,
                      or_tag("hash-seed"), which};
        parallel_ranges(nwhich, 1, nthreads, hash_range, &h);
    }
    free(indices);
    free(offsets);
    free(c.counts);
    free(c.lists);
    free(c.lens);
    free(c.caps);
    free(slot_of);
    return rc;
}

/* ----------------------------------------------------------- utilities */

uint64_t or_fnv_words(const uint64_t* w, uint64_t nwords) {
    uint64_t h = 0xcbf29ce484222325ull;
    for (uint64_t i = 0; i < nwords; ++i)
        for (unsigned b = 0; b < 8; ++b) {
            h ^= (w[i] >> (8 * b)) & 0xff;
            h *= 0x100000001b3ull;
        }
    return h;
}

void or_seed_from_int(uint64_t v, uint64_t key[4]) {
    key[0] = 0;
    key[1] = 0;
    key[2] = 0;
    key[3] = v;
}

/* ------------------------------------------------------------- protocol rounds */

typedef struct {
    const uint64_t* key;
    uint64_t n;
    double p_x, e_ph, e_bit, p_det;
    uint64_t t_a, t_b, t_det, t_bit, t_noise;
    uint8_t* out;
} rounds_ctx;

/* pipeline.cpp:31-53, one round at a time */
static void rounds_range(void* arg, uint64_t lo, uint64_t hi, int tid) {
    (void)tid;
    const rounds_ctx* c = (const rounds_ctx*)arg;
    for (uint64_t i = lo; i < hi && i < c->n; ++i) {
        uint8_t r = 0;
        const int ax = or_bernoulli(c->key, c->t_a, 0, c->p_x, i) == 1;
        const int bx = or_bernoulli(c->key, c->t_b, 0, c->p_x, i) == 1;
        if (ax) r |= 1;
        if (bx) r |= 2;
        if (ax && bx) r |= 32;
        if (or_bernoulli(c->key, c->t_det, 0, c->p_det, i) == 1) {
            r |= 4;
            const uint64_t w = or_stream_word(c->key, c->t_bit, 0, i);
            const int a = (int)(w & 1);
            int b;
            if (ax == bx)
                b = a ^ (or_bernoulli(c->key, c->t_noise, 0, ax ? c->e_ph : c->e_bit, i) == 1);
            else
                b = (int)((w >> 1) & 1);
            if (a) r |= 8;
            if (b) r |= 16;
        }
        c->out[i] = r;
    }
}

void or_simulate_rounds(uint64_t n, double p_x, double e_ph, double e_bit, double p_det,
                        const uint64_t key[4], uint8_t* out, int nthreads) {
    if (n == 0) return;
    rounds_ctx c = {key, n, p_x, e_ph, e_bit, p_det, or_tag("basis-a"), or_tag("basis-b"),
                    or_tag("detect"), or_tag("bit-a"), or_tag("noise"), out};
    parallel_ranges(n, 1, nthreads, rounds_range, &c);
}

void or_rounds_split(const uint8_t* rounds, uint64_t n, uint64_t* bits, uint8_t* keep,
                     uint64_t counts[4]) {
    memset(bits, 0, sizeof(uint64_t) * ((n + 63) / 64));
    counts[0] = counts[1] = counts[2] = counts[3] = 0;
    for (uint64_t i = 0; i < n; ++i) {
        const uint8_t r = rounds[i];
        const int det = (r >> 2) & 1, a = (r >> 3) & 1, b = (r >> 4) & 1, test = (r >> 5) & 1;
        if (a) bits[i >> 6] |= 1ull << (i & 63);
        keep[i] = det && !(r & 1) && !(r & 2);
        if (test) {
            ++counts[0];
            if (!det)
                ++counts[2];
            else if (a != b)
                ++counts[1];
        }
        counts[3] += keep[i];
    }
}

/* ------------------------------------------- whole-partition checker (configs 4-5) */
/* Eight consecutive sampling draws V_i = uniform_below(s, i) for a power-of-two s
 * (prf.cpp:87-88: block({tag, 0, i, 0})[0] & (s-1)), written lane-parallel so that the
 * compiler vectorises the 64-bit Threefry rounds (prf.cpp:47-76); target_clones picks the
 * AVX-512 / AVX2 body on the host it runs on. Same arithmetic as or_threefry. */
__attribute__((target_clones("avx512f", "avx2", "default")))
static void sample8(const uint64_t ks[5], uint64_t tag, uint64_t i0, uint64_t mask,
                    uint32_t v[8]) {
    static const unsigned rot[8][2] = {{14, 16}, {52, 57}, {23, 40}, {5, 37},
                                       {25, 33}, {46, 12}, {58, 22}, {32, 32}};
    uint64_t x0[8], x1[8], x2[8], x3[8];
    for (int l = 0; l < 8; ++l) {
        x0[l] = tag + ks[0];
        x1[l] = ks[1];
        x2[l] = i0 + (uint64_t)l + ks[2];
        x3[l] = ks[3];
    }
#pragma GCC unroll 20
    for (unsigned d = 0; d < 20; ++d) {
        const unsigned r0 = rot[d & 7][0], r1 = rot[d & 7][1];
        for (int l = 0; l < 8; ++l) {
            x0[l] += x1[l];
            const uint64_t a = ((x1[l] << r0) | (x1[l] >> (64 - r0))) ^ x0[l];
            x2[l] += x3[l];
            const uint64_t b = ((x3[l] << r1) | (x3[l] >> (64 - r1))) ^ x2[l];
            x1[l] = b; /* x1 <-> x3 swap */
            x3[l] = a;
        }
        if ((d & 3) == 3) {
            const uint64_t sidx = d / 4 + 1;
            for (int l = 0; l < 8; ++l) {
                x0[l] += ks[sidx % 5];
                x1[l] += ks[(sidx + 1) % 5];
                x2[l] += ks[(sidx + 2) % 5];
                x3[l] += ks[(sidx + 3) % 5] + sidx;
            }
        }
    }
    for (int l = 0; l < 8; ++l) v[l] = (uint32_t)(x0[l] & mask);
}

typedef struct {
    const uint64_t* input;
    uint64_t n;
    uint32_t s;
    const uint64_t* key;
    uint64_t ks[5];
    uint64_t tag;
    uint64_t* counts; /* nthreads x s: pass 1 counts, then each thread's starting ranks */
    const uint64_t* nj;
    const uint64_t* yoff;
    uint64_t* y;
    int pass;
} part_ctx;

static void part_range(void* vc, uint64_t lo, uint64_t hi, int tid) {
    part_ctx* c = (part_ctx*)vc;
    uint64_t* rank = c->counts + (uint64_t)tid * c->s;
    const int pow2 = (c->s & (c->s - 1)) == 0;
    uint32_t v[8];
    for (uint64_t i = lo; i < hi; i += 8) {
        const unsigned cnt = hi - i < 8 ? (unsigned)(hi - i) : 8u;
        if (pow2 && cnt == 8)
            sample8(c->ks, c->tag, i, c->s - 1, v);
        else
            for (unsigned l = 0; l < cnt; ++l)
                v[l] = (uint32_t)or_uniform_below(c->key, c->tag, 0, c->s, i + l);
        for (unsigned l = 0; l < cnt; ++l) {
            const uint32_t j = v[l];
            const uint64_t r = rank[j]++;
            if (c->pass == 2 && ((c->input[(i + l) >> 6] >> ((i + l) & 63)) & 1)) {
                const uint64_t pos = c->nj[j] - 1 - r; /* reversed: y[c] = x_j[n_j-1-c] */
                __atomic_fetch_or(&c->y[c->yoff[j] + (pos >> 6)], 1ull << (pos & 63),
                                  __ATOMIC_RELAXED);
            }
        }
    }
}

/* assign_subblocks + sift (all kept) + gather of EVERY block without materialising the
 * 12 B/round Partition (sampling.cpp:10-39, ssbh_main.cpp:329-331): two passes of the
 * sampling draw over contiguous per-thread round ranges (counts, then the bits placed at
 * their in-block rank). Block j's input is written REVERSED (bit c = x_j[n_j-1-c]) at u64
 * word yoff[j]; y must hold n/64 + s + 1 zeroed words. */
int or_partition_reversed(const uint64_t* input, uint64_t n, uint32_t s, const uint64_t key[4],
                          int nthreads, uint64_t* nj, uint64_t* yoff, uint64_t* y) {
    if (s == 0) return -1;
    nthreads = resolve_threads(nthreads);
    if (nthreads > 512) nthreads = 512;
    part_ctx c;
    memset(&c, 0, sizeof c);
    c.input = input;
    c.n = n;
    c.s = s;
    c.key = key;
    for (int q = 0; q < 4; ++q) c.ks[q] = key[q];
    c.ks[4] = 0x1BD11BDAA9FC1A22ull ^ key[0] ^ key[1] ^ key[2] ^ key[3];
    c.tag = or_tag("sampling");
    c.counts = (uint64_t*)calloc((size_t)nthreads * s, 8);
    c.pass = 1;
    parallel_ranges(n, 64, nthreads, part_range, &c);
    yoff[0] = 0;
    for (uint32_t j = 0; j < s; ++j) {
        uint64_t t = 0;
        for (int q = 0; q < nthreads; ++q) {
            const uint64_t v = c.counts[(uint64_t)q * s + j];
            c.counts[(uint64_t)q * s + j] = t; /* thread q's first rank in block j */
            t += v;
        }
        nj[j] = t;
        yoff[j + 1] = yoff[j] + (t + 63) / 64;
    }
    c.nj = nj;
    c.yoff = yoff;
    c.y = y;
    c.pass = 2;
    parallel_ranges(n, 64, nthreads, part_range, &c);
    free(c.counts);
    return 0;
}

typedef struct {
    const uint64_t* y;
    const uint64_t* yoff;
    const uint64_t* nj;
    const uint64_t* hash_key;
    int per_block;
    uint64_t k;
    const uint64_t* key;
    uint32_t rows;
    uint64_t row_seed;
    const uint64_t* shared_seed; /* shared mode: one seed for every block (prefix-stable) */
    uint64_t seed_words;         /* padded words of a seed buffer */
    uint64_t tag;
    uint64_t* bad;     /* per thread: mismatches */
    uint64_t* first;   /* per thread: first mismatching block (or ~0) */
} spot_ctx;

static inline uint64_t splitmix64(uint64_t z) {
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

static void spot_range(void* vc, uint64_t lo, uint64_t hi, int tid) {
    spot_ctx* c = (spot_ctx*)vc;
    uint64_t* buf = c->per_block ? (uint64_t*)malloc(c->seed_words * 8) : NULL;
    for (uint64_t j = lo; j < hi; ++j) {
        const uint64_t n = c->nj[j];
        if (n == 0) continue;
        const uint64_t* seed = c->shared_seed;
        if (c->per_block) { /* KeyedStream(hash, "hash-seed", j).bits(k + n - 1), zero padded */
            memset(buf, 0, c->seed_words * 8);
            or_stream_bits(c->hash_key, c->tag, j, c->k + n - 1, buf);
            seed = buf;
        }
        const uint64_t* yr = c->y + c->yoff[j];
        const uint64_t yw = (n + 63) / 64;
        for (uint32_t q = 0; q < c->rows; ++q) {
            /* rows 0 and k-1, then seeded rows */
            const uint64_t i = q == 0 ? 0 : q == 1 ? c->k - 1
                                                   : splitmix64(c->row_seed ^ (j << 20) ^ q) % c->k;
            uint64_t acc = 0; /* K[i] = parity(S[i .. i+n) & y), toeplitz.cpp:34-52 reversed */
            for (uint64_t w = 0; w < yw; ++w) {
                const uint64_t bit = i + 64 * w, qw = bit >> 6;
                const unsigned r = (unsigned)(bit & 63);
                uint64_t win = seed[qw] >> r;
                if (r) win |= seed[qw + 1] << (64 - r);
                acc ^= win & yr[w];
            }
            const uint64_t kb = j * c->k + i;
            const unsigned got = (unsigned)((c->key[kb >> 6] >> (kb & 63)) & 1);
            if ((unsigned)(__builtin_popcountll(acc) & 1) != got) {
                if (c->bad[tid]++ == 0) c->first[tid] = j;
            }
        }
    }
    free(buf);
}

/* Every block's sampled output rows recomputed from the definition (toeplitz.cpp:34-52 with
 * the seed of pipeline.cpp:132 / KeyedStream::bits prf.cpp:104-115) and compared with the
 * concatenated key (bitstring.cpp:42-47; block j at bits [j k, (j+1) k)). Returns the number
 * of mismatching rows; *first_bad = the first block with one (or ~0). */
uint64_t or_spot_check(const uint64_t* y, const uint64_t* yoff, const uint64_t* nj, uint32_t s,
                       const uint64_t hash_key[4], int per_block, uint64_t k,
                       const uint64_t* key, uint32_t rows, uint64_t row_seed, int nthreads,
                       uint64_t* first_bad) {
    nthreads = resolve_threads(nthreads);
    if (nthreads > 512) nthreads = 512;
    uint64_t maxn = 0;
    for (uint32_t j = 0; j < s; ++j) maxn = nj[j] > maxn ? nj[j] : maxn;
    spot_ctx c;
    memset(&c, 0, sizeof c);
    c.y = y;
    c.yoff = yoff;
    c.nj = nj;
    c.hash_key = hash_key;
    c.per_block = per_block;
    c.k = k;
    c.key = key;
    c.rows = rows;
    c.row_seed = row_seed;
    c.tag = or_tag("hash-seed");
    c.seed_words = (k + maxn + 63) / 64 + 2;
    uint64_t* shared = NULL;
    if (!per_block) { /* prefix-stable: block j uses the first k + n_j - 1 bits */
        shared = (uint64_t*)calloc(c.seed_words, 8);
        or_stream_bits(hash_key, c.tag, 0, k + maxn - 1, shared);
        c.shared_seed = shared;
    }
    c.bad = (uint64_t*)calloc(512, 8);
    c.first = (uint64_t*)malloc(512 * 8);
    for (int t = 0; t < 512; ++t) c.first[t] = ~0ull;
    parallel_ranges(s, 1, nthreads, spot_range, &c);
    uint64_t bad = 0, fb = ~0ull;
    for (int t = 0; t < 512; ++t) {
        bad += c.bad[t];
        if (c.first[t] < fb) fb = c.first[t];
    }
    if (first_bad) *first_bad = fb;
    free(shared);
    free(c.bad);
    free(c.first);
    return bad;
}
