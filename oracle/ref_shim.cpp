// ref_shim.cpp — extern "C" shim over the UNMODIFIED reference C++ API.
// TEST / BASELINE INFRASTRUCTURE ONLY. Compiled by oracle/Makefile together with the
// reference sources where they lie (/root/reference/proj/src/{bitstring,prf,sampling,
// toeplitz,pipeline,bbm92,geat}.cpp) into oracle/_ref/libssbh_ref.so. Nothing of the reference is copied
// into this repository; this file only calls its public API (proj/include/ssbh/*.hpp)
// and its thread pool (proj/src/parallel.hpp:13-41).
//
// Used to (1) pin the C restatement in oracle.c, (2) generate tests/golden/ fixtures,
// (3) time the reference CPU path for bench.py (--impl reference / cpu_baseline).
#include <chrono>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <thread>
#include <vector>

#include "parallel.hpp"  // proj/src/parallel.hpp
#include "ssbh/bitstring.hpp"
#include "ssbh/bbm92.hpp"
#include "ssbh/errors.hpp"
#include "ssbh/pipeline.hpp"
#include "ssbh/prf.hpp"
#include "ssbh/sampling.hpp"
#include "ssbh/toeplitz.hpp"

using namespace ssbh;

namespace {

MasterSeed seed_of(const uint64_t k[4]) {
    MasterSeed s;
    for (int i = 0; i < 4; ++i) s.words[i] = k[i];
    return s;
}

BitString from_words(const uint64_t* w, uint64_t nbits) {
    BitString b(nbits);
    auto dst = b.words();
    if (!dst.empty()) std::memcpy(dst.data(), w, dst.size() * 8);
    // re-establish the zero tail through the public API
    std::vector<std::uint8_t> bytes = b.to_bytes();
    return BitString::from_bytes(bytes, nbits);
}

void to_words(const BitString& b, uint64_t* out) {
    auto w = b.words();
    if (!w.empty()) std::memcpy(out, w.data(), w.size() * 8);
}

int code_of_current() {
    try {
        throw;
    } catch (const std::invalid_argument&) {
        return 1;
    } catch (const infeasible_error&) {
        return 2;
    } catch (const std::overflow_error&) {
        return 3;
    } catch (const io_error&) {
        return 4;
    } catch (...) {
        return 9;
    }
}

}  // namespace

extern "C" {

void ref_prf_block(const uint64_t key[4], const uint64_t ctr[4], uint64_t out[4]) {
    const auto r = prf::block({key[0], key[1], key[2], key[3]}, {ctr[0], ctr[1], ctr[2], ctr[3]});
    for (int i = 0; i < 4; ++i) out[i] = r[i];
}

uint64_t ref_tag(const char* purpose) { return prf::tag(purpose); }

uint64_t ref_stream_word(const uint64_t key[4], const char* purpose, uint64_t sub, uint64_t i) {
    return KeyedStream(seed_of(key), purpose, sub).word(i);
}

int ref_uniform_below(const uint64_t key[4], const char* purpose, uint64_t sub, uint64_t bound,
                      uint64_t i, uint64_t* out) {
    try {
        *out = KeyedStream(seed_of(key), purpose, sub).uniform_below(bound, i);
        return 0;
    } catch (...) {
        return code_of_current();
    }
}

int ref_bernoulli(const uint64_t key[4], const char* purpose, uint64_t sub, double p, uint64_t i) {
    try {
        return KeyedStream(seed_of(key), purpose, sub).bernoulli(p, i) ? 1 : 0;
    } catch (...) {
        return -code_of_current();
    }
}

void ref_stream_bits(const uint64_t key[4], const char* purpose, uint64_t sub, uint64_t nbits,
                     uint64_t* out) {
    to_words(KeyedStream(seed_of(key), purpose, sub).bits(nbits), out);
}

int ref_assign_subblocks(uint64_t n, uint32_t s, const uint64_t key[4], uint32_t* assignment,
                         uint64_t* raw_counts) {
    try {
        const Partition p = assign_subblocks(n, s, seed_of(key));
        std::memcpy(assignment, p.assignment.data(), n * 4);
        std::memcpy(raw_counts, p.raw_counts.data(), (size_t)s * 8);
        return 0;
    } catch (...) {
        return code_of_current();
    }
}

// CSR output: offsets[s+1], indices[total kept]
int ref_sift_partition(const uint8_t* keep, uint64_t n, const uint32_t* assignment, uint32_t s,
                       uint64_t* offsets, uint64_t* indices, uint64_t* max_len) {
    try {
        Partition p;
        p.n_subblocks = s;
        p.assignment.assign(assignment, assignment + n);
        p.raw_counts.assign(s, 0);
        for (uint64_t i = 0; i < n; ++i) ++p.raw_counts[assignment[i] - 1];
        const SiftedPartition sp = sift_partition(std::span<const uint8_t>(keep, n), p);
        offsets[0] = 0;
        for (uint32_t j = 0; j < s; ++j) {
            std::memcpy(indices + offsets[j], sp.blocks[j].data(), sp.blocks[j].size() * 8);
            offsets[j + 1] = offsets[j] + sp.blocks[j].size();
        }
        *max_len = sp.max_len;
        return 0;
    } catch (...) {
        return code_of_current();
    }
}

int ref_toeplitz_hash(const uint64_t* seed, uint64_t m, uint64_t n, const uint64_t* input,
                      uint64_t nin, uint64_t* out) {
    try {
        const ToeplitzSeed ts(from_words(seed, m + n - 1), m, n);
        to_words(toeplitz_hash(ts, from_words(input, nin)), out);
        return 0;
    } catch (...) {
        return code_of_current();
    }
}

int ref_blocked_toeplitz_hash(const uint64_t* seed, uint64_t m, uint64_t n,
                              const uint64_t* input, uint64_t nin, uint64_t mp, uint64_t np,
                              uint64_t* out) {
    try {
        const ToeplitzSeed ts(from_words(seed, m + n - 1), m, n);
        to_words(blocked_toeplitz_hash(ts, from_words(input, nin), BlockingParams{mp, np}), out);
        return 0;
    } catch (...) {
        return code_of_current();
    }
}

uint64_t ref_block_limit(uint64_t n, double p, double eps, uint64_t m_blocks, int* err) {
    try {
        *err = 0;
        return block_limit(n, p, eps, m_blocks);
    } catch (...) {
        *err = code_of_current();
        return 0;
    }
}

double ref_binomial_tail_bound(uint64_t n, uint64_t limit, double p) {
    return binomial_tail_bound(n, limit, p);
}

uint64_t ref_cycle_estimate(uint64_t in, uint64_t out, uint64_t mp, int* err) {
    try {
        *err = 0;
        return cycle_estimate(in, out, mp);
    } catch (...) {
        *err = code_of_current();
        return 0;
    }
}

// File-mode extraction (ssbh_main.cpp:306-345) with distinct sampling / hash seeds,
// blocks hashed with the reference's parallel_for (slot-indexed, order-independent),
// then concatenated in block order with BitString::append.
int ref_extract(const uint64_t* input, uint64_t n, uint32_t s, const uint64_t samp[4],
                const uint64_t hash[4], int per_block, uint64_t k, uint64_t* out_key,
                uint64_t* out_nj) {
    try {
        const BitString data = from_words(input, n);
        const Partition part = assign_subblocks(n, s, seed_of(samp));
        const std::vector<std::uint8_t> keep(n, 1);
        const SiftedPartition sifted = sift_partition(keep, part);
        for (uint32_t j = 0; j < s; ++j) out_nj[j] = sifted.blocks[j].size();
        std::vector<BitString> outs(s);
        const MasterSeed hs = seed_of(hash);
        detail::parallel_for(s, [&](std::size_t j) {
            BitString x(sifted.blocks[j].size());
            for (uint64_t q = 0; q < sifted.blocks[j].size(); ++q)
                if (data.get(sifted.blocks[j][q])) x.set(q, true);
            const KeyedStream st(hs, "hash-seed", per_block ? j : 0);
            const ToeplitzSeed ts(st.bits(k + x.size() - 1), k, x.size());
            outs[j] = toeplitz_hash(ts, x);
        });
        BitString key;
        for (uint32_t j = 0; j < s; ++j) key.append(outs[j]);
        to_words(key, out_key);
        return 0;
    } catch (...) {
        return code_of_current();
    }
}

// Streaming form of the file-mode extraction for sizes whose Partition cannot be held in
// memory: every round's V_i from the reference's own
// KeyedStream::uniform_below (contiguous per-thread index ranges, concatenated in thread
// order = round order), all n_j counted, the rounds of the `which` blocks gathered; those
// blocks hashed with the reference's KeyedStream::bits + ToeplitzSeed + toeplitz_hash.
int ref_extract_selected(const uint64_t* input, uint64_t n, uint32_t s, const uint64_t samp[4],
                         const uint64_t hash[4], int per_block, uint64_t k, const uint32_t* which,
                         uint32_t nwhich, uint64_t* out_keys, uint64_t* out_nj) {
    try {
        const KeyedStream st(seed_of(samp), "sampling");
        std::vector<int32_t> slot(s, -1);
        for (uint32_t q = 0; q < nwhich; ++q) slot[which[q]] = (int32_t)q;
        const std::size_t hw = std::max(1u, std::thread::hardware_concurrency());
        const uint64_t per = (n + hw - 1) / hw;
        std::vector<std::vector<uint64_t>> counts(hw, std::vector<uint64_t>(s, 0));
        std::vector<std::vector<std::vector<uint64_t>>> lists(
            hw, std::vector<std::vector<uint64_t>>(nwhich));
        detail::parallel_for(hw, [&](std::size_t t) {
            const uint64_t lo = t * per, hi = std::min(n, lo + per);
            for (uint64_t i = lo; i < hi; ++i) {
                const uint64_t v = st.uniform_below(s, i);
                ++counts[t][v];
                if (slot[v] >= 0) lists[t][slot[v]].push_back(i);
            }
        });
        for (uint32_t j = 0; j < s; ++j) {
            uint64_t c = 0;
            for (std::size_t t = 0; t < hw; ++t) c += counts[t][j];
            out_nj[j] = c;
        }
        const uint64_t kw = (k + 63) / 64;
        detail::parallel_for(nwhich, [&](std::size_t q) {
            std::vector<uint64_t> idx;
            for (std::size_t t = 0; t < hw; ++t)
                idx.insert(idx.end(), lists[t][q].begin(), lists[t][q].end());
            BitString x(idx.size());
            for (uint64_t r = 0; r < idx.size(); ++r)
                if ((input[idx[r] >> 6] >> (idx[r] & 63)) & 1) x.set(r, true);
            const KeyedStream hs(seed_of(hash), "hash-seed", per_block ? which[q] : 0);
            const ToeplitzSeed ts(hs.bits(k + x.size() - 1), k, x.size());
            to_words(toeplitz_hash(ts, x), out_keys + q * kw);
        });
        return 0;
    } catch (...) {
        return code_of_current();
    }
}

// Bounded CPU sample of the reference hot path for bench.py (cpu_baseline and
// --impl reference): assign_subblocks over `n_sample` rounds (the shipped, single-threaded
// sampler) + gather + toeplitz_hash of `nblocks` sub-blocks of that partition's shape
// (each of length ~n/s drawn from the real sampler on a prefix), run on all host threads
// with the reference's parallel_for. Returns the wall seconds; *bits_hashed = sum n_j.
double ref_time_sample(uint64_t n_sample, uint32_t s_sample, uint64_t k, double p,
                       const uint64_t in_key[4], const uint64_t samp[4], const uint64_t hash[4],
                       uint32_t nblocks, uint64_t* bits_hashed, uint64_t* digest) {
    const MasterSeed is = seed_of(in_key), ss = seed_of(samp), hs = seed_of(hash);
    // synthetic input (not timed): SURVEY §8a convention
    const KeyedStream in(is, "input");
    BitString data = p == 0.5 ? in.bits(n_sample) : BitString(n_sample);
    if (p != 0.5)
        for (uint64_t i = 0; i < n_sample; ++i)
            if (in.bernoulli(p, i)) data.set(i, true);
    const auto t0 = std::chrono::steady_clock::now();
    const Partition part = assign_subblocks(n_sample, s_sample, ss);
    const std::vector<std::uint8_t> keep(n_sample, 1);
    const SiftedPartition sifted = sift_partition(keep, part);
    std::vector<BitString> outs(nblocks);
    detail::parallel_for(nblocks, [&](std::size_t q) {
        const auto& idx = sifted.blocks[q % s_sample];
        BitString x(idx.size());
        for (uint64_t t = 0; t < idx.size(); ++t)
            if (data.get(idx[t])) x.set(t, true);
        const KeyedStream st(hs, "hash-seed", 0);
        const ToeplitzSeed ts(st.bits(k + x.size() - 1), k, x.size());
        outs[q] = toeplitz_hash(ts, x);
    });
    BitString key;
    for (auto& o : outs) key.append(o);
    const double secs =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    uint64_t bits = 0;
    for (uint32_t q = 0; q < nblocks; ++q) bits += sifted.blocks[q % s_sample].size();
    *bits_hashed = bits;
    uint64_t h = 0xcbf29ce484222325ull;
    for (uint64_t w : key.words())
        for (int b = 0; b < 8; ++b) {
            h ^= (w >> (8 * b)) & 0xff;
            h *= 0x100000001b3ull;
        }
    *digest = h;
    return secs;
}

// ---- protocol rounds / run_extraction (pipeline.hpp:41-99) ------------------------------
// Flat parameter block for ctypes; the remaining Bbm92Params fields keep their defaults.
struct ref_bbm92 {
    uint64_t n_rounds;
    double p_x, e_ph, e_bit, q_tol, eta_tol, f_ec, p_det, eps_sec, eps_abort;
};

static Bbm92Params params_of(const ref_bbm92* r) {
    Bbm92Params p;
    p.n_rounds = r->n_rounds;
    p.p_x = r->p_x;
    p.e_ph = r->e_ph;
    p.e_bit = r->e_bit;
    p.q_tol = r->q_tol;
    p.eta_tol = r->eta_tol;
    p.f_ec = r->f_ec;
    p.p_det = r->p_det;
    p.eps_sec = r->eps_sec;
    p.eps_abort = r->eps_abort;
    return p;
}

int ref_simulate_rounds(const ref_bbm92* rp, const uint64_t seed[4], uint8_t* out) {
    try {
        const auto rounds = simulate_rounds(params_of(rp), seed_of(seed));
        for (std::size_t i = 0; i < rounds.size(); ++i) out[i] = rounds[i].raw;
        return 0;
    } catch (...) {
        return code_of_current();
    }
}

// key_length(params, ns == 1 ? full : splitting(ns)) as run_extraction sizes it
// (pipeline.cpp:115-117).
int ref_key_length(const ref_bbm92* rp, uint32_t ns, uint64_t* length, int* feasible) {
    try {
        const KeyLengthResult kl =
            key_length(params_of(rp), ns == 1 ? Scenario::full() : Scenario::splitting(ns));
        *length = kl.length;
        *feasible = kl.feasible;
        return 0;
    } catch (...) {
        return code_of_current();
    }
}

// The reference's plan_for (test_pipeline.cpp:27-35 / ssbh_main.cpp:276-282): block_limit of
// the sifting probability p_z^2 p_det / ns.
int ref_plan_block_limit(const ref_bbm92* rp, uint32_t ns, uint64_t* limit) {
    try {
        const Bbm92Params p = params_of(rp);
        const double p_sift = p.p_z() * p.p_z() * p.p_det / static_cast<double>(ns);
        *limit = block_limit(p.n_rounds, p_sift, p.eps_abort, ns);
        return 0;
    } catch (...) {
        return code_of_current();
    }
}

// run_extraction (pipeline.cpp:75-138) on caller rounds. out_key capacity key_cap_words;
// meta = {abort, bits_per_block, key bits, cycle_count, block_lengths count};
// dmeta = {total_epsilon, wall_seconds}.
int ref_run_extraction(const uint8_t* rounds_raw, const ref_bbm92* rp, uint32_t ns,
                       uint64_t block_limit_, const uint64_t seed[4], uint64_t m_prime,
                       uint64_t* out_key, uint64_t key_cap_words, uint64_t* out_lengths,
                       uint64_t meta[5], double dmeta[2]) {
    try {
        const Bbm92Params p = params_of(rp);
        std::vector<RoundRecord> rounds(p.n_rounds);
        for (uint64_t i = 0; i < p.n_rounds; ++i) rounds[i].raw = rounds_raw[i];
        SamplingPlan plan;
        plan.n_subblocks = ns;
        plan.eps_abort = p.eps_abort;
        plan.block_limit = block_limit_;
        plan.seed = seed_of(seed);
        BlockingParams blk;
        blk.m_prime = m_prime;
        const ExtractionReport rep = run_extraction(rounds, plan, p, blk);
        meta[0] = static_cast<uint64_t>(rep.abort);
        meta[1] = rep.bits_per_block;
        meta[2] = rep.key.size();
        meta[3] = rep.cycle_count;
        meta[4] = rep.block_lengths.size();
        dmeta[0] = rep.total_epsilon;
        dmeta[1] = rep.wall_seconds;
        if ((rep.key.size() + 63) / 64 > key_cap_words) return 8;
        to_words(rep.key, out_key);
        for (std::size_t j = 0; j < rep.block_lengths.size(); ++j)
            out_lengths[j] = rep.block_lengths[j];
        return 0;
    } catch (...) {
        return code_of_current();
    }
}

// timing_model (pipeline.hpp:60-62, pipeline.cpp:139-160). kind: 0 full, 1 splitting,
// 2 small-block.
int ref_timing_model(uint64_t input_len, uint64_t output_len, int kind, uint32_t ns,
                     uint64_t m_prime, double eps_abort, uint64_t limit_override, int pad,
                     uint64_t* out) {
    try {
        const Scenario sc = kind == 0   ? Scenario::full()
                            : kind == 1 ? Scenario::splitting(ns)
                                        : Scenario::small_block(ns);
        BlockingParams blk;
        blk.m_prime = m_prime;
        *out = timing_model(input_len, output_len, sc, blk, eps_abort, limit_override, pad != 0);
        return 0;
    } catch (...) {
        return code_of_current();
    }
}

}  // extern "C"
