// ssbh_api.cpp — the reference's C++ API (include/ssbh/*.hpp) as a drop-in over the C-ABI
// (include/ssbh_cuda.h). Container operations on BitString and the scalar PRF draws are
// host code; sampling, bulk bit streams, hashing and the fused extraction call the sm_100a
// kernels. C-ABI statuses are rethrown as the reference's exception types.
#include <algorithm>
#include <bit>
#include <cstdio>
#include <cstring>
#include <memory>

#include "ssbh/bitstring.hpp"
#include "ssbh/errors.hpp"
#include "ssbh/extract.hpp"
#include "ssbh/prf.hpp"
#include "ssbh/sampling.hpp"
#include "ssbh/toeplitz.hpp"
#include "ssbh_cuda.h"

namespace ssbh {

// ---------------------------------------------------------------------------- errors
void detail::throw_status(int status) {
    if (status == SSBH_OK) return;
    const std::string msg = ssbh_last_error();
    switch (status) {
        case SSBH_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case SSBH_INFEASIBLE: throw infeasible_error(msg);
        case SSBH_OVERFLOW: throw std::overflow_error(msg);
        case SSBH_IO: throw io_error(msg);
        default: throw device_error(msg);
    }
}

namespace {
inline void check(ssbh_status s) { detail::throw_status(s); }
}  // namespace

// ------------------------------------------------------------------------- BitString
BitString BitString::from_bools(std::span<const int> bits) {
    BitString out(bits.size());
    for (std::uint64_t i = 0; i < bits.size(); ++i)
        if (bits[i] != 0) out.set(i, true);
    return out;
}

BitString BitString::from_bytes(std::span<const std::uint8_t> bytes, std::uint64_t nbits) {
    if (bytes.size() * 8 < nbits)
        throw std::invalid_argument("from_bytes: byte buffer shorter than bit count");
    BitString out(nbits);
    const std::uint64_t nbytes = (nbits + 7) / 8;
    for (std::uint64_t b = 0; b < nbytes; ++b)
        out.words_[b / 8] |= static_cast<std::uint64_t>(bytes[b]) << (8 * (b % 8));
    out.mask_tail();
    return out;
}

std::uint64_t BitString::popcount() const {
    std::uint64_t c = 0;
    for (const std::uint64_t w : words_) c += static_cast<std::uint64_t>(std::popcount(w));
    return c;
}

void BitString::xor_with(const BitString& other) {
    if (other.len_ != len_) throw std::invalid_argument("xor_with: length mismatch");
    for (std::size_t i = 0; i < words_.size(); ++i) words_[i] ^= other.words_[i];
}

void BitString::append(const BitString& tail) {
    const std::uint64_t at = len_;
    len_ += tail.len_;
    words_.resize((len_ + 63) / 64, 0);
    xor_bit_range(words_, at, tail.words_, 0, tail.len_);
}

BitString BitString::slice(std::uint64_t first, std::uint64_t count) const {
    if (first + count > len_ || first + count < first)
        throw std::invalid_argument("slice: range out of bounds");
    BitString out(count);
    xor_bit_range(out.words_, 0, words_, first, count);
    return out;
}

std::vector<std::uint8_t> BitString::to_bytes() const {
    std::vector<std::uint8_t> out((len_ + 7) / 8);
    for (std::uint64_t b = 0; b < out.size(); ++b)
        out[b] = static_cast<std::uint8_t>(words_[b / 8] >> (8 * (b % 8)));
    return out;
}

void BitString::write_file(const std::string& path) const {
    std::unique_ptr<std::FILE, int (*)(std::FILE*)> f(std::fopen(path.c_str(), "wb"),
                                                       std::fclose);
    if (!f) throw io_error("cannot open for writing: " + path);
    const auto bytes = to_bytes();
    if (!bytes.empty() && std::fwrite(bytes.data(), 1, bytes.size(), f.get()) != bytes.size())
        throw io_error("short write: " + path);
}

BitString BitString::read_file(const std::string& path, std::uint64_t nbits) {
    std::unique_ptr<std::FILE, int (*)(std::FILE*)> f(std::fopen(path.c_str(), "rb"),
                                                       std::fclose);
    if (!f) throw io_error("cannot open for reading: " + path);
    std::vector<std::uint8_t> bytes((nbits + 7) / 8);
    if (!bytes.empty() && std::fread(bytes.data(), 1, bytes.size(), f.get()) != bytes.size())
        throw io_error("file shorter than requested bit count: " + path);
    return from_bytes(bytes, nbits);
}

void BitString::mask_tail() {
    if ((len_ & 63) != 0 && !words_.empty()) words_.back() &= (std::uint64_t{1} << (len_ & 63)) - 1;
}

void xor_bit_range(std::span<std::uint64_t> dst, std::uint64_t dst_off,
                   std::span<const std::uint64_t> src, std::uint64_t src_off,
                   std::uint64_t nbits) {
    // 64 source bits starting at `bit`; words past src.size() read as zero.
    auto window = [&](std::uint64_t bit) {
        const std::uint64_t q = bit / 64;
        const unsigned r = static_cast<unsigned>(bit % 64);
        const std::uint64_t lo = q < src.size() ? src[q] : 0;
        if (r == 0) return lo;
        const std::uint64_t hi = q + 1 < src.size() ? src[q + 1] : 0;
        return (lo >> r) | (hi << (64 - r));
    };
    std::uint64_t done = 0;
    while (done < nbits) {
        const std::uint64_t d = dst_off + done;
        const unsigned dr = static_cast<unsigned>(d % 64);
        const std::uint64_t take = std::min<std::uint64_t>(64 - dr, nbits - done);
        std::uint64_t chunk = window(src_off + done);
        if (take < 64) chunk &= (std::uint64_t{1} << take) - 1;
        dst[d / 64] ^= chunk << dr;
        done += take;
    }
}

// ------------------------------------------------------------------------------- PRF
MasterSeed MasterSeed::from_hex(std::string_view hex) {
    if (hex.size() != 64) throw std::invalid_argument("master seed must be 64 hex digits");
    MasterSeed s;
    for (std::size_t i = 0; i < 64; ++i) {
        const char c = hex[i];
        int d = -1;
        if (c >= '0' && c <= '9') d = c - '0';
        else if (c >= 'a' && c <= 'f') d = c - 'a' + 10;
        else if (c >= 'A' && c <= 'F') d = c - 'A' + 10;
        if (d < 0) throw std::invalid_argument("master seed contains a non-hex digit");
        s.words[i / 16] = (s.words[i / 16] << 4) | static_cast<std::uint64_t>(d);
    }
    return s;
}

std::string MasterSeed::to_hex() const {
    static constexpr char kDigits[] = "0123456789abcdef";
    std::string out;
    out.reserve(64);
    for (const std::uint64_t w : words)
        for (int sh = 60; sh >= 0; sh -= 4) out.push_back(kDigits[(w >> sh) & 0xF]);
    return out;
}

std::array<std::uint64_t, 4> prf::block(const std::array<std::uint64_t, 4>& key,
                                        const std::array<std::uint64_t, 4>& ctr) {
    std::array<std::uint64_t, 4> out{};
    check(ssbh_prf_block(key.data(), ctr.data(), out.data()));
    return out;
}

std::uint64_t KeyedStream::word(std::uint64_t index) const {
    return prf::block(key_, {tag_, sub_, index, 0})[0];
}

std::uint64_t KeyedStream::uniform_below(std::uint64_t bound, std::uint64_t index) const {
    if (bound == 0) throw std::invalid_argument("uniform_below: bound must be positive");
    if (std::has_single_bit(bound)) return word(index) & (bound - 1);
    const std::uint64_t limit = ~std::uint64_t{0} - (~std::uint64_t{0} % bound + 1) % bound;
    for (std::uint64_t attempt = 0;; ++attempt) {
        const std::uint64_t r = prf::block(key_, {tag_, sub_, index, attempt})[0];
        if (r <= limit) return r % bound;
    }
}

bool KeyedStream::bernoulli(double p, std::uint64_t index) const {
    if (p < 0.0 || p > 1.0) throw std::invalid_argument("bernoulli: p outside [0,1]");
    return static_cast<double>(word(index) >> 11) * 0x1.0p-53 < p;
}

BitString KeyedStream::bits(std::uint64_t nbits) const {
    BitString out(nbits);
    if (nbits) check(ssbh_stream_bits(key_.data(), tag_, sub_, nbits, out.words().data()));
    return out;
}

// -------------------------------------------------------------------------- sampling
Partition assign_subblocks(std::uint64_t n_rounds, std::uint32_t n_subblocks,
                           const MasterSeed& seed) {
    if (n_subblocks == 0)
        throw std::invalid_argument("assign_subblocks: n_subblocks must be positive");
    Partition p;
    p.n_subblocks = n_subblocks;
    p.assignment.resize(n_rounds);
    p.raw_counts.assign(n_subblocks, 0);
    check(ssbh_assign_subblocks(n_rounds, n_subblocks, seed.words.data(), p.assignment.data(),
                                p.raw_counts.data()));
    return p;
}

SiftedPartition sift_partition(std::span<const std::uint8_t> keep, const Partition& partition) {
    if (keep.size() != partition.assignment.size())
        throw std::invalid_argument("sift_partition: flag count does not match partition");
    const std::uint32_t s = partition.n_subblocks;
    std::vector<std::uint64_t> off(static_cast<std::size_t>(s) + 1, 0), idx(keep.size());
    std::uint64_t max_len = 0;
    check(ssbh_sift_partition(keep.data(), keep.size(), partition.assignment.data(), s,
                              off.data(), idx.data(), &max_len));
    SiftedPartition out;
    out.blocks.resize(s);
    for (std::uint32_t j = 0; j < s; ++j)
        out.blocks[j].assign(idx.begin() + static_cast<std::ptrdiff_t>(off[j]),
                             idx.begin() + static_cast<std::ptrdiff_t>(off[j + 1]));
    out.max_len = max_len;
    return out;
}

double relative_entropy(double x, double p) {
    double v = 0;
    check(ssbh_relative_entropy(x, p, &v));
    return v;
}

double binomial_tail_bound(std::uint64_t n_rounds, std::uint64_t limit, double p_sift) {
    double v = 0;
    check(ssbh_binomial_tail_bound(n_rounds, limit, p_sift, &v));
    return v;
}

std::uint64_t block_limit(std::uint64_t n_rounds, double p_sift, double eps_abort,
                          std::uint64_t m_blocks) {
    std::uint64_t v = 0;
    check(ssbh_block_limit(n_rounds, p_sift, eps_abort, m_blocks, &v));
    return v;
}

bool abort_check(std::span<const std::uint64_t> lengths, std::uint64_t limit) {
    return ssbh_abort_check(lengths.data(), lengths.size(), limit) != 0;
}

// -------------------------------------------------------------------------- toeplitz
ToeplitzSeed::ToeplitzSeed(BitString s, std::uint64_t m_, std::uint64_t n_)
    : seed(std::move(s)), m(m_), n(n_) {
    if (m == 0 || n == 0) throw std::invalid_argument("toeplitz: m and n must be positive");
    if (seed.size() != m + n - 1) throw std::invalid_argument("toeplitz: seed must hold m+n-1 bits");
}

BitString toeplitz_hash(const ToeplitzSeed& seed, const BitString& input) {
    BitString out(seed.m);
    check(ssbh_toeplitz_hash(seed.seed.words().data(), seed.m, seed.n, input.words().data(),
                             input.size(), out.words().data()));
    return out;
}

BitString blocked_toeplitz_hash(const ToeplitzSeed& seed, const BitString& input,
                                const BlockingParams& blocking) {
    BitString out(seed.m);
    check(ssbh_blocked_toeplitz_hash(seed.seed.words().data(), seed.m, seed.n,
                                     input.words().data(), input.size(), blocking.m_prime,
                                     blocking.n_prime, out.words().data()));
    return out;
}

std::uint64_t cycle_estimate(std::uint64_t input_len, std::uint64_t output_len,
                             std::uint64_t m_prime) {
    std::uint64_t v = 0;
    check(ssbh_cycle_estimate(input_len, output_len, m_prime, &v));
    return v;
}

// ------------------------------------------------------------------- B200 additions
ExtractResult extract(const BitString& input, std::uint32_t n_subblocks,
                      std::uint64_t out_bits_per_block, const MasterSeed& sampling_seed,
                      const MasterSeed& hash_seed, const ExtractOptions& opt) {
    if (opt.device >= 0) check(ssbh_set_device(opt.device));
    ssbh_extract_params p{};
    p.n_rounds = input.size();
    p.n_subblocks = n_subblocks;
    p.per_block_seed = opt.seed_mode == SeedMode::PerBlock ? 1u : 0u;
    p.out_bits = out_bits_per_block;
    std::memcpy(p.samp_key, sampling_seed.words.data(), 32);
    std::memcpy(p.hash_key, hash_seed.words.data(), 32);
    p.block_first = opt.block_first;
    p.block_count = opt.block_count;
    p.block_limit = opt.block_limit;
    const std::uint64_t owned = opt.block_count ? opt.block_count : n_subblocks;
    ExtractResult r;
    r.block_lengths.assign(owned, 0);
    BitString key(owned * out_bits_per_block);
    ssbh_extract_stats st{};
    const ssbh_status s =
        opt.devices.size() > 1
            ? ssbh_extract_multi(&p, input.words().data(), opt.devices.data(),
                                 static_cast<std::uint32_t>(opt.devices.size()), key.words().data(),
                                 r.block_lengths.data(), &st)
            : ssbh_extract(&p, input.words().data(), key.words().data(), r.block_lengths.data(),
                           &st);
    if (s == SSBH_ABORT_OVERSIZE) {
        r.aborted = true;
        return r;
    }
    check(s);
    r.key = std::move(key);
    r.hash_word_ops = st.hash_word_ops;
    r.device_ms = st.ms_total;
    return r;
}

BitString toeplitz_hash_batch(const std::vector<ToeplitzSeed>& seeds,
                              const std::vector<BitString>& inputs) {
    if (seeds.size() != inputs.size())
        throw std::invalid_argument("toeplitz_hash_batch: seeds/inputs count mismatch");
    if (seeds.empty()) return BitString();
    const std::uint64_t m = seeds[0].m;
    std::vector<std::uint64_t> n(seeds.size());
    std::vector<const std::uint64_t*> in_ptr(seeds.size()), seed_ptr(seeds.size());
    for (std::size_t b = 0; b < seeds.size(); ++b) {
        if (seeds[b].m != m)
            throw std::invalid_argument("toeplitz_hash_batch: output lengths differ");
        if (inputs[b].size() != seeds[b].n)
            throw std::invalid_argument("toeplitz: input length does not match seed.n");
        n[b] = seeds[b].n;
        in_ptr[b] = inputs[b].words().data();
        seed_ptr[b] = seeds[b].seed.words().data();
    }
    BitString out(m * seeds.size());
    check(ssbh_toeplitz_hash_batch_ptrs(seeds.size(), m, n.data(), in_ptr.data(),
                                        seed_ptr.data(), out.words().data()));
    return out;
}

PreparedHashBatch::PreparedHashBatch(const std::vector<ToeplitzSeed>& seeds,
                                     const std::vector<BitString>& inputs) {
    if (seeds.size() != inputs.size())
        throw std::invalid_argument("toeplitz_hash_batch: seeds/inputs count mismatch");
    if (seeds.empty()) throw std::invalid_argument("toeplitz: m and n must be positive");
    const std::uint64_t m = seeds[0].m;
    std::vector<std::uint64_t> n(seeds.size());
    std::vector<const std::uint64_t*> in_ptr(seeds.size()), seed_ptr(seeds.size());
    for (std::size_t b = 0; b < seeds.size(); ++b) {
        if (seeds[b].m != m)
            throw std::invalid_argument("toeplitz_hash_batch: output lengths differ");
        if (inputs[b].size() != seeds[b].n)
            throw std::invalid_argument("toeplitz: input length does not match seed.n");
        n[b] = seeds[b].n;
        in_ptr[b] = inputs[b].words().data();
        seed_ptr[b] = seeds[b].seed.words().data();
    }
    ssbh_hash_batch* h = nullptr;
    check(ssbh_hash_batch_create(seeds.size(), m, n.data(), in_ptr.data(), seed_ptr.data(), &h));
    handle_ = h;
    out_bits_ = m * seeds.size();
}

PreparedHashBatch::~PreparedHashBatch() {
    ssbh_hash_batch_destroy(static_cast<ssbh_hash_batch*>(handle_));
}

BitString PreparedHashBatch::run() const {
    BitString out(out_bits_);
    check(ssbh_hash_batch_run(static_cast<ssbh_hash_batch*>(handle_), out.words().data()));
    return out;
}

}  // namespace ssbh
