// Fused extraction (GPU) == the reference's own per-block loop written with the drop-in
// API (proj/tools/ssbh_main.cpp:317-336 with distinct seeds; proj/tests/test_pipeline.cpp
// :126-149 single-block case; test_cli.cpp:162-181 file-mode case).
#include <random>

#include "mini_test.hpp"
#include "ssbh/errors.hpp"
#include "ssbh/extract.hpp"
#include "ssbh/sampling.hpp"
#include "ssbh/toeplitz.hpp"

using namespace ssbh;

namespace {

BitString loop_extract(const BitString& data, std::uint32_t ns, std::uint64_t k,
                       const MasterSeed& samp, const MasterSeed& hash, bool per_block) {
    const Partition part = assign_subblocks(data.size(), ns, samp);
    const SiftedPartition sifted = sift_partition(std::vector<std::uint8_t>(data.size(), 1), part);
    BitString key;
    for (std::uint32_t j = 0; j < ns; ++j) {
        BitString x(sifted.blocks[j].size());
        for (std::uint64_t q = 0; q < x.size(); ++q)
            if (data.get(sifted.blocks[j][q])) x.set(q, true);
        const KeyedStream st(hash, "hash-seed", per_block ? j : 0);
        key.append(toeplitz_hash(ToeplitzSeed(st.bits(k + x.size() - 1), k, x.size()), x));
    }
    return key;
}

MasterSeed seed_n(unsigned v) {
    char buf[65];
    std::snprintf(buf, sizeof buf, "%064x", v);
    return MasterSeed::from_hex(buf);
}

}  // namespace

TEST_CASE("fused extract equals the per-block reference loop") {
    std::mt19937_64 rng(41);
    const std::uint64_t ks[] = {64, 77, 96, 1000, 4096};
    const std::uint32_t ss[] = {1, 3, 8, 16, 64};
    for (int it = 0; it < 10; ++it) {
        const std::uint64_t n = 20000 + rng() % 200000;
        const std::uint32_t ns = ss[rng() % 5];
        const std::uint64_t k = ks[rng() % 5];
        const bool pb = rng() & 1;
        const BitString data = KeyedStream(seed_n(it), "input").bits(n);
        const ExtractResult r = extract(data, ns, k, seed_n(100 + it), seed_n(200 + it),
                                        {pb ? SeedMode::PerBlock : SeedMode::Shared});
        REQUIRE_FALSE(r.aborted);
        CHECK(r.key == loop_extract(data, ns, k, seed_n(100 + it), seed_n(200 + it), pb));
        std::uint64_t tot = 0;
        for (auto l : r.block_lengths) tot += l;
        CHECK(tot == n);
        CHECK(r.hash_word_ops == n * k / 32);
    }
}

TEST_CASE("single sub-block extraction is the direct hash of the whole string") {
    const BitString data = KeyedStream(seed_n(7), "input").bits(300000);
    const ExtractResult r = extract(data, 1, 5000, seed_n(8), seed_n(9));
    const ToeplitzSeed ts(KeyedStream(seed_n(9), "hash-seed", 0).bits(5000 + data.size() - 1),
                          5000, data.size());
    CHECK(r.key == toeplitz_hash(ts, data));
}

TEST_CASE("BASELINE config 1 digest (golden, from the compiled reference)") {
    const BitString data = KeyedStream(seed_n(1), "input").bits(1 << 20);
    const ExtractResult r = extract(data, 64, 8192, seed_n(2), seed_n(3));
    std::uint64_t h = 0xcbf29ce484222325ull;
    for (auto w : r.key.words())
        for (int b = 0; b < 8; ++b) h = (h ^ ((w >> (8 * b)) & 0xff)) * 0x100000001b3ull;
    CHECK(h == 0xa32d120e3143264bull);
    CHECK(r.key.popcount() == 262107);
    CHECK(r.key.words()[0] == 0xc2ad7a9ff67db7bbull);
}

TEST_CASE("owned block ranges, abort and empty blocks") {
    const BitString data = KeyedStream(seed_n(3), "input").bits(100000);
    const ExtractResult full = extract(data, 16, 512, seed_n(4), seed_n(5));
    BitString joined;
    for (std::uint32_t f = 0; f < 16; f += 4) {
        ExtractOptions o;
        o.block_first = f;
        o.block_count = 4;
        joined.append(extract(data, 16, 512, seed_n(4), seed_n(5), o).key);
    }
    CHECK(joined == full.key);
    std::uint64_t mx = 0;
    for (auto l : full.block_lengths) mx = std::max(mx, l);
    ExtractOptions lim;
    lim.block_limit = mx - 1;
    CHECK(extract(data, 16, 512, seed_n(4), seed_n(5), lim).aborted);
    lim.block_limit = mx;
    CHECK_FALSE(extract(data, 16, 512, seed_n(4), seed_n(5), lim).aborted);
    CHECK_THROWS_AS(extract(BitString(64), 1000, 8, seed_n(1), seed_n(2)), std::invalid_argument);
}

TEST_CASE("one process over several devices equals one device") {
    // ssbh_extract_multi with ranks on repeated device ids (a 1-GPU box): sharded sampling,
    // owner split through device pointers, per-owner hashing, bit-offset concatenation
    const BitString data = KeyedStream(seed_n(6), "input").bits(300001);
    for (std::uint64_t k : {512ull, 77ull}) {
        ExtractOptions pb;
        pb.seed_mode = SeedMode::PerBlock;
        const ExtractResult one = extract(data, 33, k, seed_n(7), seed_n(8), pb);
        for (std::size_t nd : {2u, 3u}) {
            ExtractOptions m = pb;
            m.devices.assign(nd, 0);
            const ExtractResult multi = extract(data, 33, k, seed_n(7), seed_n(8), m);
            CHECK(multi.key == one.key);
            CHECK(multi.block_lengths == one.block_lengths);
            CHECK(multi.hash_word_ops > 0);
        }
    }
    std::uint64_t mx = 0;
    const ExtractResult full = extract(data, 33, 512, seed_n(7), seed_n(8));
    for (auto l : full.block_lengths) mx = std::max(mx, l);
    ExtractOptions lim;
    lim.devices = {0, 0};
    lim.block_limit = mx - 1;
    CHECK(extract(data, 33, 512, seed_n(7), seed_n(8), lim).aborted);
}
