// ssbh/extract.hpp — B200 additions beside the drop-in API (no reference header):
// the fused extraction and the batched hash that the reference performs as a per-block
// loop (proj/tools/ssbh_main.cpp:317-336, proj/src/pipeline.cpp:111-136). Needed at
// BASELINE scale, where the reference's Partition/SiftedPartition (12 B per round) cannot
// be held in host memory.
#pragma once

#include <cstdint>
#include <vector>

#include "ssbh/bitstring.hpp"
#include "ssbh/prf.hpp"
#include "ssbh/toeplitz.hpp"

namespace ssbh {

enum class SeedMode {
    Shared,    ///< every block: KeyedStream(hash_seed, "hash-seed", 0).bits(k + n_j - 1)
    PerBlock,  ///< block j:     KeyedStream(hash_seed, "hash-seed", j).bits(k + n_j - 1)
};

struct ExtractOptions {
    SeedMode seed_mode = SeedMode::Shared;
    std::uint32_t block_first = 0;  ///< owned block range (multi-GPU sharding)
    std::uint32_t block_count = 0;  ///< 0 = all blocks
    std::uint64_t block_limit = 0;  ///< 0 = no abort check; else strict n_j > limit aborts
    int device = -1;                ///< CUDA device, -1 = current
    /// > 1 entries: one process over these GPUs (sharded sampling, owner split through peer
    /// memory; the whole key — block_first/block_count must be 0). Entries may repeat.
    std::vector<int> devices;
};

struct ExtractResult {
    BitString key;                         ///< concatenation of the owned blocks' outputs
    std::vector<std::uint64_t> block_lengths;  ///< owned n_j
    bool aborted = false;                  ///< oversize abort (key empty)
    std::uint64_t hash_word_ops = 0;       ///< sum n_j * k / 32
    double device_ms = 0;                  ///< device time of the fused run
};

/// The file-mode hot path with distinct seeds: assign_subblocks(n, s, samp)
/// -> sift (all rounds kept) -> per block j: gather, Toeplitz seed, toeplitz_hash ->
/// concatenate. Bit-identical to running those reference calls one by one.
/// std::invalid_argument on an empty owned sub-block (as ToeplitzSeed throws).
ExtractResult extract(const BitString& input, std::uint32_t n_subblocks,
                      std::uint64_t out_bits_per_block, const MasterSeed& sampling_seed,
                      const MasterSeed& hash_seed, const ExtractOptions& options = {});

/// One GPU launch for many independent hashes with a common output length; returns the
/// concatenation of toeplitz_hash(seeds[b], inputs[b]) in order.
BitString toeplitz_hash_batch(const std::vector<ToeplitzSeed>& seeds,
                              const std::vector<BitString>& inputs);

/// The same batch with the seeds and inputs uploaded once and kept on the device: run() hashes
/// every block and returns the concatenation. What the reference's cmd_bench times
/// (ssbh_main.cpp:405-410: the toeplitz_hash calls alone, gather and seed generation untimed)
/// corresponds to run().
class PreparedHashBatch {
public:
    PreparedHashBatch(const std::vector<ToeplitzSeed>& seeds, const std::vector<BitString>& inputs);
    ~PreparedHashBatch();
    PreparedHashBatch(const PreparedHashBatch&) = delete;
    PreparedHashBatch& operator=(const PreparedHashBatch&) = delete;
    BitString run() const;

private:
    void* handle_ = nullptr;
    std::uint64_t out_bits_ = 0;
};

}  // namespace ssbh
