/*
 * ssbh_cuda.h — C-ABI of the B200-native sampled sub-block Toeplitz extractor.
 *
 * Plain pointers and sizes only (no C++ / torch types). Every entry point returns an
 * ssbh_status; on failure ssbh_last_error() holds a thread-local message. The C++
 * drop-in layer (include/ssbh/*.hpp) maps the codes back to the reference's exception
 * types (std::invalid_argument, ssbh::infeasible_error, std::overflow_error,
 * ssbh::io_error — proj/include/ssbh/errors.hpp:10-18).
 *
 * Bit layout (proj/include/ssbh/bitstring.hpp:11-15): bit k of a stream is bit k%64 of
 * uint64 word k/64, storage past the length is zero. Host buffers are uint64 words;
 * device buffers may be viewed as uint32 words (little-endian, same bit order).
 *
 * "Reference:" lines cite the reference interface each entry point replaces
 * (paths under the reference tree proj/).
 *
 * Every compute entry point runs on the GPU (sm_100a); there is no CPU fallback.
 * Without a usable CUDA device they return SSBH_NO_DEVICE.
 */
#ifndef SSBH_CUDA_H
#define SSBH_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SSBH_ABI_VERSION 1

typedef enum {
    SSBH_OK = 0,
    SSBH_INVALID_ARGUMENT = 1, /* std::invalid_argument in the reference */
    SSBH_INFEASIBLE = 2,       /* ssbh::infeasible_error (errors.hpp:10-13) */
    SSBH_OVERFLOW = 3,         /* std::overflow_error (toeplitz.cpp:86-87) */
    SSBH_IO = 4,               /* ssbh::io_error (errors.hpp:15-18) */
    SSBH_CUDA = 5,             /* CUDA runtime / launch failure */
    SSBH_NO_DEVICE = 6,        /* no usable sm_100 device */
    SSBH_ABORT_OVERSIZE = 7    /* abort_check failed (ssbh_main.cpp:324-326) */
} ssbh_status;

/* ------------------------------------------------------------------ runtime */
int ssbh_abi_version(void);
const char* ssbh_last_error(void);
/* Number of CUDA devices usable by the library (0 when none). */
int ssbh_device_count(void);
/* Selects the device used by subsequent calls from this host thread. */
ssbh_status ssbh_set_device(int device);

/* ---------------------------------------------------------------------- PRF */
/* Reference: prf::block — proj/include/ssbh/prf.hpp:26-27, proj/src/prf.cpp:47-76.
 * Scalar Threefry4x64-20 (same __host__ __device__ function as the kernels). */
ssbh_status ssbh_prf_block(const uint64_t key[4], const uint64_t ctr[4], uint64_t out[4]);

/* Reference: prf::tag — proj/include/ssbh/prf.hpp:29-37 (FNV-1a-64). */
uint64_t ssbh_prf_tag(const char* purpose, size_t len);

/* Reference: KeyedStream::bits — proj/include/ssbh/prf.hpp:65, proj/src/prf.cpp:104-115.
 * Host output, ceil(nbits/64) words, zero tail. GPU-generated. */
ssbh_status ssbh_stream_bits(const uint64_t key[4], uint64_t tag, uint64_t sub, uint64_t nbits,
                             uint64_t* out_words);

/* Reference: KeyedStream::word — prf.hpp:56, prf.cpp:80-82; out[q] = word(first + q). */
ssbh_status ssbh_stream_words(const uint64_t key[4], uint64_t tag, uint64_t sub, uint64_t first,
                              uint64_t count, uint64_t* out);

/* Reference: KeyedStream::uniform_below — prf.hpp:59, prf.cpp:84-94 (rejection sampled,
 * retry counter in ctr[3]); out[q] = uniform_below(bound, first + q). bound == 0 ->
 * SSBH_INVALID_ARGUMENT. */
ssbh_status ssbh_stream_uniform_below(const uint64_t key[4], uint64_t tag, uint64_t sub,
                                      uint64_t bound, uint64_t first, uint64_t count,
                                      uint64_t* out);

/* Reference: KeyedStream::bernoulli — prf.hpp:62, prf.cpp:96-102. Packed output: bit q of
 * out_words = bernoulli(p, first + q). p outside [0,1] -> SSBH_INVALID_ARGUMENT. */
ssbh_status ssbh_stream_bernoulli(const uint64_t key[4], uint64_t tag, uint64_t sub, double p,
                                  uint64_t first, uint64_t count, uint64_t* out_words);

/* ------------------------------------------------------------------ sampler */
/* Reference: assign_subblocks — proj/include/ssbh/sampling.hpp:37-38,
 * proj/src/sampling.cpp:10-25. assignment[i] = V_i in [1, s] (uint32), raw_counts[s]. */
ssbh_status ssbh_assign_subblocks(uint64_t n_rounds, uint32_t n_subblocks, const uint64_t key[4],
                                  uint32_t* assignment, uint64_t* raw_counts);

/* Reference: sift_partition — sampling.hpp:41, sampling.cpp:27-39. CSR result: block j's
 * kept round indices (round order) are indices[offsets[j] .. offsets[j+1]);
 * offsets has s+1 entries, indices capacity >= number of kept rounds. keep may be NULL
 * (all rounds kept). Assignment values outside [1, s] -> SSBH_INVALID_ARGUMENT. */
ssbh_status ssbh_sift_partition(const uint8_t* keep, uint64_t n, const uint32_t* assignment,
                                uint32_t n_subblocks, uint64_t* offsets, uint64_t* indices,
                                uint64_t* max_len);

/* Reference: block_limit / binomial_tail_bound / relative_entropy / abort_check —
 * sampling.hpp:45-57, sampling.cpp:41-96. Host scalar numerics (not data-parallel). */
ssbh_status ssbh_block_limit(uint64_t n_rounds, double p_sift, double eps_abort,
                             uint64_t m_blocks, uint64_t* limit);
ssbh_status ssbh_binomial_tail_bound(uint64_t n_rounds, uint64_t limit, double p_sift,
                                     double* out);
ssbh_status ssbh_relative_entropy(double x, double p, double* out);
int ssbh_abort_check(const uint64_t* lengths, uint64_t count, uint64_t limit);

/* Key digest used by reports and golden fixtures (not a reference entry point): FNV-1a-64
 * over the little-endian bytes of `count` u64 words (offset 0xcbf29ce484222325, prime
 * 0x100000001b3). Host memory, host computation. */
uint64_t ssbh_fnv1a64(const uint64_t* words, uint64_t count);

/* ----------------------------------------------------------------- toeplitz */
/* Reference: toeplitz_hash — proj/include/ssbh/toeplitz.hpp:27, proj/src/toeplitz.cpp:34-52
 * (and ToeplitzSeed validation toeplitz.cpp:9-15): K = T x over GF(2) with
 * T[i][j] = seed[(n-1)+i-j]; seed has m+n-1 bits, input n bits, out m bits (host words). */
ssbh_status ssbh_toeplitz_hash(const uint64_t* seed, uint64_t m, uint64_t n,
                               const uint64_t* input, uint64_t input_bits, uint64_t* out);

/* Reference: blocked_toeplitz_hash — toeplitz.hpp:31-32, toeplitz.cpp:54-76. The product is
 * bit-identical for every blocking; m_prime/n_prime are validated like the reference. */
ssbh_status ssbh_blocked_toeplitz_hash(const uint64_t* seed, uint64_t m, uint64_t n,
                                       const uint64_t* input, uint64_t input_bits,
                                       uint64_t m_prime, uint64_t n_prime, uint64_t* out);

/* Reference: cycle_estimate — toeplitz.hpp:36-37, toeplitz.cpp:78-89 (host scalar). */
ssbh_status ssbh_cycle_estimate(uint64_t input_len, uint64_t output_len, uint64_t m_prime,
                                uint64_t* out);

/* Batched hash (the per-block loop of ssbh_main.cpp:328-336 / pipeline.cpp:129-136 in one
 * launch): block b has input bits inputs[in_off[b]*64 ...] of length n[b], seed words
 * seeds[seed_off[b] ...] of m+n[b]-1 bits; all blocks have m output bits; the results are
 * concatenated (bitstring.cpp:42-47) into out (ceil(count*m/64) words). Host buffers. */
ssbh_status ssbh_toeplitz_hash_batch(uint64_t count, uint64_t m, const uint64_t* n,
                                     const uint64_t* inputs, const uint64_t* in_off,
                                     const uint64_t* seeds, const uint64_t* seed_off,
                                     uint64_t* out);

/* The same batch with one host pointer per block (no host-side concatenation: each block's
 * input and seed are copied straight from the caller's BitStrings); what the C++ drop-in's
 * toeplitz_hash_batch (include/ssbh/extract.hpp) binds. */
ssbh_status ssbh_toeplitz_hash_batch_ptrs(uint64_t count, uint64_t m, const uint64_t* n,
                                          const uint64_t* const* inputs,
                                          const uint64_t* const* seeds, uint64_t* out);

/* Prepared batch: the same hashes with the inputs and seeds resident on the device. create
 * uploads and packs them once (what the reference's cmd_bench does untimed before its timed
 * toeplitz_hash loop, ssbh_main.cpp:388-404); run hashes every block and copies the
 * concatenated result (ceil(count*m/64) words) to out — the call that corresponds to the
 * reference's timed region (ssbh_main.cpp:405-410). A B200 addition (no reference symbol). */
typedef struct ssbh_hash_batch ssbh_hash_batch;
ssbh_status ssbh_hash_batch_create(uint64_t count, uint64_t m, const uint64_t* n,
                                   const uint64_t* const* inputs, const uint64_t* const* seeds,
                                   ssbh_hash_batch** out);
ssbh_status ssbh_hash_batch_run(ssbh_hash_batch* batch, uint64_t* out);
ssbh_status ssbh_hash_batch_destroy(ssbh_hash_batch* batch);

/* The reference-facing calls above (toeplitz_hash, KeyedStream::bits, assign_subblocks,
 * sift_partition, ...) keep a per-thread, per-device stream and device arena between calls,
 * so that steady-state calls allocate nothing. This frees the calling thread's arenas (they
 * are also freed when the thread exits). */
ssbh_status ssbh_release_thread_cache(void);

/* -------------------------------------------------------- fused extraction */
/* The whole file-mode hot path (ssbh_main.cpp:306-345 with distinct seeds):
 * assign_subblocks(n, s, samp) -> sift (all kept, or keep mask) -> per block j gather ->
 * seed = KeyedStream(hash, "hash-seed", per_block ? j : 0).bits(k + n_j - 1) ->
 * toeplitz_hash -> concatenation in block order.
 *
 * Blocks [block_first, block_first + block_count) are produced (multi-GPU sharding:
 * each rank owns a contiguous block range; block_count == 0 means all s blocks).
 * block_limit != 0 enables the reference's strict abort (any n_j > block_limit ->
 * SSBH_ABORT_OVERSIZE, key untouched). An empty owned sub-block -> SSBH_INVALID_ARGUMENT
 * ("toeplitz: m and n must be positive", as ToeplitzSeed throws, toeplitz.cpp:11-12). */
typedef struct {
    uint64_t n_rounds;      /* n input bits */
    uint32_t n_subblocks;   /* s */
    uint32_t per_block_seed;/* 0: shared seed (sub 0); 1: sub = j (pipeline.cpp:132) */
    uint64_t out_bits;      /* k output bits per sub-block */
    uint64_t samp_key[4];   /* MasterSeed for "sampling" */
    uint64_t hash_key[4];   /* MasterSeed for "hash-seed" */
    uint32_t block_first;
    uint32_t block_count;   /* 0 = all */
    uint64_t block_limit;   /* 0 = no abort check */
} ssbh_extract_params;

typedef struct {
    double ms_sample;       /* Threefry + count + scan (device, CUDA events) */
    double ms_scatter;      /* stable partition + reversed bit pack */
    double ms_seed;         /* Toeplitz seed generation */
    double ms_hash;         /* GF(2) Toeplitz hash */
    double ms_total;
    uint64_t hash_word_ops; /* sum_j n_j * k / 32 over owned blocks (algorithmic LOP3) */
    uint64_t max_len;       /* max owned n_j */
    uint64_t min_len;       /* min owned n_j */
    uint32_t hash_launches; /* kernel launches of the hash kernel */
    uint32_t launches;      /* all kernel launches of the run */
} ssbh_extract_stats;

/* Opaque device plan: buffers sized once for (n, s, k, ownership), reused across runs. */
typedef struct ssbh_plan ssbh_plan;

ssbh_status ssbh_plan_create(const ssbh_extract_params* params, ssbh_plan** plan);
ssbh_status ssbh_plan_destroy(ssbh_plan* plan);
/* Device bytes held by the plan. */
uint64_t ssbh_plan_device_bytes(const ssbh_plan* plan);

/* Device-resident run on `stream` (cudaStream_t as void*; NULL = legacy default stream).
 * d_input: ceil(n/32) uint32 words on the plan's device; d_key: output words
 * (ceil(owned*k/32) uint32, written in full); d_lengths: owned n_j (uint64, may be NULL).
 * Asynchronous: errors detected on the device are reported by ssbh_plan_check. The
 * sampling / hash seeds may be changed per run (samp_key/hash_key may be NULL = plan's). */
ssbh_status ssbh_plan_run_device(ssbh_plan* plan, const uint32_t* d_input, uint32_t* d_key,
                                 uint64_t* d_lengths, const uint64_t* samp_key,
                                 const uint64_t* hash_key, void* stream);
/* Synchronizes the plan's last run and converts device-side flags to a status
 * (empty block / oversize abort). Fills stats when non-NULL (timings need
 * ssbh_plan_set_timing(plan, 1) before the run). */
ssbh_status ssbh_plan_check(ssbh_plan* plan, ssbh_extract_stats* stats);
ssbh_status ssbh_plan_set_timing(ssbh_plan* plan, int enable);

/* Hash engine of a plan (not a reference interface: the reference has one CPU loop).
 *   SSBH_ENGINE_LOP3   : GF(2) product on the integer ALUs (LOP3/SHF/POPC; north_star's kernel).
 *   SSBH_ENGINE_TENSOR : the product as exact integer counts mod 2 on the tcgen05 tensor cores
 *                        (kind::mxf4, E2M1 0 / 1.0 operands, f32 accumulators): shared seeds =
 *                        one GEMM of all blocks against the one Hankel matrix, per-block seeds
 *                        and long shared blocks = each block's matrix-vector product tiled into
 *                        128 x 128 Hankel blocks; long keys through the 3-for-4 split.
 *   SSBH_ENGINE_AUTO   : the plan's default: TENSOR (unless ssbh_set_plan_overrides says LOP3).
 * Both engines produce identical keys. ssbh_plan_engine returns the engine in use. */
#define SSBH_ENGINE_AUTO 0
#define SSBH_ENGINE_LOP3 1
#define SSBH_ENGINE_TENSOR 2
ssbh_status ssbh_plan_set_engine(ssbh_plan* plan, int engine);
int ssbh_plan_engine(const ssbh_plan* plan);
/* Name of the hash kernel a plan launches: "k_toeplitz_f4" (shared seeds, all-blocks GEMM),
 * "k_toeplitz_mma_pb" (per-block seeds / long shared blocks, tiled), either with "+split"
 * when the 3-for-4 split runs (the leaves' kernel), or "k_toeplitz_hash" (LOP3). */
const char* ssbh_plan_hash_kernel(const ssbh_plan* plan);

/* Plan-construction overrides: explicit testing / A-B hooks that steer which code path a plan
 * takes at sizes where the cost models would not (the parity suite forces every path at small
 * sizes). Never read from the environment. Process-wide; plans copy them when created;
 * NULL restores the defaults. */
typedef struct ssbh_plan_overrides {
    int32_t engine;             /* SSBH_ENGINE_AUTO (default) / _LOP3 / _TENSOR */
    int32_t split_levels;       /* -1: cost model; 0: no 3-for-4 split; L: force L levels */
    int32_t split_tiled_leaves; /* 0: shared-seed leaves on the all-blocks GEMM; 1: tiled kernel */
    int32_t shared_tiled;       /* -1: heuristic (mean n_j >= 620 K bits); 0/1: force the tiled
                                   kernel off/on for shared seeds */
    int32_t buckets;            /* -1: heuristic (>= 4096 owned blocks); 0/1: force the
                                   two-level sampler split off/on */
    uint32_t split_budget_mb;   /* leaf buffer budget; 0: default 8192 MiB */
    int32_t scatter_window;     /* ranked scatter (in-memory single-level plans): 0: model (a
                                   shared-memory window of mean cell + 6 sigma when a (chunk,
                                   block) cell holds >= 8 rounds); W > 0: force W window words;
                                   -1: per-bit global atomics */
} ssbh_plan_overrides;
ssbh_status ssbh_set_plan_overrides(const ssbh_plan_overrides* overrides);
ssbh_status ssbh_get_plan_overrides(ssbh_plan_overrides* overrides);
/* 3-for-4 Toeplitz split of long shared-seed blocks (csrc/toeplitz_split.cu; a B200 addition,
   no reference counterpart): levels L (0 = direct product), squares T of k positions per block,
   owned blocks per leaf batch. The hash then runs T*3^L leaf products of k/2^L per block plus
   the remainder past T*k. */
ssbh_status ssbh_plan_split_geometry(const ssbh_plan* plan, uint32_t* levels, uint32_t* squares,
                                     uint32_t* batch_blocks);

/* Host-buffer entry point (what a reference caller binds): input host words (n bits),
 * out_key host words (ceil(owned*k/64)), out_lengths host (owned entries, may be NULL).
 * H2D, device run, D2H; synchronous. */
ssbh_status ssbh_extract(const ssbh_extract_params* params, const uint64_t* input,
                         uint64_t* out_key, uint64_t* out_lengths, ssbh_extract_stats* stats);
/* Same through an existing plan (no re-allocation); copies through pinned staging. */
ssbh_status ssbh_plan_run_host(ssbh_plan* plan, const uint64_t* input, uint64_t* out_key,
                               uint64_t* out_lengths, ssbh_extract_stats* stats);

/* Sifted runs (the reference's keep flags, sift_partition sampling.cpp:27-39 as used by
 * run_extraction pipeline.cpp:109-112): only rounds with keep bit set join their sub-block;
 * n_j counts kept rounds. keep is bit-packed like the input (bit i = keep[i]; device: uint32
 * words, host: uint64 words); NULL keeps every round. */
ssbh_status ssbh_plan_run_device_sifted(ssbh_plan* plan, const uint32_t* d_input,
                                        const uint32_t* d_keep, uint32_t* d_key,
                                        uint64_t* d_lengths, const uint64_t* samp_key,
                                        const uint64_t* hash_key, void* stream);
ssbh_status ssbh_plan_run_host_sifted(ssbh_plan* plan, const uint64_t* input,
                                      const uint64_t* keep, uint64_t* out_key,
                                      uint64_t* out_lengths, ssbh_extract_stats* stats);
ssbh_status ssbh_extract_sifted(const ssbh_extract_params* params, const uint64_t* input,
                                const uint64_t* keep, uint64_t* out_key, uint64_t* out_lengths,
                                ssbh_extract_stats* stats);

/* Streaming plans — inputs fed in pieces (BASELINE config 5: 2^37 rounds "streamed in 8
 * chunks"; also any input larger than device memory). No per-round payload buffer: V_i is
 * recomputed by Threefry in the scatter pass. Every chunk except the last holds exactly
 * chunk_bits rounds (a multiple of 1024), each chunk once. Plans with fewer than 4096 owned
 * blocks take their chunks in any order; larger plans (two-level partition, config 5) keep the
 * blocks' running lengths from chunk to chunk instead of counting the whole input first and
 * take them in order 0, 1, 2, ... (another index -> SSBH_INVALID_ARGUMENT).
 *   ssbh_plan_stream_begin  : count pass over all n rounds (needs no input), scan, layout
 *                             (two-level plans: only zeroes the blocks' regions)
 *   ssbh_plan_stream_chunk  : chunk c's rounds [c*chunk_bits, ...) as uint32 words on device
 *   ssbh_plan_stream_finish : (two-level plans: lengths, layout, block reversal,) seeds, hash,
 *                             concatenation into d_key (+ lengths)
 * then ssbh_plan_check as for in-memory plans. */
ssbh_status ssbh_plan_create_streaming(const ssbh_extract_params* params, uint64_t chunk_bits,
                                       ssbh_plan** plan);
ssbh_status ssbh_plan_stream_begin(ssbh_plan* plan, const uint64_t* samp_key,
                                   const uint64_t* hash_key, void* stream);
ssbh_status ssbh_plan_stream_chunk(ssbh_plan* plan, uint64_t chunk_index, const uint32_t* d_chunk,
                                   void* stream);
ssbh_status ssbh_plan_stream_finish(ssbh_plan* plan, uint32_t* d_key, uint64_t* d_lengths,
                                    void* stream);

/* ------------------------------------------------------- multi-GPU shards (one process/GPU)
 * Sharded sampling: rank r of W owns blocks [r*s/W, (r+1)*s/W) and samples only
 * its slice of rounds [slice_first, slice_first + slice_rounds); every sampled round's
 * payload is stored straight into the owning rank's receive buffer through NVLink peer
 * memory (CUDA IPC mappings) — the all-to-all is fused into the stable owner split — and each
 * owner then partitions, seeds and hashes only its own rounds. Per run:
 *   ssbh_shard_sample(slice input)  -> this rank's per-owner round counts (W values)
 *   [host: all-gather the W x W count matrix; row r = rank r's counts]
 *   ssbh_shard_exchange(matrix)     -> peer stores; returns when this rank's stores are done
 *   [host: barrier across ranks]
 *   ssbh_shard_finish(d_key)        -> the owned blocks' key slice (concatenate in rank order)
 * Setup once: ssbh_shard_ipc_handle on every rank, all-gather the handles (W x 64 bytes),
 * ssbh_shard_open_peers. No kernel waits on another rank. */
#define SSBH_IPC_HANDLE_BYTES 64
typedef struct ssbh_shard ssbh_shard;
ssbh_status ssbh_shard_create(const ssbh_extract_params* params, uint32_t rank, uint32_t world,
                              ssbh_shard** shard);
ssbh_status ssbh_shard_destroy(ssbh_shard* shard);
ssbh_status ssbh_shard_info(const ssbh_shard* shard, uint64_t* slice_first,
                            uint64_t* slice_rounds, uint32_t* block_first, uint32_t* block_count);
ssbh_status ssbh_shard_ipc_handle(ssbh_shard* shard, void* handle_out);
ssbh_status ssbh_shard_open_peers(ssbh_shard* shard, const void* handles);
ssbh_status ssbh_shard_sample(ssbh_shard* shard, const uint32_t* d_slice_input,
                              const uint64_t* samp_key, uint64_t* owner_counts, void* stream);
ssbh_status ssbh_shard_exchange(ssbh_shard* shard, const uint64_t* counts, void* stream);
ssbh_status ssbh_shard_finish(ssbh_shard* shard, uint32_t* d_key, uint64_t* d_lengths,
                              const uint64_t* hash_key, void* stream);
ssbh_status ssbh_shard_check(ssbh_shard* shard, ssbh_extract_stats* stats);
ssbh_status ssbh_shard_set_timing(ssbh_shard* shard, int enable);
/* Hash kernel of the shard's owner plan (see ssbh_plan_hash_kernel). */
const char* ssbh_shard_hash_kernel(const ssbh_shard* shard);
/* Split geometry of the shard's owner plan (see ssbh_plan_split_geometry). */
ssbh_status ssbh_shard_split_geometry(const ssbh_shard* shard, uint32_t* levels,
                                      uint32_t* squares, uint32_t* batch_blocks);

/* The same sharded extraction driven from ONE process over several GPUs (the reference's
 * callers are single-process C++): rank r runs on devices[r] (entries may repeat), receive
 * buffers are exchanged as device pointers with peer access enabled between distinct devices,
 * one host thread per rank, thread joins as the barriers. Host input / key / lengths as in
 * ssbh_extract; the whole key (block_first = 0, all blocks). ndev == 1 is ssbh_extract on
 * devices[0]. stats: hash_word_ops and min/max length over all blocks. */
ssbh_status ssbh_extract_multi(const ssbh_extract_params* params, const uint64_t* input,
                               const int* devices, uint32_t ndev, uint64_t* out_key,
                               uint64_t* out_lengths, ssbh_extract_stats* stats);

/* ----------------------------------------- protocol rounds (run_extraction's hash stage)
 * RoundRecord bytes (proj/include/ssbh/pipeline.hpp:15-38): bit 0 BasisAx, 1 BasisBx,
 * 2 Detected, 3 BitA, 4 BitB, 5 IsTest; is_key_round = Detected && !BasisAx && !BasisBx. */
typedef struct {
    uint64_t n_rounds;
    double p_x;   /* test-basis probability */
    double e_ph;  /* phase error rate (X/X flips) */
    double e_bit; /* bit error rate (Z/Z flips) */
    double p_det; /* detection probability */
} ssbh_round_params;

/* Reference: simulate_rounds — pipeline.hpp:41, pipeline.cpp:20-55 (streams "basis-a",
 * "basis-b", "detect", "bit-a", "noise" of `seed`). One byte per round; _device writes
 * d_rounds on `stream` (asynchronous), the host form copies back (synchronous). Parameter
 * ranges are the caller's (Bbm92Params::validate); probabilities outside [0,1] ->
 * SSBH_INVALID_ARGUMENT as bernoulli throws (prf.cpp:97-98). */
ssbh_status ssbh_simulate_rounds_device(const ssbh_round_params* params, const uint64_t seed[4],
                                        uint8_t* d_rounds, void* stream);
ssbh_status ssbh_simulate_rounds(const ssbh_round_params* params, const uint64_t seed[4],
                                 uint8_t* rounds);

/* run_extraction after the key-length solver (pipeline.cpp:84-136): statistics check on the
 * test rounds, sift of the key rounds, assign_subblocks(n, s, seed), oversize abort,
 * bits_per_block = key_length / s, per-block seeds KeyedStream(seed, "hash-seed", j),
 * toeplitz_hash of gathered bit_a, concatenation. key_length is the caller's
 * key_length(params, scenario).length (0 when infeasible): the finite-key solver is the
 * reference's host code and stays there. */
typedef struct {
    uint32_t n_subblocks;   /* plan.n_subblocks */
    uint32_t pad;
    uint64_t block_limit;   /* plan.block_limit (must be set) */
    uint64_t seed[4];       /* plan.seed: sampling and hash-seed streams */
    double eps_abort;       /* plan.eps_abort */
    double eps_sec, p_x, eta_tol, q_tol; /* Bbm92Params */
    uint64_t key_length;    /* kl.length */
} ssbh_extraction_params;

typedef struct {
    int32_t abort;          /* 0 None, 1 OversizeBlock, 2 Statistics (ExtractionReport::Abort) */
    uint32_t pad;
    uint64_t bits_per_block;
    uint64_t key_bits;      /* bits written to out_key (s * bits_per_block, or 0) */
    double total_epsilon;
    double hash_seconds;    /* device time of seed generation + hash (CUDA events) */
    uint64_t test_rounds;
    uint64_t phase_errors;  /* c1: detected test rounds with bit_a != bit_b */
    uint64_t no_detections; /* c2: undetected test rounds */
    uint64_t key_rounds;    /* sifted length */
    int32_t lengths_valid;  /* out_lengths written (not for a statistics abort) */
    uint32_t pad2;
} ssbh_extraction_result;

/* Host rounds (n bytes); out_key capacity ceil(key_length_floor / 64) words where
 * key_length_floor = s * (key_length / s); out_lengths has s entries. Synchronous. */
ssbh_status ssbh_run_extraction(const uint8_t* rounds, uint64_t n_rounds,
                                const ssbh_extraction_params* params, uint64_t* out_key,
                                uint64_t* out_lengths, ssbh_extraction_result* result);
/* Same from device-resident rounds (e.g. ssbh_simulate_rounds_device); host outputs. */
ssbh_status ssbh_run_extraction_device(const uint8_t* d_rounds, uint64_t n_rounds,
                                       const ssbh_extraction_params* params, uint64_t* out_key,
                                       uint64_t* out_lengths, ssbh_extraction_result* result);

/* Synthetic input on the device: p == 0.5 -> KeyedStream(key,"input").bits(n);
 * else bit i = bernoulli(p, i) of the same stream. d_out: ceil(n/32) uint32 words. */
ssbh_status ssbh_make_input_device(const uint64_t key[4], double p, uint64_t nbits,
                                   uint32_t* d_out, void* stream);

/* Diagnostics (not a reference interface): measured LOP3 lane-ops/s of the current device
 * (the int-ALU roofline denominator of the hash kernel) over one timed launch. */
ssbh_status ssbh_measure_lop3_peak(uint32_t iters, double* lop3_per_s, double* ms);
/* FP4 roofline of the shared-seed tensor kernel: tcgen05.mma kind::mxf4 (E2M1, unit UE8M0
 * scales) 128x256x64 back to back with the hash kernel's operand layouts. */
ssbh_status ssbh_measure_mma_f4_peak(uint32_t iters, double* macs_per_s, double* ms);
/* FP4 probe: mode 0 = rate (plain tiles), 1 = exactness (every MMA adds exactly 1 to every f32
 * accumulator; *mismatches counts elements != iters after `iters` MMAs, *sample_bits = one
 * accumulator's bits), 2 = rate with the hash kernel's layouts. */
ssbh_status ssbh_probe_mma_f4(uint32_t iters, int mode, double* macs_per_s, double* ms,
                              uint32_t* mismatches, uint32_t* sample_bits);

#ifdef __cplusplus
}
#endif
#endif /* SSBH_CUDA_H */
