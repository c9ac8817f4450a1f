// ssbh_cli.cpp — `ssbh-b200`, the B200 counterpart of the reference CLI's hot-path commands
// (proj/tools/ssbh_main.cpp), on the drop-in API (libssbh.so -> libssbh_cuda.so):
//
//   ssbh-b200 extract --in FILE --in-bits N --out-bits L [--ns S] [--seed HEX64]
//                     [--eps-abort E] [--out FILE] [--partition-csv FILE] [--gpus G]
//       file mode of cmd_extract (ssbh_main.cpp:306-345): the master seed keys both the
//       sampling and the per-block "hash-seed" streams (sub = j), L/S bits per block, strict
//       oversize abort against block_limit(N, 1/S, eps_abort, S) (N when S == 1).
//       --gpus G > 1: one process over GPUs 0..G-1 (ssbh_extract_multi).
//   ssbh-b200 extract --simulate --n-rounds N --key-length L [--ns S] [--seed HEX64]
//                     [--p-x P] [--e-ph E] [--e-bit E] [--q-tol Q] [--eta-tol T] [--p-det D]
//                     [--eps-sec E] [--eps-abort E] [--out FILE] [--partition-csv FILE]
//       simulate mode of cmd_extract (ssbh_main.cpp:274-303): simulate_rounds + run_extraction
//       on the GPU. L is key_length(params, scenario).length from the reference's finite-key
//       solver (out of scope here, see pipeline.hpp); the block cap is block_limit(N,
//       p_z^2 p_det / S, eps_abort, S) as the reference derives it.
//   ssbh-b200 limit --n N --p-sift P --eps-abort E [--m M]
//       cmd_limit (ssbh_main.cpp:435-440): prints block_limit(N, P, E, M).
//   ssbh-b200 bench --sizes A,B,... [--ns S] [--seed HEX64] [--out-ratio R]
//       cmd_bench (ssbh_main.cpp:368-426): direct hash of the whole input vs sub-block
//       hashing, measured on the GPU, beside the FPGA cycle-model ratio
//       (cycle_estimate / timing_model semantics, pipeline.cpp:142-163).
//
// Exit codes follow ssbh_main.cpp:26-33: 0 ok, 2 parse/invalid, 3 infeasible,
// 4 oversize abort, 5 statistics abort, 6 io; device failures exit 7.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "ssbh/bitstring.hpp"
#include "ssbh/errors.hpp"
#include "ssbh/extract.hpp"
#include "ssbh/pipeline.hpp"
#include "ssbh/prf.hpp"
#include "ssbh/sampling.hpp"
#include "ssbh/toeplitz.hpp"

using namespace ssbh;

namespace {

enum : int {
    kOk = 0,
    kParse = 2,
    kInfeasible = 3,
    kAbortOversize = 4,
    kAbortStats = 5,
    kIo = 6,
    kDevice = 7
};

struct Args {
    std::string cmd, in, out, partition_csv, seed_hex = std::string(64, '0');
    std::uint64_t in_bits = 0, out_bits = 0;
    std::uint32_t ns = 1, gpus = 1;
    double eps_abort = 1e-8, out_ratio = 0.06303;
    int repeats = 5;  // bench: median of this many timed calls per size
    std::vector<std::uint64_t> sizes;
    // simulate mode (Bbm92Params defaults, bbm92.hpp:14-26) and limit
    bool simulate = false;
    Bbm92Params params;
    std::uint64_t key_length = 0, limit_n = 0, limit_m = 1;
    bool have_key_length = false;
    double p_sift = 0;
};

std::uint64_t parse_u64(const std::string& s) {
    std::size_t pos = 0;
    const unsigned long long v = std::stoull(s, &pos);
    if (pos != s.size()) throw std::invalid_argument("not an integer: " + s);
    return v;
}

Args parse(int argc, char** argv) {
    if (argc < 2) throw std::invalid_argument("usage: ssbh-b200 extract|limit|bench [options]");
    Args a;
    a.cmd = argv[1];
    for (int i = 2; i < argc; ++i) {
        const std::string f = argv[i];
        auto val = [&]() -> std::string {
            if (i + 1 >= argc) throw std::invalid_argument("missing value for " + f);
            return argv[++i];
        };
        if (f == "--in") a.in = val();
        else if (f == "--out") a.out = val();
        else if (f == "--partition-csv") a.partition_csv = val();
        else if (f == "--seed") a.seed_hex = val();
        else if (f == "--in-bits") a.in_bits = parse_u64(val());
        else if (f == "--out-bits") a.out_bits = parse_u64(val());
        else if (f == "--ns") a.ns = static_cast<std::uint32_t>(parse_u64(val()));
        else if (f == "--gpus") a.gpus = static_cast<std::uint32_t>(parse_u64(val()));
        else if (f == "--eps-abort") a.eps_abort = std::stod(val());
        else if (f == "--out-ratio") a.out_ratio = std::stod(val());
        else if (f == "--repeats") a.repeats = std::max(1, std::stoi(val()));
        else if (f == "--simulate") a.simulate = true;
        else if (f == "--n-rounds") a.params.n_rounds = parse_u64(val());
        else if (f == "--p-x") a.params.p_x = std::stod(val());
        else if (f == "--e-ph") a.params.e_ph = std::stod(val());
        else if (f == "--e-bit") a.params.e_bit = std::stod(val());
        else if (f == "--q-tol") a.params.q_tol = std::stod(val());
        else if (f == "--eta-tol") a.params.eta_tol = std::stod(val());
        else if (f == "--p-det") a.params.p_det = std::stod(val());
        else if (f == "--eps-sec") a.params.eps_sec = std::stod(val());
        else if (f == "--key-length") {
            a.key_length = parse_u64(val());
            a.have_key_length = true;
        } else if (f == "--n") a.limit_n = parse_u64(val());
        else if (f == "--m") a.limit_m = parse_u64(val());
        else if (f == "--p-sift") a.p_sift = std::stod(val());
        else if (f == "--sizes") {
            std::stringstream ss(val());
            std::string tok;
            while (std::getline(ss, tok, ',')) a.sizes.push_back(parse_u64(tok));
        } else
            throw std::invalid_argument("unknown flag " + f);
    }
    return a;
}

void emit(const std::string& path, const std::string& text) {
    if (path.empty()) {
        std::fwrite(text.data(), 1, text.size(), stdout);
        return;
    }
    std::ofstream o(path, std::ios::binary);
    if (!o) throw io_error("cannot open output: " + path);
    o << text;
}

int cmd_extract(const Args& a) {
    if (a.in.empty() || a.in_bits == 0)
        throw std::invalid_argument("extract: need --in with --in-bits");
    if (a.out_bits == 0) throw std::invalid_argument("extract: file mode needs --out-bits");
    if (a.ns == 0) throw std::invalid_argument("assign_subblocks: n_subblocks must be positive");
    const MasterSeed seed = MasterSeed::from_hex(a.seed_hex);
    const BitString data = BitString::read_file(a.in, a.in_bits);
    const std::uint64_t limit =
        a.ns == 1 ? a.in_bits
                  : block_limit(a.in_bits, 1.0 / static_cast<double>(a.ns), a.eps_abort, a.ns);
    std::string report = "# b200: seed " + seed.to_hex() + ", ns " + std::to_string(a.ns) + "\n";
    report += "mode: file\n";
    report += "block_limit: " + std::to_string(limit) + "\n";
    ExtractOptions opt;
    opt.seed_mode = SeedMode::PerBlock;  // KeyedStream(seed, "hash-seed", j)
    opt.block_limit = limit;
    for (std::uint32_t g = 0; a.gpus > 1 && g < a.gpus; ++g)  // one process over N GPUs
        opt.devices.push_back(static_cast<int>(g));
    const auto t0 = std::chrono::steady_clock::now();
    const ExtractResult r = extract(data, a.ns, a.out_bits / a.ns, seed, seed, opt);
    const double secs =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (r.aborted) {  // no partition dump on an abort (ssbh_main.cpp:347-357)
        report += "abort: oversize_block\n";
        emit("", report);
        return kAbortOversize;
    }
    if (!a.partition_csv.empty()) {
        const Partition part = assign_subblocks(a.in_bits, a.ns, seed);
        std::string dump = "round_index,v_i,kept\n";
        for (std::uint64_t i = 0; i < a.in_bits; ++i)
            dump += std::to_string(i) + "," + std::to_string(part.assignment[i]) + ",1\n";
        emit(a.partition_csv, dump);
    }
    report += "key_length_bits: " + std::to_string(r.key.size()) + "\n";
    report += "hash_seconds: " + std::to_string(secs) + "\n";
    report += "device_ms: " + std::to_string(r.device_ms) + "\n";
    if (!a.out.empty()) r.key.write_file(a.out);
    emit("", report);
    return kOk;
}

// simulate mode (ssbh_main.cpp:274-303): rounds and the extraction's data path on the GPU
int cmd_extract_simulate(const Args& a) {
    if (!a.have_key_length)
        throw std::invalid_argument(
            "extract --simulate: --key-length required (the finite-key solver stays host-side)");
    if (a.ns == 0) throw std::invalid_argument("scenario: n_subblocks must be positive");
    const MasterSeed seed = MasterSeed::from_hex(a.seed_hex);
    Bbm92Params p = a.params;
    p.eps_abort = a.eps_abort;
    const auto rounds = simulate_rounds(p, seed);
    SamplingPlan plan;
    plan.n_subblocks = a.ns;
    plan.eps_abort = p.eps_abort;
    const double p_sift = p.p_z() * p.p_z() * p.p_det / static_cast<double>(a.ns);
    plan.block_limit = block_limit(p.n_rounds, p_sift, plan.eps_abort, a.ns);
    plan.seed = seed;
    const ExtractionReport rep = run_extraction(rounds, plan, p, a.key_length);
    std::string report = "# b200: seed " + seed.to_hex() + ", ns " + std::to_string(a.ns) + "\n";
    report += "mode: simulate\n";
    report += "block_limit: " + std::to_string(plan.block_limit) + "\n";
    report += "bits_per_block: " + std::to_string(rep.bits_per_block) + "\n";
    report += "key_length_bits: " + std::to_string(rep.key.size()) + "\n";
    char buf[64];
    std::snprintf(buf, sizeof buf, "%.17g", rep.total_epsilon);
    report += std::string("total_epsilon: ") + buf + "\n";
    report += "modeled_cycles: " + std::to_string(rep.cycle_count) + "\n";
    std::snprintf(buf, sizeof buf, "%.6g", rep.wall_seconds);
    report += std::string("hash_seconds: ") + buf + "\n";
    report += "block_lengths:";
    for (const auto b : rep.block_lengths) report += " " + std::to_string(b);
    report += "\n";
    if (rep.abort == ExtractionReport::Abort::OversizeBlock) {
        report += "abort: oversize_block\n";
        emit("", report);
        return kAbortOversize;
    }
    if (rep.abort == ExtractionReport::Abort::Statistics) {
        report += "abort: statistics\n";
        emit("", report);
        return kAbortStats;
    }
    if (!a.partition_csv.empty()) {
        const Partition part = assign_subblocks(p.n_rounds, a.ns, seed);
        std::string dump = "round_index,v_i,kept\n";
        for (std::uint64_t i = 0; i < rounds.size(); ++i)
            dump += std::to_string(i) + "," + std::to_string(part.assignment[i]) + "," +
                    (rounds[i].is_key_round() ? "1" : "0") + "\n";
        emit(a.partition_csv, dump);
    }
    if (!a.out.empty()) rep.key.write_file(a.out);
    emit("", report);
    return kOk;
}

int cmd_limit(const Args& a) {
    std::printf("%llu\n", static_cast<unsigned long long>(
                               block_limit(a.limit_n, a.p_sift, a.eps_abort, a.limit_m)));
    return kOk;
}

// FPGA cycle model of the reference: full vs splitting(ns) padded to the abort limit
// (timing_model, pipeline.cpp:139-160).
std::uint64_t model_cycles(std::uint64_t in, std::uint64_t out, std::uint32_t ns, double eps) {
    const BlockingParams blk;
    return timing_model(in, out, ns == 1 ? Scenario::full() : Scenario::splitting(ns), blk, eps);
}

int cmd_bench(const Args& a) {
    if (a.sizes.empty()) throw std::invalid_argument("bench: --sizes required");
    const MasterSeed seed = MasterSeed::from_hex(a.seed_hex);
    // The reference's columns (ssbh_main.cpp:371) + the same two timings with the operands
    // resident on the device (PreparedHashBatch::run): the reference times toeplitz_hash on
    // operands that sit where it computes; through host containers both GPU calls are bound by
    // the host-to-device copy of input and seed (2 x size/8 bytes either way).
    std::string out =
        "size_bits,full_seconds,split_seconds,measured_ratio,modeled_ratio,"
        "full_device_seconds,split_device_seconds,device_ratio\n";
    for (const std::uint64_t size : a.sizes) {
        if (size == 0) throw std::invalid_argument("bench: sizes must be positive");
        const std::uint64_t m_full =
            std::max<std::uint64_t>(1, static_cast<std::uint64_t>(size * a.out_ratio));
        const BitString input = KeyedStream(seed, "bench-input").bits(size);
        const ToeplitzSeed fseed(KeyedStream(seed, "bench-seed-full").bits(m_full + size - 1),
                                 m_full, size);
        // median of a.repeats timed calls each (the reference times one call, :381-385)
        auto median_s = [&](auto&& fn) {
            fn();  // warm-up (module load, the per-thread device arena)
            std::vector<double> t(a.repeats);
            for (double& v : t) {
                const auto t0 = std::chrono::steady_clock::now();
                fn();
                v = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            }
            std::sort(t.begin(), t.end());
            return t[t.size() / 2];
        };
        const double full_s = median_s([&] { (void)toeplitz_hash(fseed, input); });
        // split: partition + gather + per-block seeds untimed (ssbh_main.cpp:388-404), then
        // the hashing of every block timed — one batched launch on the GPU (:405-410)
        const std::uint64_t m_block = std::max<std::uint64_t>(1, m_full / a.ns);
        const Partition part = assign_subblocks(size, a.ns, seed);
        const SiftedPartition sifted =
            sift_partition(std::vector<std::uint8_t>(size, 1), part);
        std::vector<BitString> inputs(a.ns);
        std::vector<ToeplitzSeed> seeds;
        for (std::uint32_t j = 0; j < a.ns; ++j) {
            inputs[j] = BitString(sifted.blocks[j].size());
            for (std::uint64_t q = 0; q < sifted.blocks[j].size(); ++q)
                if (input.get(sifted.blocks[j][q])) inputs[j].set(q, true);
            seeds.emplace_back(KeyedStream(seed, "hash-seed", j).bits(m_block + inputs[j].size() - 1),
                               m_block, inputs[j].size());
        }
        const double split_s = median_s([&] { (void)toeplitz_hash_batch(seeds, inputs); });
        double full_dev_s = 0, split_dev_s = 0;
        {
            const PreparedHashBatch full_dev({fseed}, {input});
            full_dev_s = median_s([&] { (void)full_dev.run(); });
            const PreparedHashBatch split_dev(seeds, inputs);
            split_dev_s = median_s([&] { (void)split_dev.run(); });
        }
        const double modeled = static_cast<double>(model_cycles(size, m_full, 1, a.eps_abort)) /
                               static_cast<double>(model_cycles(size, m_block * a.ns, a.ns,
                                                                a.eps_abort));
        char line[320];
        std::snprintf(line, sizeof line, "%llu,%.6g,%.6g,%.6g,%.6g,%.6g,%.6g,%.6g\n",
                      static_cast<unsigned long long>(size), full_s, split_s, full_s / split_s,
                      modeled, full_dev_s, split_dev_s, full_dev_s / split_dev_s);
        out += line;
    }
    emit(a.out, out);
    return kOk;
}

}  // namespace

int main(int argc, char** argv) {
    try {
        const Args a = parse(argc, argv);
        if (a.cmd == "extract") return a.simulate ? cmd_extract_simulate(a) : cmd_extract(a);
        if (a.cmd == "limit") return cmd_limit(a);
        if (a.cmd == "bench") return cmd_bench(a);
        throw std::invalid_argument("unknown command " + a.cmd);
    } catch (const infeasible_error& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return kInfeasible;
    } catch (const io_error& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return kIo;
    } catch (const device_error& e) {
        std::fprintf(stderr, "device error: %s\n", e.what());
        return kDevice;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return kParse;
    }
}
