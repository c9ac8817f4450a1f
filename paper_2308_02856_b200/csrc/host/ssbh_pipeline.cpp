// ssbh_pipeline.cpp — include/ssbh/{bbm92,pipeline}.hpp over the C-ABI: the protocol-round
// simulation and run_extraction's hash stage on the GPU, plus the host-scalar pieces
// around them (parameter validation, scenario constructors, the FPGA timing model).
#include <cstring>
#include <stdexcept>

#include "ssbh/bbm92.hpp"
#include "ssbh/errors.hpp"
#include "ssbh/pipeline.hpp"
#include "ssbh_cuda.h"

namespace ssbh {

namespace {
inline void check(ssbh_status s) { detail::throw_status(s); }
}  // namespace

// ------------------------------------------------------------------- parameter types
// Ranges of bbm92.cpp:19-44 (the messages are part of the error contract).
void Bbm92Params::validate() const {
    auto bad = [](const char* what) { throw std::invalid_argument(what); };
    if (n_rounds == 0) bad("bbm92: n_rounds must be positive");
    if (!(p_x > 0.0 && p_x < 1.0)) bad("bbm92: p_x must lie in (0,1)");
    if (!(e_ph >= 0.0 && e_ph < 0.5)) bad("bbm92: e_ph must lie in [0,0.5)");
    if (!(e_bit >= 0.0 && e_bit <= 0.5)) bad("bbm92: e_bit must lie in [0,0.5]");
    if (!(q_tol >= e_ph && q_tol < 0.5)) bad("bbm92: q_tol must lie in [e_ph, 0.5)");
    if (!(eta_tol > 0.0 && eta_tol <= 1.0)) bad("bbm92: eta_tol must lie in (0,1]");
    if (!(f_ec >= 1.0)) bad("bbm92: f_ec must be at least 1");
    if (!(p_det >= 0.0 && p_det <= 1.0)) bad("bbm92: p_det must lie in [0,1]");
    if (d_x < 2) bad("bbm92: d_x must be at least 2");
    if (!(eps_sec > 0.0 && eps_sec < 1.0)) bad("bbm92: eps_sec must lie in (0,1)");
    if (!(eps_abort >= 0.0 && eps_abort < 1.0)) bad("bbm92: eps_abort must lie in [0,1)");
    if (!(p_omega > 0.0 && p_omega <= 1.0)) bad("bbm92: p_omega must lie in (0,1]");
}

Scenario Scenario::splitting(std::uint32_t ns) {
    if (ns == 0) throw std::invalid_argument("scenario: n_subblocks must be positive");
    return {Kind::Splitting, ns};
}

Scenario Scenario::small_block(std::uint32_t ns) {
    if (ns == 0) throw std::invalid_argument("scenario: n_subblocks must be positive");
    return {Kind::SmallBlock, ns};
}

const char* Scenario::name() const {
    return kind == Kind::Full ? "full" : kind == Kind::Splitting ? "splitting" : "smallblock";
}

// ---------------------------------------------------------------------- rounds (GPU)
std::vector<RoundRecord> simulate_rounds(const Bbm92Params& params, const MasterSeed& seed) {
    params.validate();
    ssbh_round_params rp{params.n_rounds, params.p_x, params.e_ph, params.e_bit, params.p_det};
    std::vector<RoundRecord> rounds(params.n_rounds);
    check(ssbh_simulate_rounds(&rp, seed.words.data(),
                               reinterpret_cast<std::uint8_t*>(rounds.data())));
    return rounds;
}

// ---------------------------------------------------------------------- timing model
// pipeline.cpp:139-160: Full -> one product; Splitting -> ns products padded to the block
// cap (derived from eps_abort unless overridden); SmallBlock -> ns products of n/ns.
std::uint64_t timing_model(std::uint64_t input_len, std::uint64_t output_len,
                           const Scenario& scenario, const BlockingParams& blocking,
                           double eps_abort, std::uint64_t block_limit_override,
                           bool pad_to_limit) {
    const std::uint64_t ns = scenario.n_subblocks;
    auto ceil_div = [](std::uint64_t a, std::uint64_t b) { return (a + b - 1) / b; };
    if (scenario.kind == Scenario::Kind::Full)
        return cycle_estimate(input_len, output_len, blocking.m_prime);
    if (scenario.kind == Scenario::Kind::Splitting) {
        std::uint64_t cap = block_limit_override;
        if (cap == 0)
            cap = ns == 1 ? input_len
                          : block_limit(input_len, 1.0 / static_cast<double>(ns), eps_abort, ns);
        const std::uint64_t per_in = pad_to_limit ? cap : ceil_div(input_len, ns);
        return ns * cycle_estimate(per_in, ceil_div(output_len, ns), blocking.m_prime);
    }
    return ns * cycle_estimate(ceil_div(input_len, ns), ceil_div(output_len, ns),
                               blocking.m_prime);
}

// -------------------------------------------------------------------- run_extraction
namespace {
// hash_bits: the solver's key length when feasible, else 0 (bits_per_block = hash_bits / ns);
// model_bits: the solver's length as the reference feeds it to timing_model (pipeline.cpp:118)
ExtractionReport run_extraction_impl(const std::vector<RoundRecord>& rounds,
                                     const SamplingPlan& plan, const Bbm92Params& params,
                                     std::uint64_t key_length, std::uint64_t model_bits,
                                     const BlockingParams& blocking);
}  // namespace

// The reference's signature (pipeline.hpp:56-60). key_length is the reference's own solver
// (proj/src/bbm92.cpp), bound weakly: linked by callers that keep the reference's security
// library, absent otherwise.
KeyLengthResult key_length(const Bbm92Params& params, const Scenario& scenario)
    __attribute__((weak));

ExtractionReport run_extraction(const std::vector<RoundRecord>& rounds, const SamplingPlan& plan,
                                const Bbm92Params& params, const BlockingParams& blocking) {
    if (!&key_length)
        throw std::logic_error(
            "run_extraction: the finite-key solver ssbh::key_length (the reference's "
            "bbm92.cpp) is not linked; link it or pass the key length explicitly");
    params.validate();
    if (plan.n_subblocks == 0)
        throw std::invalid_argument("run_extraction: plan.n_subblocks must be positive");
    const std::uint32_t ns = plan.n_subblocks;
    const KeyLengthResult kl =
        key_length(params, ns == 1 ? Scenario::full() : Scenario::splitting(ns));
    return run_extraction_impl(rounds, plan, params, kl.feasible ? kl.length : 0, kl.length,
                               blocking);
}

ExtractionReport run_extraction(const std::vector<RoundRecord>& rounds, const SamplingPlan& plan,
                                const Bbm92Params& params, std::uint64_t key_length,
                                const BlockingParams& blocking) {
    return run_extraction_impl(rounds, plan, params, key_length, key_length, blocking);
}

namespace {
ExtractionReport run_extraction_impl(const std::vector<RoundRecord>& rounds,
                                     const SamplingPlan& plan, const Bbm92Params& params,
                                     std::uint64_t key_length, std::uint64_t model_bits,
                                     const BlockingParams& blocking) {
    params.validate();
    if (plan.n_subblocks == 0)
        throw std::invalid_argument("run_extraction: plan.n_subblocks must be positive");
    if (plan.block_limit == 0)
        throw std::invalid_argument("run_extraction: plan.block_limit must be set");
    if (rounds.size() != params.n_rounds)
        throw std::invalid_argument("run_extraction: round count does not match params");

    const std::uint32_t ns = plan.n_subblocks;
    ssbh_extraction_params ep{};
    ep.n_subblocks = ns;
    ep.block_limit = plan.block_limit;
    std::memcpy(ep.seed, plan.seed.words.data(), 32);
    ep.eps_abort = plan.eps_abort;
    ep.eps_sec = params.eps_sec;
    ep.p_x = params.p_x;
    ep.eta_tol = params.eta_tol;
    ep.q_tol = params.q_tol;
    ep.key_length = key_length;

    ExtractionReport report;
    std::vector<std::uint64_t> lengths(ns, 0);
    BitString key(static_cast<std::uint64_t>(ns) * (key_length / ns));
    ssbh_extraction_result res{};
    check(ssbh_run_extraction(reinterpret_cast<const std::uint8_t*>(rounds.data()), rounds.size(),
                              &ep, key.words().data(), lengths.data(), &res));
    report.total_epsilon = res.total_epsilon;
    if (res.abort == 2) {
        report.abort = ExtractionReport::Abort::Statistics;
        return report;
    }
    report.block_lengths = std::move(lengths);
    if (res.abort == 1) {
        report.abort = ExtractionReport::Abort::OversizeBlock;
        return report;
    }
    std::uint64_t sifted_total = 0;
    for (const std::uint64_t b : report.block_lengths) sifted_total += b;
    report.bits_per_block = res.bits_per_block;
    report.cycle_count =
        timing_model(sifted_total, model_bits, ns == 1 ? Scenario::full() : Scenario::splitting(ns),
                     blocking, plan.eps_abort, plan.block_limit);
    if (report.bits_per_block == 0) return report;  // nothing extractable; not an abort
    report.key = std::move(key);
    report.wall_seconds = res.hash_seconds;
    return report;
}
}  // namespace

}  // namespace ssbh
