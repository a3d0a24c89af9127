// SPDX-License-Identifier: Apache-2.0
// The reference's command-line front end (cli.hpp:72-252)
// as a drop-in header over the device path: cpd::run_command(args, out)
// with the same subcommands, file formats, output lines and exit codes --
// 0 ok, 2 file error, 3 malformed file, 4 numerical failure, 1 otherwise
// (bad flags, unknown algorithm, count deviation) -- and no CLI11: options
// are parsed by the small parser below (--name value, -n value,
// --name=value).  The cpd-b200 binary (csrc/cli.cpp) is main() around it.
//
//   decompose -i X.cpdt --alg als|qr|qr-dt|qr-br|qr-bre --rank R [--iters N]
//             [--tol T] [--seed S] [--trace T.csv] [-o M.cpdf] [--alpha A]
//             [--beta B] [--gap G]          X streams straight into HBM
//   synth     --dims a,b,c --rank R [--collinearity c,..] [--l1 x] [--l2 x]
//             [--seed S] -o X.cpdt [--truth M.cpdf]     (reference construction)
//   synth     --baseline c1..c5 -o X.cpdt    BASELINE config on the device
//   counts    --order 3|4 --dims a,b,c --rank R
//   info      -i FILE
#pragma once

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <iostream>
#include <map>
#include <optional>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "cpd/dim_tree.hpp"
#include "cpd/io.hpp"
#include "cpd/kruskal.hpp"
#include "cpd/solvers.hpp"
#include "cpd/synth.hpp"
#include "cpd/tensor.hpp"

namespace cpd {
namespace cli_b200 {

struct usage_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// --name value / -n value / --name=value
class Args {
public:
    Args(const std::vector<std::string>& args, std::size_t first) {
        for (std::size_t i = first; i < args.size(); ++i) {
            std::string a = args[i];
            if (a.size() < 2 || a[0] != '-') throw usage_error("unexpected argument " + a);
            std::string v;
            const auto eq = a.find('=');
            if (eq != std::string::npos) {
                v = a.substr(eq + 1);
                a = a.substr(0, eq);
            } else {
                if (i + 1 >= args.size()) throw usage_error(a + " needs a value");
                v = args[++i];
            }
            kv_[a] = v;
        }
    }
    std::optional<std::string> get(const std::string& l, const std::string& s = "") {
        for (const std::string& k : {l, s}) {
            if (k.empty()) continue;
            const auto it = kv_.find(k);
            if (it != kv_.end()) {
                used_.push_back(k);
                return it->second;
            }
        }
        return std::nullopt;
    }
    std::string need(const std::string& l, const std::string& s = "") {
        auto v = get(l, s);
        if (!v) throw usage_error(l + " is required");
        return *v;
    }
    void finish() const {
        for (const auto& [k, v] : kv_) {
            bool ok = false;
            for (const std::string& u : used_) ok = ok || u == k;
            if (!ok) throw usage_error("unknown option " + k);
        }
    }

private:
    std::map<std::string, std::string> kv_;
    std::vector<std::string> used_;
};

inline uint64_t to_u64(const std::string& s, const char* what) {
    try {
        size_t pos = 0;
        const unsigned long long v = std::stoull(s, &pos);
        if (pos != s.size()) throw std::invalid_argument(s);
        return v;
    } catch (const std::exception&) {
        throw usage_error(std::string(what) + ": not an integer: " + s);
    }
}

inline double to_f64(const std::string& s, const char* what) {
    try {
        size_t pos = 0;
        const double v = std::stod(s, &pos);
        if (pos != s.size()) throw std::invalid_argument(s);
        return v;
    } catch (const std::exception&) {
        throw usage_error(std::string(what) + ": not a number: " + s);
    }
}

template <class T, class F>
std::vector<T> list(const std::string& s, F conv, const char* what) {
    std::vector<T> out;
    std::stringstream ss(s);
    std::string tok;
    while (std::getline(ss, tok, ',')) out.push_back(conv(tok, what));
    return out;
}

struct Ctx {
    cpdb_ctx* c = nullptr;
    Ctx() {
        const char* env = std::getenv("CPD_DEVICE");
        cpd::abi::check(cpdb_create(env ? std::atoi(env) : 0, &c));
    }
    ~Ctx() { cpdb_destroy(c); }
};

inline int run_decompose(Args& a, std::ostream& out) {
    const std::string input = a.need("--input", "-i");
    const std::string alg = a.need("--alg");
    cpd::SolverConfig cfg;
    cfg.rank = to_u64(a.need("--rank"), "--rank");
    cfg.max_iterations = to_u64(a.get("--iters").value_or("50"), "--iters");
    cfg.fitness_threshold = to_f64(a.get("--tol").value_or("1.0"), "--tol");
    cfg.seed = to_u64(a.get("--seed").value_or("0"), "--seed");
    cfg.alpha = to_f64(a.get("--alpha").value_or("0.1"), "--alpha");
    if (auto b = a.get("--beta")) cfg.beta_override = to_f64(*b, "--beta");
    cfg.activation_gap = to_f64(a.get("--gap").value_or("0.03"), "--gap");
    const std::string trace = a.get("--trace").value_or("");
    const std::string output = a.get("--output", "-o").value_or("");
    a.finish();

    bool bre = false, als = false;
    if (alg == "qr") {
        cfg.strategy = cpd::Strategy::naive;
    } else if (alg == "qr-dt") {
        cfg.strategy = cpd::Strategy::dim_tree;
    } else if (alg == "qr-br") {
        cfg.strategy = cpd::Strategy::branch_reuse;
    } else if (alg == "qr-bre") {
        cfg.strategy = cpd::Strategy::branch_reuse;
        bre = true;
    } else if (alg == "als") {
        als = true;
    } else {
        throw usage_error("--alg: unknown algorithm " + alg);
    }
    cfg.algorithm = als ? cpd::Algorithm::als : cpd::Algorithm::als_qr;
    cfg.validate();

    // header first (host only): file / format errors surface before any device work
    uint32_t order = 0;
    uint64_t d[CPDB_MAX_ORDER];
    const int st = cpdb_cpdt_info(input.c_str(), &order, d);
    if (st == CPDB_FILE_ERROR) throw cpd::file_error(cpdb_last_error());
    if (st == CPDB_FORMAT_ERROR) throw cpd::format_error(cpdb_last_error());
    cpd::abi::check(st);
    const std::vector<std::size_t> dims(d, d + order);
    Ctx ctx;
    cpd::load_tensor_to_device(ctx.c, input);  // straight into HBM
    const cpd::SolveResult r =
        als ? cpd::detail::run_als_on_context(ctx.c, dims, cfg, nullptr, nullptr)
            : cpd::detail::run_on_context(ctx.c, dims, cfg, nullptr, nullptr, bre);
    if (!output.empty()) cpd::write_model_file(output, r.model, cpd::Shape(dims));
    if (!trace.empty()) cpd::write_trace_file(trace, r.trace);
    char buf[40];
    std::snprintf(buf, sizeof buf, "%.17g", r.trace.back().fitness);
    out << "final_fitness " << buf << "\n";
    return 0;
}

inline int run_synth(Args& a, std::ostream& out) {
    const std::string path = a.need("--output", "-o");
    if (auto base = a.get("--baseline")) {
        a.finish();
        struct Cfg {
            int kind;
            std::vector<uint64_t> dims;
            uint64_t rank;
            double rho;
            uint64_t seed;
        };
        const std::map<std::string, Cfg> cfgs = {
            {"c1", {0, {100, 100, 100}, 10, 1e-2, 20250001}},
            {"c2", {0, {512, 512, 512}, 32, 1e-3, 20250002}},
            {"c3", {0, {128, 128, 128, 128}, 16, 1e-2, 20250003}},
            {"c4", {1, {256, 256, 256}, 20, 1e-4, 20250004}},
            {"c5", {0, {256, 256, 256, 256}, 64, 1e-3, 20250005}},
        };
        const auto it = cfgs.find(*base);
        if (it == cfgs.end()) throw usage_error("--baseline: one of c1..c5");
        Ctx ctx;
        const Cfg& c = it->second;
        cpd::abi::check(cpdb_tensor_synth(ctx.c, c.kind, c.dims.data(), uint32_t(c.dims.size()),
                                          c.rank, c.rho, c.seed));
        const int st = cpdb_tensor_save_cpdt(ctx.c, path.c_str());
        if (st == CPDB_FILE_ERROR) throw cpd::file_error(cpdb_last_error());
        cpd::abi::check(st);
        uint64_t n = 1;
        for (uint64_t v : c.dims) n *= v;
        out << "wrote " << path << " (" << n << " values)\n";
        return 0;
    }
    cpd::SynthSpec spec;
    spec.dims = cpd::Shape(list<std::size_t>(a.need("--dims"), to_u64, "--dims"));
    spec.true_rank = to_u64(a.need("--rank"), "--rank");
    if (auto c = a.get("--collinearity")) spec.collinearity = list<double>(*c, to_f64, "--collinearity");
    spec.l1 = to_f64(a.get("--l1").value_or("0"), "--l1");
    spec.l2 = to_f64(a.get("--l2").value_or("0"), "--l2");
    spec.seed = to_u64(a.get("--seed").value_or("0"), "--seed");
    const std::string truth = a.get("--truth").value_or("");
    a.finish();
    const std::size_t order = spec.dims.order();
    if (spec.collinearity.empty()) spec.collinearity.assign(order, 0.0);
    if (spec.collinearity.size() == 1 && order > 1)
        spec.collinearity.assign(order, spec.collinearity[0]);
    const cpd::SynthResult r = cpd::assemble_noisy_tensor(spec);
    cpd::write_tensor_file(path, r.tensor);
    if (!truth.empty()) cpd::write_model_file(truth, r.truth, spec.dims);
    out << "wrote " << path << " (" << r.tensor.size() << " values)\n";
    return 0;
}

inline int run_counts(Args& a, std::ostream& out) {
    const std::size_t order = to_u64(a.need("--order"), "--order");
    const auto dims = list<std::size_t>(a.need("--dims"), to_u64, "--dims");
    const std::size_t rank = to_u64(a.need("--rank"), "--rank");
    a.finish();
    if (order != 3 && order != 4) throw usage_error("--order: 3 or 4");
    if (dims.size() != order) throw usage_error("--dims: need one extent per mode");
    const std::vector<uint64_t> expected =
        order == 3 ? std::vector<uint64_t>{9, 6, 4} : std::vector<uint64_t>{12, 6, 4};
    out << "order " << order << "  dims ";
    for (std::size_t k = 0; k < dims.size(); ++k) out << (k ? "," : "") << dims[k];
    out << "  rank " << rank << "  (first 3 iterations)\n";
    bool ok = true;
    const cpd::Strategy ss[] = {cpd::Strategy::naive, cpd::Strategy::dim_tree,
                                cpd::Strategy::branch_reuse};
    for (std::size_t s = 0; s < 3; ++s) {
        const cpd::Schedule sch = cpd::build_schedule(order, ss[s], 3);
        const cpd::CostReport m = cpd::measured_cost(sch, dims, rank, 3);
        const uint64_t closed = cpd::closed_form_cost(order, ss[s], dims, rank);
        out << cpd::strategy_name(ss[s]) << ": root_ttms=" << m.root_ttm_count
                  << " (expected " << expected[s] << ")  measured_flops=" << m.total_flops
                  << "  closed_form_flops=" << closed << "\n";
        for (const auto& [key, b] : m.categories)
            out << "  " << cpd::CostReport::category_label(key, order) << " x" << b.count
                      << " = " << b.flops << "\n";
        ok = ok && m.root_ttm_count == expected[s];
    }
    if (!ok) {
        std::cerr << "error: measured root-TTM counts deviate from expected values\n";
        return 1;
    }
    return 0;
}

inline int run_info(Args& a, std::ostream& out) {
    const std::string path = a.need("--input", "-i");
    a.finish();
    const std::vector<unsigned char> head = [&] {
        std::vector<unsigned char> b;
        std::FILE* f = std::fopen(path.c_str(), "rb");
        if (!f) throw cpd::file_error("cannot open " + path);
        b.resize(4);
        b.resize(std::fread(b.data(), 1, 4, f));
        std::fclose(f);
        return b;
    }();
    auto is = [&](const char* m) {
        return head.size() == 4 && std::equal(head.begin(), head.end(), m);
    };
    if (is("CPDT")) {  // header only: the payload may be tens of GB
        uint32_t order = 0;
        uint64_t d[CPDB_MAX_ORDER];
        const int st = cpdb_cpdt_info(path.c_str(), &order, d);
        if (st == CPDB_FORMAT_ERROR) throw cpd::format_error(cpdb_last_error());
        if (st == CPDB_FILE_ERROR) throw cpd::file_error(cpdb_last_error());
        cpd::abi::check(st);
        uint64_t n = 1;
        out << "tensor file, version 1, order " << order << ", dims ";
        for (uint32_t k = 0; k < order; ++k) {
            out << (k ? "x" : "") << d[k];
            n *= d[k];
        }
        out << ", " << n << " values\n";
        return 0;
    }
    if (is("CPDF")) {
        const cpd::DecodedModel m = cpd::read_model_file(path);
        out << "model file, version 1, order " << m.model.order() << ", rank "
                  << m.model.rank() << ", dims ";
        for (std::size_t k = 0; k < m.shape.order(); ++k)
            out << (k ? "x" : "") << m.shape.extent(k);
        out << "\n";
        return 0;
    }
    throw cpd::format_error("unrecognized file magic in " + path);
}

inline void usage() {
    std::cerr << "usage: cpd-b200 <decompose|synth|counts|info> [options]\n"
                 "  decompose -i X.cpdt --alg als|qr|qr-dt|qr-br|qr-bre --rank R [--iters N]\n"
                 "            [--tol T] [--seed S] [--trace T.csv] [-o M.cpdf] [--alpha A]\n"
                 "            [--beta B] [--gap G]\n"
                 "  synth     --dims a,b,c --rank R [--collinearity c] [--l1 x] [--l2 x]\n"
                 "            [--seed S] -o X.cpdt [--truth M.cpdf]\n"
                 "  synth     --baseline c1|c2|c3|c4|c5 -o X.cpdt\n"
                 "  counts    --order 3|4 --dims a,b,c --rank R\n"
                 "  info      -i FILE\n";
}

}  // namespace cli_b200

/// Command-line entry point (cli.hpp:212-252): args without the program name.
inline int run_command(const std::vector<std::string>& args, std::ostream& out = std::cout) {
    using namespace cli_b200;
    if (args.empty()) {
        usage();
        return 1;
    }
    const std::string cmd = args[0];
    try {
        Args a(args, 1);
        if (cmd == "decompose") return run_decompose(a, out);
        if (cmd == "synth") return run_synth(a, out);
        if (cmd == "counts") return run_counts(a, out);
        if (cmd == "info") return run_info(a, out);
        usage();
        return 1;
    } catch (const file_error& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 2;
    } catch (const format_error& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 3;
    } catch (const singular_system_error& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 4;
    } catch (const singular_triangular_error& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 4;
    } catch (const generation_error& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 4;
    } catch (const usage_error& e) {
        std::cerr << "error: " << e.what() << "\n";
        usage();
        return 1;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    }
}

}  // namespace cpd
