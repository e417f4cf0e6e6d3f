// comerge_cuda -- the reference's command line tool (proj/tools/comerge_main.cpp)
// with the merge running on the B200 ("CLI and file
// formats to GPU").  Same subcommands, arguments, output lines, CSV schema and
// exit codes; every merge and co-rank goes through the drop-in
// comerge::cuda API (include/comerge/cuda.hpp -> libcomerge_cuda.so).
//
//   corank fileA fileB i [--no-validate]                      comerge_main.cpp:91-99
//   merge  fileA fileB out [--threads N] [--format F] [--no-validate]   :101-127
//   verify fileA fileB merged [--no-validate]                           :175-192
//   bench  [--dist D] [--m M] [--n N] [--p-list L] [--reps R] [--seed S]
//          [--csv PATH|-] [--verify-cap C] [--simulated]                :129-173
//   sort   fileIn out [--format F]         (B200 addition: stable GPU merge sort)
//
// Exit codes (comerge_main.cpp:19-27): 0 success, 1 verification failure,
// 2 usage or contract error, 3 I/O error.
#include <cuda_runtime.h>

#include <algorithm>
#include <charconv>
#include <cstdint>
#include <cstdio>
#include <fstream>
#include <iostream>
#include <limits>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "comerge/cuda.hpp"
#include "comerge_cuda_testkit.h"
#include "keyfile.hpp"

namespace cm = comerge::cuda;
using comerge_cli::key_format;
using comerge_cli::keyfile_error;
using keys_t = std::vector<std::uint64_t>;

namespace {

constexpr int kOk = 0, kVerify = 1, kUsage = 2, kIo = 3;

struct usage_error : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};

const char* kUsageText =
    "usage: comerge_cuda <command> [args]\n"
    "  corank fileA fileB i [--no-validate]\n"
    "  merge  fileA fileB out [--threads N] [--format text|binary|auto] [--no-validate]\n"
    "  verify fileA fileB merged [--no-validate]\n"
    "  bench  [--dist D] [--m M] [--n N] [--p-list L] [--reps R] [--seed S]\n"
    "         [--csv PATH|-] [--verify-cap C] [--simulated]\n"
    "  sort   fileIn out [--format text|binary|auto]\n"
    "distributions: uniform|all-equal|few-distinct[:d]|disjoint|interleaved|organ-pipe|runs[:len]\n";

// ------------------------------------------------------------ arguments
struct args {
    std::vector<std::string> pos;
    std::vector<std::pair<std::string, std::string>> opts;  // --name value
    std::vector<std::string> flags;                         // --name
    bool flag(const std::string& f) const {
        return std::find(flags.begin(), flags.end(), f) != flags.end();
    }
    const std::string* opt(const std::string& o) const {
        for (const auto& [k, v] : opts)
            if (k == o) return &v;
        return nullptr;
    }
};

args parse(int argc, char** argv, int first, const std::vector<std::string>& value_opts,
           const std::vector<std::string>& flag_opts, std::size_t npos) {
    args a;
    for (int i = first; i < argc; ++i) {
        const std::string t = argv[i];
        if (t.rfind("--", 0) == 0) {
            std::string name = t, value;
            const bool inline_value = t.find('=') != std::string::npos;
            if (inline_value) {
                name = t.substr(0, t.find('='));
                value = t.substr(t.find('=') + 1);
            }
            if (std::find(flag_opts.begin(), flag_opts.end(), name) != flag_opts.end() &&
                !inline_value) {
                a.flags.push_back(name);
            } else if (std::find(value_opts.begin(), value_opts.end(), name) != value_opts.end()) {
                if (!inline_value) {
                    if (i + 1 >= argc) throw usage_error(name + ": missing value");
                    value = argv[++i];
                }
                a.opts.emplace_back(name, value);
            } else {
                throw usage_error("unknown option " + name);
            }
        } else {
            a.pos.push_back(t);
        }
    }
    if (a.pos.size() != npos)
        throw usage_error("expected " + std::to_string(npos) + " positional arguments, got " +
                          std::to_string(a.pos.size()));
    return a;
}

std::uint64_t to_u64(const std::string& text, const std::string& what) {
    std::uint64_t v = 0;
    const auto [end, ec] = std::from_chars(text.data(), text.data() + text.size(), v);
    if (ec != std::errc{} || end != text.data() + text.size())
        throw usage_error(what + ": expected a nonnegative integer, got '" + text + "'");
    return v;
}

std::vector<std::size_t> parse_p_list(const std::string& text) {  // comerge_main.cpp:29-46
    std::vector<std::size_t> list;
    std::size_t pos = 0;
    while (pos <= text.size()) {
        std::size_t comma = text.find(',', pos);
        if (comma == std::string::npos) comma = text.size();
        std::size_t v = 0;
        const auto [end, ec] = std::from_chars(text.data() + pos, text.data() + comma, v);
        if (ec != std::errc{} || end != text.data() + comma || v == 0)
            throw std::invalid_argument("--p-list: expected comma-separated positive integers");
        list.push_back(v);
        pos = comma + 1;
    }
    return list;
}

std::size_t default_threads() {
    const unsigned hw = std::thread::hardware_concurrency();
    return hw == 0 ? 1 : hw;
}

key_format out_format(const std::string& choice, key_format input) {
    if (choice == "text") return key_format::text;
    if (choice == "binary") return key_format::binary;
    if (choice != "auto") throw std::invalid_argument("--format: expected text, binary or auto");
    return input;
}

// ------------------------------------------------- verification (host)
// The stable merge the output must equal (merge.hpp:18-33, ties A-first).
keys_t host_two_finger(const keys_t& a, const keys_t& b) {
    keys_t out(a.size() + b.size());
    std::size_t x = 0, y = 0, o = 0;
    while (x < a.size() && y < b.size()) out[o++] = b[y] < a[x] ? b[y++] : a[x++];
    while (x < a.size()) out[o++] = a[x++];
    while (y < b.size()) out[o++] = b[y++];
    return out;
}

std::uint64_t mix64(std::uint64_t x) {  // keys.hpp:17-26 (multiset checksum hash)
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

std::uint64_t checksum(const keys_t& k) {  // keys.hpp:50-55
    std::uint64_t s = 0;
    for (const std::uint64_t x : k) s += mix64(x);
    return s;
}

// experiment.cpp:25-47: exact up to the cap, sortedness + checksum above
bool verify_output(const keys_t& a, const keys_t& b, const keys_t& out, std::size_t cap,
                   std::string* why) {
    if (out.size() != a.size() + b.size()) {
        *why = "length mismatch: expected " + std::to_string(a.size() + b.size()) +
               " keys, found " + std::to_string(out.size());
        return false;
    }
    if (out.size() <= cap) {
        const keys_t expect = host_two_finger(a, b);
        for (std::size_t t = 0; t < out.size(); ++t)
            if (out[t] != expect[t]) {
                *why = "key mismatch at index " + std::to_string(t);
                return false;
            }
        return true;
    }
    if (!std::is_sorted(out.begin(), out.end())) {
        *why = "output is not nondecreasing";
        return false;
    }
    if (checksum(out) != checksum(a) + checksum(b)) {
        *why = "multiset checksum mismatch";
        return false;
    }
    return true;
}

// ------------------------------------------------------------ commands
int cmd_corank(int argc, char** argv) {
    const args p = parse(argc, argv, 2, {}, {"--no-validate"}, 3);
    const bool v = !p.flag("--no-validate");
    const auto a = comerge_cli::read_keys(p.pos[0], v);
    const auto b = comerge_cli::read_keys(p.pos[1], v);
    const std::uint64_t rank = to_u64(p.pos[2], "i");
    cm::co_rank_stats st;
    const cm::co_ranks r = cm::co_rank(rank, a.keys, b.keys, {}, &st);
    std::cout << r.a << ' ' << r.b << ' ' << st.iterations << ' ' << st.comparisons << '\n';
    return kOk;
}

int cmd_merge(int argc, char** argv) {
    const args p = parse(argc, argv, 2, {"--threads", "--format"}, {"--no-validate"}, 3);
    const bool v = !p.flag("--no-validate");
    const auto a = comerge_cli::read_keys(p.pos[0], v);
    const auto b = comerge_cli::read_keys(p.pos[1], v);
    const std::size_t threads = p.opt("--threads") ? to_u64(*p.opt("--threads"), "--threads") : 0;
    const std::size_t workers = threads == 0 ? default_threads() : threads;
    keys_t out(a.keys.size() + b.keys.size());
    const cm::merge_report rep = cm::merge_parallel(a.keys, b.keys, out, workers);
    const key_format fmt = out_format(p.opt("--format") ? *p.opt("--format") : "auto", a.format);
    comerge_cli::write_keys(p.pos[2], out, fmt);
    const auto [lo, hi] = std::minmax_element(rep.block_sizes.begin(), rep.block_sizes.end());
    std::uint32_t max_it = 0;
    for (const std::uint32_t it : rep.corank_iterations) max_it = std::max(max_it, it);
    std::cout << "merged " << rep.m << " + " << rep.n << " keys with " << rep.workers
              << " workers in " << static_cast<double>(rep.wall_ns) / 1e6 << " ms\n"
              << "block sizes " << *lo << ".." << *hi << ", co-rank iterations max " << max_it
              << '\n';
    return kOk;
}

int cmd_verify(int argc, char** argv) {
    const args p = parse(argc, argv, 2, {}, {"--no-validate"}, 3);
    const bool v = !p.flag("--no-validate");
    const auto a = comerge_cli::read_keys(p.pos[0], v);
    const auto b = comerge_cli::read_keys(p.pos[1], v);
    const auto merged = comerge_cli::read_keys(p.pos[2], false);  // judged, never pre-validated
    std::string why;
    bool ok;
    if (merged.keys.size() != a.keys.size() + b.keys.size()) {
        ok = verify_output(a.keys, b.keys, merged.keys, 0, &why);
    } else {  // the stable merge, computed on the device, against the file
        keys_t expect(merged.keys.size());
        cm::stable_merge(a.keys, b.keys, expect);
        ok = true;
        for (std::size_t t = 0; t < expect.size() && ok; ++t)
            if (expect[t] != merged.keys[t]) {
                why = "key mismatch at index " + std::to_string(t);
                ok = false;
            }
    }
    if (!ok) {
        std::cerr << "verification failed: " << why << '\n';
        return kVerify;
    }
    std::cout << "ok: " << merged.keys.size() << " keys are the stable merge\n";
    return kOk;
}

int cmd_sort(int argc, char** argv) {
    const args p = parse(argc, argv, 2, {"--format"}, {}, 2);
    const auto in = comerge_cli::read_keys(p.pos[0], false);
    keys_t out(in.keys.size());
    const std::size_t n = in.keys.size();
    if (n) {
        std::uint64_t* d = nullptr;
        if (cudaMalloc(&d, n * 8) != cudaSuccess) throw std::runtime_error("sort: cudaMalloc failed");
        cudaMemcpy(d, in.keys.data(), n * 8, cudaMemcpyHostToDevice);
        const int rc = comerge_cuda_sort_keys_u64(d, n, d, nullptr, 0, nullptr);
        cudaMemcpy(out.data(), d, n * 8, cudaMemcpyDeviceToHost);
        cudaFree(d);
        if (rc) throw std::runtime_error(comerge_cuda_last_error());
    }
    comerge_cli::write_keys(p.pos[1], out,
                            out_format(p.opt("--format") ? *p.opt("--format") : "auto", in.format));
    std::cout << "sorted " << n << " keys\n";
    return kOk;
}

// ------------------------------------------------------------ bench
// distributions: generate.hpp:16-46 / generate.cpp (restated; the seeded
// ones draw the reference's splitmix64 streams on the device through the
// testkit generator, whose output the parity tests pin to the reference)
struct dist_spec {
    std::string kind;
    std::uint64_t param = 0;
};

dist_spec parse_dist(const std::string& token) {  // generate.cpp:100-141
    dist_spec d;
    std::string name = token;
    bool has_param = false;
    if (const auto c = token.find(':'); c != std::string::npos) {
        name = token.substr(0, c);
        const std::string tail = token.substr(c + 1);
        std::uint64_t v = 0;
        const auto [end, ec] = std::from_chars(tail.data(), tail.data() + tail.size(), v);
        if (ec != std::errc{} || end != tail.data() + tail.size() || v == 0)
            throw std::invalid_argument("distribution: bad parameter in '" + token + "'");
        d.param = v;
        has_param = true;
    }
    static const char* kinds[] = {"uniform", "all-equal", "few-distinct", "disjoint",
                                  "interleaved", "organ-pipe", "runs"};
    if (std::find(std::begin(kinds), std::end(kinds), name) == std::end(kinds))
        throw std::invalid_argument("distribution: unknown kind '" + token + "'");
    d.kind = name;
    const bool takes = name == "few-distinct" || name == "runs";
    if (has_param && !takes)
        throw std::invalid_argument("distribution: '" + name + "' takes no parameter");
    if (takes && !has_param) d.param = name == "few-distinct" ? 16 : 32;
    return d;
}

std::string dist_token(const dist_spec& d) {  // generate.cpp:143-162
    if (d.kind == "few-distinct" || d.kind == "runs") return d.kind + ":" + std::to_string(d.param);
    return d.kind;
}

keys_t sorted_stream(std::uint64_t seed, std::uint64_t lane, std::size_t len, std::uint64_t base,
                     std::uint64_t width) {
    keys_t out(len);
    if (!len) return out;
    std::uint64_t* d = nullptr;
    if (cudaMalloc(&d, len * 8) != cudaSuccess) throw std::runtime_error("bench: cudaMalloc failed");
    const int rc = comerge_testkit_generate_sorted(COMERGE_KEY_U64, seed, lane, len, width, d, nullptr);
    cudaMemcpy(out.data(), d, len * 8, cudaMemcpyDeviceToHost);
    cudaFree(d);
    if (rc) throw std::runtime_error(comerge_testkit_last_error());
    for (auto& k : out) k += base;
    return out;
}

keys_t organ_pipe(std::size_t len) {  // generate.cpp:38-56
    keys_t keys;
    keys.reserve(len);
    const std::uint64_t values = std::max<std::uint64_t>(1, std::min<std::uint64_t>(len, 63));
    std::uint64_t wsum = 0;
    for (std::uint64_t v = 0; v < values; ++v) wsum += std::min(v + 1, values - v);
    std::uint64_t acc = 0;
    std::size_t written = 0;
    for (std::uint64_t v = 0; v < values; ++v) {
        acc += std::min(v + 1, values - v);
        const auto upto = static_cast<std::size_t>(static_cast<unsigned __int128>(len) * acc / wsum);
        for (; written < upto; ++written) keys.push_back(v);
    }
    return keys;
}

std::pair<keys_t, keys_t> generate(const dist_spec& d, std::uint64_t seed, std::size_t m,
                                   std::size_t n) {  // generate.cpp:68-98
    if (d.kind == "uniform") return {sorted_stream(seed, 0, m, 0, 0), sorted_stream(seed, 1, n, 0, 0)};
    if (d.kind == "all-equal") return {keys_t(m, 42), keys_t(n, 42)};
    if (d.kind == "few-distinct")
        return {sorted_stream(seed, 0, m, 0, d.param), sorted_stream(seed, 1, n, 0, d.param)};
    if (d.kind == "disjoint") {
        const std::uint64_t w = std::uint64_t{1} << 32;
        return {sorted_stream(seed, 0, m, 0, w), sorted_stream(seed, 1, n, w, w)};
    }
    if (d.kind == "interleaved") {
        keys_t a(m), b(n);
        for (std::size_t t = 0; t < m; ++t) a[t] = 2 * t;
        for (std::size_t t = 0; t < n; ++t) b[t] = 2 * t + 1;
        return {a, b};
    }
    if (d.kind == "organ-pipe") return {organ_pipe(m), organ_pipe(n)};
    keys_t a(m), b(n);  // runs
    for (std::size_t t = 0; t < m; ++t) a[t] = t / d.param;
    for (std::size_t t = 0; t < n; ++t) b[t] = t / d.param;
    return {a, b};
}

// experiment.cpp:49-121 (run_experiment) + :123-155 (CSV), device merges
int cmd_bench(int argc, char** argv) {
    const args p = parse(argc, argv, 2,
                         {"--dist", "--m", "--n", "--p-list", "--reps", "--seed", "--csv",
                          "--verify-cap"},
                         {"--simulated"}, 0);
    const dist_spec dist = parse_dist(p.opt("--dist") ? *p.opt("--dist") : "uniform");
    const std::size_t m = p.opt("--m") ? to_u64(*p.opt("--m"), "--m") : 1'000'000;
    const std::size_t n = p.opt("--n") ? to_u64(*p.opt("--n"), "--n") : 1'000'000;
    const auto p_list = parse_p_list(p.opt("--p-list") ? *p.opt("--p-list") : "1,2,4,8");
    const std::size_t reps = p.opt("--reps") ? to_u64(*p.opt("--reps"), "--reps") : 3;
    const std::uint64_t seed = p.opt("--seed") ? to_u64(*p.opt("--seed"), "--seed") : 1;
    const std::string csv = p.opt("--csv") ? *p.opt("--csv") : "-";
    const std::size_t cap =
        p.opt("--verify-cap") ? to_u64(*p.opt("--verify-cap"), "--verify-cap") : (std::size_t{1} << 20);
    // --simulated is accepted: the device schedule has no thread mode
    if (reps < 1) throw std::invalid_argument("run_experiment: repetitions must be at least 1");

    const auto [a, b] = generate(dist, seed, m, n);
    const std::size_t total = a.size() + b.size();
    const bool full_check = total <= cap;
    // provenance tags (oracle.hpp:22-37): payload = index, B side marked
    std::vector<std::uint32_t> ta(a.size()), tb(b.size());
    for (std::size_t t = 0; t < a.size(); ++t) ta[t] = std::uint32_t(t);
    for (std::size_t t = 0; t < b.size(); ++t) tb[t] = std::uint32_t(t) | 0x80000000u;
    std::vector<std::uint32_t> tag_expect;
    if (full_check) {  // tagged two-finger merge (oracle.hpp:65-93)
        tag_expect.resize(total);
        std::size_t x = 0, y = 0, o = 0;
        while (x < a.size() && y < b.size()) tag_expect[o++] = b[y] < a[x] ? tb[y++] : ta[x++];
        while (x < a.size()) tag_expect[o++] = ta[x++];
        while (y < b.size()) tag_expect[o++] = tb[y++];
    }

    std::vector<cm::merge_report> reports;
    keys_t out(total), tout(full_check ? total : 0);
    std::vector<std::uint32_t> tvals(full_check ? total : 0);
    for (const std::size_t w : p_list) {
        cm::merge_options counted;
        counted.count_comparisons = true;
        const cm::merge_report inst = cm::merge_parallel(a, b, out, w, {}, counted);
        bool stable_ok = true;
        if (full_check) {
            cm::merge_parallel_pairs(a, std::span<const std::uint32_t>(ta), b,
                                     std::span<const std::uint32_t>(tb), tout,
                                     std::span<std::uint32_t>(tvals), w);
            stable_ok = tvals == tag_expect;
        }
        for (std::size_t r = 0; r < reps; ++r) {
            cm::merge_report rep = cm::merge_parallel(a, b, out, w);
            rep.comparisons = inst.comparisons;
            std::string why;
            const bool ok = verify_output(a, b, out, cap, &why) && stable_ok;
            rep.verified = ok;
            if (!ok) rep.note = why.empty() ? "tagged run deviates from the stable-merge oracle" : why;
            reports.push_back(rep);
        }
    }
    // speedups from median wall times, relative to the p = 1 batch
    auto batch_median = [&](std::size_t batch) {
        std::vector<std::uint64_t> walls;
        for (std::size_t r = 0; r < reps; ++r) walls.push_back(reports[batch * reps + r].wall_ns);
        std::sort(walls.begin(), walls.end());
        const std::size_t h = walls.size() / 2;
        return walls.size() % 2 ? double(walls[h]) : (double(walls[h - 1]) + double(walls[h])) / 2;
    };
    if (const auto one = std::find(p_list.begin(), p_list.end(), std::size_t{1}); one != p_list.end()) {
        const double base = batch_median(std::size_t(one - p_list.begin()));
        for (std::size_t batch = 0; batch < p_list.size(); ++batch) {
            const double own = batch_median(batch);
            const double s = p_list[batch] == 1 ? 1.0 : (own > 0 ? base / own : 0.0);
            for (std::size_t r = 0; r < reps; ++r) reports[batch * reps + r].speedup_vs_p1 = s;
        }
    }
    std::ostringstream table;
    table << "dist,seed,m,n,p,rep,wall_ns,comparisons,max_block,min_block,verified,speedup\n";
    for (std::size_t row = 0; row < reports.size(); ++row) {
        const auto& rep = reports[row];
        const auto [lo, hi] = std::minmax_element(rep.block_sizes.begin(), rep.block_sizes.end());
        table << dist_token(dist) << ',' << seed << ',' << rep.m << ',' << rep.n << ','
              << rep.workers << ',' << row % reps << ',' << rep.wall_ns << ','
              << (rep.comparisons ? std::to_string(*rep.comparisons) : std::string()) << ','
              << *hi << ',' << *lo << ',' << (rep.verified.value_or(false) ? 1 : 0) << ',';
        if (rep.speedup_vs_p1) {
            std::ostringstream ratio;
            ratio << *rep.speedup_vs_p1;
            table << ratio.str();
        }
        table << '\n';
    }
    if (csv == "-") {
        std::cout << table.str();
    } else {
        std::ofstream f(csv, std::ios::trunc);
        if (!f) throw keyfile_error(csv + ": cannot open for writing");
        f << table.str();
        if (!f.flush()) throw keyfile_error(csv + ": write failed");
    }
    for (std::size_t batch = 0; batch < p_list.size(); ++batch) {
        std::vector<std::uint64_t> walls;
        for (std::size_t r = 0; r < reps; ++r) walls.push_back(reports[batch * reps + r].wall_ns);
        std::sort(walls.begin(), walls.end());
        std::cerr << "p=" << p_list[batch] << ": median "
                  << static_cast<double>(walls[walls.size() / 2]) / 1e6 << " ms, min "
                  << static_cast<double>(walls.front()) / 1e6 << " ms";
        if (const auto& s = reports[batch * reps].speedup_vs_p1) std::cerr << ", speedup " << *s;
        std::cerr << '\n';
    }
    bool all = true;
    for (const auto& rep : reports)
        if (!rep.verified.value_or(false)) {
            all = false;
            std::cerr << "unverified run at p=" << rep.workers << ": " << rep.note << '\n';
        }
    return all ? kOk : kVerify;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        std::cerr << kUsageText;
        return kUsage;
    }
    const std::string cmd = argv[1];
    if (cmd == "--help" || cmd == "-h") {
        std::cout << kUsageText;
        return kOk;
    }
    try {
        if (cmd == "corank") return cmd_corank(argc, argv);
        if (cmd == "merge") return cmd_merge(argc, argv);
        if (cmd == "verify") return cmd_verify(argc, argv);
        if (cmd == "bench") return cmd_bench(argc, argv);
        if (cmd == "sort") return cmd_sort(argc, argv);
        std::cerr << "error: unknown command '" << cmd << "'\n" << kUsageText;
        return kUsage;
    } catch (const usage_error& e) {
        std::cerr << "error: " << e.what() << '\n' << kUsageText;
        return kUsage;
    } catch (const keyfile_error& e) {
        std::cerr << "error: " << e.what() << '\n';
        return kIo;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << '\n';
        return kUsage;
    }
}
