// specmoe -- command-line front end of the harness (CLI verbs from SPEC.md:497; the reference's
// tools/ directory is absent, proj/CMakeLists.txt:14).  Exit codes follow SPEC.md:503: 0 success,
// 1 configuration error, 2 runtime invariant breach (3: CUDA / unexpected failure).
//
//   specmoe run --config F [--out PATH] [--format csv|json] [--policy P] [--batch LIST]
//               [--gamma LIST] [--n-draft LIST] [--seed LIST]
//   specmoe affinity build --config F --out PATH
//   specmoe trace analyze --in PATH [--out PATH] [--top N]
//   specmoe selftest
#include <fstream>
#include <iomanip>
#include <iostream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "specmoe/harness.hpp"

namespace {

int usage() {
    std::cerr << "usage:\n"
                 "  specmoe run --config F [--out PATH] [--format csv|json] [--policy P] [--batch LIST]\n"
                 "              [--gamma LIST] [--n-draft LIST] [--seed LIST]\n"
                 "  specmoe affinity build --config F --out PATH\n"
                 "  specmoe trace analyze --in PATH [--out PATH] [--top N]\n"
                 "  specmoe selftest\n";
    return 1;
}

std::map<std::string, std::string> flags(int argc, char** argv, int first) {
    std::map<std::string, std::string> f;
    for (int i = first; i < argc; ++i) {
        std::string k = argv[i];
        if (k.rfind("--", 0) != 0 || i + 1 >= argc) throw specmoe::ConfigError("bad argument: " + k);
        f[k.substr(2)] = argv[++i];
    }
    return f;
}

std::string read_file(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw specmoe::ConfigError("cannot open " + path);
    std::stringstream ss;
    ss << in.rdbuf();
    return ss.str();
}

// config text with `key = value` overrides: the file's own line for that key is dropped
std::string with_overrides(const std::string& text, const std::map<std::string, std::string>& ov) {
    std::istringstream in(text);
    std::string line, out;
    while (std::getline(in, line)) {
        std::string key = line.substr(0, line.find('='));
        key.erase(0, key.find_first_not_of(" \t"));
        key.erase(key.find_last_not_of(" \t") + 1);
        if (!ov.count(key)) out += line + "\n";
    }
    for (const auto& kv : ov) out += kv.first + " = " + kv.second + "\n";
    return out;
}

int run(int argc, char** argv) {
    if (argc < 2) return usage();
    const std::string verb = argv[1];
    if (verb == "selftest") return specmoe::selftest(std::cout) ? 0 : 2;
    if (verb == "run") {
        auto f = flags(argc, argv, 2);
        if (!f.count("config")) return usage();
        std::map<std::string, std::string> ov;
        const std::map<std::string, std::string> names{
            {"policy", "policy"}, {"batch", "batch"}, {"gamma", "gamma"}, {"n-draft", "n_draft"}, {"seed", "seeds"}};
        for (const auto& kv : names)
            if (f.count(kv.first)) ov[kv.second] = f[kv.first];
        const auto cfg = specmoe::parse_config_text(with_overrides(read_file(f["config"]), ov));
        const auto rows = specmoe::run_experiment(cfg);
        const std::string fmt = f.count("format") ? f["format"] : "csv";
        if (f.count("out")) specmoe::emit_results(rows, fmt, f["out"], cfg.verbose);
        else specmoe::emit_results(rows, fmt, std::cout, cfg.verbose);
        return 0;
    }
    if (verb == "affinity") {
        if (argc < 3 || std::string(argv[2]) != "build") return usage();
        auto f = flags(argc, argv, 3);
        if (!f.count("config") || !f.count("out")) return usage();
        const auto cfg = specmoe::parse_config(f["config"]);
        specmoe::save_affinity_csv(specmoe::build_affinity_table(specmoe::build_model(cfg.model)), f["out"]);
        return 0;
    }
    if (verb == "trace") {
        if (argc < 3 || std::string(argv[2]) != "analyze") return usage();
        auto f = flags(argc, argv, 3);
        if (!f.count("in")) return usage();
        const auto rep = specmoe::analyze_trace(specmoe::ingest_trace(f["in"]), f.count("top") ? std::stoi(f["top"]) : 10);
        std::cout << std::setprecision(17) << "skewness " << rep.skewness << " routed_tokens " << rep.routed_tokens << "\n";
        for (size_t l = 0; l < rep.hottest.size(); ++l) {
            std::cout << "layer " << l << " hottest";
            for (int e : rep.hottest[l]) std::cout << ' ' << e;
            std::cout << "\n";
        }
        if (f.count("out")) specmoe::write_trace_report(rep, f["out"]);
        return 0;
    }
    return usage();
}

}  // namespace

int main(int argc, char** argv) {
    try {
        return run(argc, argv);
    } catch (const specmoe::ConfigError& e) {
        std::cerr << "config error: " << e.what() << "\n";
        return 1;
    } catch (const specmoe::InvariantError& e) {
        std::cerr << "invariant error: " << e.what() << "\n";
        return 2;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 3;
    }
}
