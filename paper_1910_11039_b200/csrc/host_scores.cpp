// Result / score path of the reference CLI, host side:
//   write_scores / read_scores   /root/reference/proj/src/score_io.cpp:12-52
//   compare_scores               score_io.cpp:98-122 (max abs error, vertices above eps, top-10 / top-100 overlap)
//   run_meta                     /root/reference/proj/tools/epochbc.cpp:179-190
//   stats_to_json key order      /root/reference/proj/src/stats.cpp:7-40
// File format: "# key=value" header lines (sorted by key, as std::map iterates), then one
// "original_vertex_id<TAB>%.12g" line per vertex.
#include "host_scores.hpp"

#include <algorithm>
#include <charconv>
#include <cinttypes>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <sstream>
#include <unordered_map>

namespace ebc {

void write_scores(const std::string &path, const ScoreTable &t) {
    std::ofstream out(path, std::ios::binary);
    if (!out)
        throw ParseError("cannot open output file: " + path);
    for (const auto &kv : t.meta)
        out << "# " << kv.first << "=" << kv.second << "\n";
    char buf[64];
    for (std::size_t i = 0; i < t.vertex_ids.size(); ++i) {
        std::snprintf(buf, sizeof(buf), "%" PRIu64 "\t%.12g", t.vertex_ids[i], t.scores[i]);
        out << buf << "\n";
    }
    if (!out)
        throw ParseError("failed writing score file: " + path);
}

ScoreTable read_scores(const std::string &path) {
    std::ifstream in(path, std::ios::binary);
    if (!in)
        throw ParseError("cannot open score file: " + path);
    ScoreTable t;
    std::string line;
    std::uint64_t lineno = 0;
    while (std::getline(in, line)) {
        ++lineno;
        if (line.empty())
            continue;
        if (line[0] == '#') {
            const std::string body = line.substr(1);
            const auto eq = body.find('=');
            if (eq != std::string::npos) {
                std::string key = body.substr(0, eq);
                const auto first = key.find_first_not_of(" \t");
                key = first == std::string::npos ? std::string() : key.substr(first);
                key.erase(key.find_last_not_of(" \t") + 1);
                t.meta[key] = body.substr(eq + 1);
            }
            continue;
        }
        std::istringstream ls(line);
        std::uint64_t id;
        double score;
        if (!(ls >> id >> score))
            throw ParseError("score file: malformed line " + std::to_string(lineno));
        t.vertex_ids.push_back(id);
        t.scores.push_back(score);
    }
    return t;
}

namespace {

// Top-k ids by (score desc, id asc), returned sorted by id.
std::vector<std::uint64_t> top_ids(const ScoreTable &t, std::size_t k) {
    std::vector<std::size_t> order(t.vertex_ids.size());
    for (std::size_t i = 0; i < order.size(); ++i)
        order[i] = i;
    k = std::min(k, order.size());
    std::partial_sort(order.begin(), order.begin() + k, order.end(), [&](std::size_t a, std::size_t b) {
        return t.scores[a] != t.scores[b] ? t.scores[a] > t.scores[b] : t.vertex_ids[a] < t.vertex_ids[b];
    });
    std::vector<std::uint64_t> ids(k);
    for (std::size_t i = 0; i < k; ++i)
        ids[i] = t.vertex_ids[order[i]];
    std::sort(ids.begin(), ids.end());
    return ids;
}

double overlap(const ScoreTable &a, const ScoreTable &b, std::size_t k) {
    const auto ta = top_ids(a, k), tb = top_ids(b, k);
    if (ta.empty())
        return 1.0;
    std::vector<std::uint64_t> common;
    std::set_intersection(ta.begin(), ta.end(), tb.begin(), tb.end(), std::back_inserter(common));
    return static_cast<double>(common.size()) / static_cast<double>(ta.size());
}

} // namespace

CompareReport compare_scores(const ScoreTable &approx, const ScoreTable &exact, double eps) {
    auto sorted = [](std::vector<std::uint64_t> ids) {
        std::sort(ids.begin(), ids.end());
        return ids;
    };
    if (sorted(approx.vertex_ids) != sorted(exact.vertex_ids))
        throw ConfigError("compare: vertex sets differ");
    std::unordered_map<std::uint64_t, double> exact_of;
    exact_of.reserve(exact.vertex_ids.size() * 2);
    for (std::size_t i = 0; i < exact.vertex_ids.size(); ++i)
        exact_of[exact.vertex_ids[i]] = exact.scores[i]; // a repeated id keeps its last score, as std::map[] does
    CompareReport r;
    r.vertices = approx.vertex_ids.size();
    for (std::size_t i = 0; i < approx.vertex_ids.size(); ++i) {
        const double err = std::abs(approx.scores[i] - exact_of[approx.vertex_ids[i]]);
        r.max_abs_error = std::max(r.max_abs_error, err);
        if (err > eps)
            ++r.vertices_above_eps;
    }
    r.top10_overlap = overlap(approx, exact, 10);
    r.top100_overlap = overlap(approx, exact, 100);
    return r;
}

std::map<std::string, std::string> run_meta(double eps, double delta, std::uint64_t seed, std::uint64_t tau) {
    std::map<std::string, std::string> meta;
    std::ostringstream e, d;
    e << eps;
    d << delta;
    meta["eps"] = e.str();
    meta["delta"] = d.str();
    meta["tau"] = std::to_string(tau);
    meta["seed"] = std::to_string(seed);
    meta["algo"] = "2"; // the epoch-based driver (Algo::kEpochBased)
    return meta;
}

namespace {
std::string json_number(double v) {
    char buf[64];
    auto res = std::to_chars(buf, buf + sizeof(buf), v); // shortest round-trip form
    std::string s(buf, res.ptr);
    if (s.find_first_of(".en") == std::string::npos) // integral doubles print as "1.0"
        s += ".0";
    return s;
}
} // namespace

std::string stats_json(const RunStats &s, double eps, double delta, std::uint64_t seed, int bound, int allocator,
                       int gpus) {
    std::ostringstream j;
    bool first = true;
    auto key = [&](const char *k) -> std::ostringstream & {
        j << (first ? "{\n" : ",\n") << "  \"" << k << "\": ";
        first = false;
        return j;
    };
    key("schema_version") << 1;
    key("epochs") << s.epochs;
    key("samples") << s.samples;
    key("barrier_s") << json_number(0.0);
    key("comm_mib_per_epoch") << json_number(gpus > 1 ? static_cast<double>(s.n + 1) * 4.0 * (gpus - 1) / (1024.0 * 1024.0) : 0.0);
    key("adaptive_s") << json_number(s.adaptive_s);
    key("diameter_s") << json_number(s.diameter_s);
    key("calibration_s") << json_number(s.calibration_s);
    key("transition_s") << json_number(0.0);
    key("reduce_s") << json_number(s.reduce_s);
    key("check_s") << json_number(s.check_s);
    key("bcast_s") << json_number(0.0);
    key("wall_s") << json_number(s.wall_s);
    key("tau") << s.tau;
    key("omega") << s.omega;
    key("calibration_samples") << s.calibration_samples;
    key("discarded_samples") << s.discarded_samples;
    key("n0") << s.n0;
    key("n") << s.n;
    key("m") << s.m;
    key("diameter_upper_bound") << s.diameter_upper_bound;
    key("vertex_diameter_bound") << s.vertex_diameter_bound;
    key("eps") << json_number(eps);
    key("delta") << json_number(delta);
    key("ranks") << gpus;
    key("threads") << 1;
    key("seed") << seed;
    key("algo") << 2;
    key("bound") << (bound == 0 ? "\"hoeffding\"" : "\"eb\"");
    key("allocator") << (allocator == 0 ? "\"uniform\"" : "\"weighted\"");
    j << "\n}\n";
    return j.str();
}

} // namespace ebc
