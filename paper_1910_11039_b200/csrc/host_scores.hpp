// Score files, score comparison and the stats JSON of the reference CLI (see host_scores.cpp).
#pragma once

#include <cstdint>
#include <map>
#include <string>
#include <vector>

#include "epoch_driver.hpp"
#include "host_common.hpp"

namespace ebc {

struct ScoreTable { // ScoreFile (score_io.hpp:20-24)
    std::map<std::string, std::string> meta;
    std::vector<std::uint64_t> vertex_ids;
    std::vector<double> scores;
};

struct CompareReport { // score_io.hpp:31-37
    double max_abs_error = 0.0;
    std::uint64_t vertices_above_eps = 0;
    double top10_overlap = 0.0, top100_overlap = 0.0;
    std::uint64_t vertices = 0;
};

void write_scores(const std::string &path, const ScoreTable &t);
ScoreTable read_scores(const std::string &path);
CompareReport compare_scores(const ScoreTable &approx, const ScoreTable &exact, double eps);
std::map<std::string, std::string> run_meta(double eps, double delta, std::uint64_t seed, std::uint64_t tau);
std::string stats_json(const RunStats &s, double eps, double delta, std::uint64_t seed, int bound, int allocator,
                       int gpus);

} // namespace ebc
