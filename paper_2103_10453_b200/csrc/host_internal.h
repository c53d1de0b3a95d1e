// host_internal.h -- host-side types shared by the C-ABI implementation.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "common.cuh"

namespace plse_host {

// ReducedGraph (lsgraph.hpp:67-109) restricted to what the device path and
// the ABI view need: cells, CSR domains, l, prefilled triples.
struct GraphH {
    int n = 0, nv = 0, l = 0;
    std::vector<int32_t> cell_row, cell_col, dom_off;
    std::vector<uint16_t> dom;
    std::vector<int32_t> prefilled;  // row, col, symbol triples
};

std::vector<uint16_t> generate_instance(int n, double r, uint64_t seed);
std::vector<uint16_t> parse_instance(const std::string& text, int& n_out);
GraphH preprocess(int n, const uint16_t* grid);

struct VerifyResult {
    bool legal = false;
    int score = 0;
    std::vector<std::string> problems;
};
std::vector<uint16_t> to_grid(const GraphH& g, const uint16_t* colors);
VerifyResult verify_certificate(int n, const uint16_t* inst, int m, const uint16_t* cert);

struct ExactResult {
    int optimum_f = 0;
    bool exact = true;
    int64_t nodes = 0;
    std::vector<uint16_t> certificate;  // |V| colours
};
ExactResult solve_exact(const GraphH& g, int64_t node_budget);

}  // namespace plse_host

struct plse_graph_h {
    plse_host::GraphH g;
};
