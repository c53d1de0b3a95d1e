// host_graph.cpp -- host side of the boundary that the north star keeps on the
// CPU: instance generation / parsing and the PLSE -> partial-colouring
// reduction.  Same semantics as the reference (cited per function), written
// for this library; exported through include/plse_b200.h.
#include <cstring>
#include <sstream>
#include <algorithm>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "host_internal.h"

namespace plse_host {

using plse_dev::Xoshiro;
using plse_dev::derive_seed;

// instance.hpp:204-262 -- random partial Latin square: uniform empty cell,
// uniform admissible symbol, resample on dead cells, restart with stream
// (seed, 4, restart) after 50 n^2 consecutive failures, at most 100 restarts.
std::vector<uint16_t> generate_instance(int n, double r, uint64_t seed) {
    if (n <= 0) throw std::invalid_argument("order must be positive");
    if (!(r > 0.0 && r < 1.0)) throw std::invalid_argument("fill ratio must be in (0,1)");
    const int cells = n * n;
    const int want = static_cast<int>(r * cells);
    const int fail_cap = 50 * cells;
    std::vector<uint16_t> grid(static_cast<size_t>(cells));
    std::vector<uint8_t> row_has(static_cast<size_t>(n) * (n + 1)), col_has(static_cast<size_t>(n) * (n + 1));
    std::vector<int> open(static_cast<size_t>(cells));
    std::vector<uint16_t> cand;
    for (int attempt = 0; attempt < 100; ++attempt) {
        Xoshiro rng(derive_seed(seed, 4, static_cast<uint64_t>(attempt)));
        std::fill(grid.begin(), grid.end(), 0);
        std::fill(row_has.begin(), row_has.end(), 0);
        std::fill(col_has.begin(), col_has.end(), 0);
        for (int q = 0; q < cells; ++q) open[q] = q;
        int n_open = cells, placed = 0, misses = 0;
        while (placed < want && misses < fail_cap) {
            const int slot = static_cast<int>(rng.below(static_cast<uint64_t>(n_open)));
            const int cell = open[slot];
            const int rr = cell / n, cc = cell % n;
            cand.clear();
            for (int s = 1; s <= n; ++s)
                if (!row_has[rr * (n + 1) + s] && !col_has[cc * (n + 1) + s]) cand.push_back(static_cast<uint16_t>(s));
            if (cand.empty()) {
                ++misses;
                continue;
            }
            const uint16_t s = cand[rng.below(cand.size())];
            grid[cell] = s;
            row_has[rr * (n + 1) + s] = 1;
            col_has[cc * (n + 1) + s] = 1;
            open[slot] = open[--n_open];
            ++placed;
            misses = 0;
        }
        if (placed == want) return grid;
    }
    throw std::runtime_error("instance generation failed: (n=" + std::to_string(n) + ", r=" + std::to_string(r) +
                             ") exhausted the retry budget");
}

// instance.hpp:107-170 -- "n" header line, then n rows of n integers; blank
// lines skipped; errors carry the 1-based line number.
std::vector<uint16_t> parse_instance(const std::string& text, int& n_out) {
    std::istringstream in(text);
    std::string line;
    int lineno = 0;
    auto fail = [&](int at, const std::string& msg) -> void {
        throw std::runtime_error("line " + std::to_string(at) + ": " + msg);
    };
    auto next = [&](const char* what) {
        while (std::getline(in, line)) {
            ++lineno;
            if (line.find_first_not_of(" \t\r") != std::string::npos) return;
        }
        fail(lineno + 1, std::string("unexpected end of input, expected ") + what);
    };
    next("grid order");
    long n = 0;
    {
        std::istringstream ls(line);
        if (!(ls >> n) || n <= 0) fail(lineno, "malformed header: expected positive grid order");
        std::string rest;
        if (ls >> rest) fail(lineno, "malformed header: trailing tokens");
    }
    if (n > 0xFFFF) fail(lineno, "grid order too large");
    std::vector<uint16_t> grid(static_cast<size_t>(n) * n);
    for (long rr = 0; rr < n; ++rr) {
        next("grid row");
        std::istringstream ls(line);
        for (long cc = 0; cc < n; ++cc) {
            long v = 0;
            if (!(ls >> v)) fail(lineno, "malformed row: expected " + std::to_string(n) + " entries");
            if (v < 0 || v > n) fail(lineno, "symbol out of range: " + std::to_string(v));
            grid[rr * n + cc] = static_cast<uint16_t>(v);
        }
        std::string rest;
        if (ls >> rest) fail(lineno, "malformed row: trailing tokens");
    }
    for (long rr = 0; rr < n; ++rr) {
        std::vector<int> seen(static_cast<size_t>(n) + 1, 0);
        for (long cc = 0; cc < n; ++cc) {
            const int s = grid[rr * n + cc];
            if (s && seen[s]++) fail(static_cast<int>(2 + rr), "duplicate symbol " + std::to_string(s) + " in row " + std::to_string(rr));
        }
    }
    for (long cc = 0; cc < n; ++cc) {
        std::vector<int> seen(static_cast<size_t>(n) + 1, 0);
        for (long rr = 0; rr < n; ++rr) {
            const int s = grid[rr * n + cc];
            if (s && seen[s]++) fail(static_cast<int>(2 + rr), "duplicate symbol " + std::to_string(s) + " in column " + std::to_string(cc));
        }
    }
    n_out = static_cast<int>(n);
    return grid;
}

// lsgraph.hpp:115-211 -- drop prefilled cells (removing their symbol from the
// row/column domains), drop cells left with domain {0} (counted in l), keep
// the rest row-major with domains {0} u free symbols.
GraphH preprocess(int n, const uint16_t* grid) {
    GraphH g;
    g.n = n;
    std::vector<uint8_t> used(static_cast<size_t>(2) * n * (n + 1), 0);
    for (int cell = 0; cell < n * n; ++cell) {
        const int s = grid[cell];
        if (!s) continue;
        used[(cell / n) * (n + 1) + s] = 1;
        used[(n + cell % n) * (n + 1) + s] = 1;
        g.prefilled.push_back(cell / n);
        g.prefilled.push_back(cell % n);
        g.prefilled.push_back(s);
    }
    g.dom_off.push_back(0);
    for (int cell = 0; cell < n * n; ++cell) {
        if (grid[cell]) continue;
        const int rr = cell / n, cc = cell % n;
        const size_t mark = g.dom.size();
        g.dom.push_back(0);
        for (int s = 1; s <= n; ++s)
            if (!used[rr * (n + 1) + s] && !used[(n + cc) * (n + 1) + s]) g.dom.push_back(static_cast<uint16_t>(s));
        if (g.dom.size() == mark + 1) {
            g.dom.resize(mark);
            ++g.l;
            continue;
        }
        g.cell_row.push_back(rr);
        g.cell_col.push_back(cc);
        g.dom_off.push_back(static_cast<int32_t>(g.dom.size()));
    }
    g.nv = static_cast<int>(g.cell_row.size());
    return g;
}


// coloring.hpp:171-183 to_grid: prefilled symbols plus the solution's
// coloured cells (colours are symbols; 0 leaves the cell empty).
std::vector<uint16_t> to_grid(const GraphH& g, const uint16_t* colors) {
    std::vector<uint16_t> out(static_cast<size_t>(g.n) * g.n, 0);
    for (size_t t = 0; t + 2 < g.prefilled.size(); t += 3)
        out[g.prefilled[t] * g.n + g.prefilled[t + 1]] = static_cast<uint16_t>(g.prefilled[t + 2]);
    for (int v = 0; v < g.nv; ++v) {
        const int k = colors[v];
        if (k == 0) continue;
        // Coloring::assign (coloring.hpp:44-48) rejects colours outside the domain
        if (!std::binary_search(g.dom.begin() + g.dom_off[v], g.dom.begin() + g.dom_off[v + 1], (uint16_t)k))
            throw std::invalid_argument("assignment leaves vertex domain");
        out[g.cell_row[v] * g.n + g.cell_col[v]] = static_cast<uint16_t>(k);
    }
    return out;
}

// verify.hpp:20-73: order, pre-filled cells, then row and column duplicates,
// in that order and with the same wording.
VerifyResult verify_certificate(int n, const uint16_t* inst, int m, const uint16_t* cert) {
    VerifyResult r;
    if (m != n) {
        r.problems.push_back("order mismatch: instance " + std::to_string(n) + ", certificate " + std::to_string(m));
        return r;
    }
    auto cell = [](int a, int b) { return "(" + std::to_string(a) + "," + std::to_string(b) + ")"; };
    for (int a = 0; a < n; ++a)
        for (int b = 0; b < n; ++b) {
            const int e = inst[a * n + b], got = cert[a * n + b];
            if (e != 0 && got != e)
                r.problems.push_back("pre-filled cell " + cell(a, b) + " altered: expected " + std::to_string(e) +
                                     ", got " + std::to_string(got));
        }
    std::vector<int> first(static_cast<size_t>(n) + 1);
    for (int pass = 0; pass < 2; ++pass)
        for (int line = 0; line < n; ++line) {
            std::fill(first.begin(), first.end(), -1);
            for (int t = 0; t < n; ++t) {
                const int s = pass == 0 ? cert[line * n + t] : cert[t * n + line];
                if (s == 0) continue;
                if (s > n) throw std::invalid_argument("symbol out of range");
                if (first[s] < 0) {
                    first[s] = t;
                    continue;
                }
                r.problems.push_back("duplicate symbol " + std::to_string(s) + (pass == 0 ? " in row " : " in column ") +
                                     std::to_string(line) + (pass == 0 ? " at columns " : " at rows ") +
                                     std::to_string(first[s]) + " and " + std::to_string(t));
            }
        }
    for (int q = 0; q < n * n; ++q) r.score += cert[q] != 0;
    r.legal = r.problems.empty();
    return r;
}

// oracle.hpp:24-136 ExactSolver / solve_exact: fail-first branch and bound (fewest feasible non-zero
// colours first, lowest id on ties), colours ascending with 0 last, pruning on zeros + forced zeros
// >= incumbent, node budget.  used(v, k) -- neighbours of v coloured k -- is the row + column count of
// k, since the neighbours of a cell are exactly the vertices of its row and column.  The recursion of
// the reference is an explicit stack here (|V| can be deep).
ExactResult solve_exact(const GraphH& g, int64_t node_budget) {
    const int n = g.n, nv = g.nv, w = n + 1;
    ExactResult res;
    std::vector<int16_t> assign(nv, -1), best(nv, 0);
    std::vector<int32_t> rcnt((size_t)n * w, 0), ccnt((size_t)n * w, 0);
    int best_f = nv;
    bool exhausted = false;
    int64_t nodes = 0;
    auto used = [&](int v, int k) { return rcnt[(size_t)g.cell_row[v] * w + k] + ccnt[(size_t)g.cell_col[v] * w + k]; };
    auto adjust = [&](int v, int k, int d) {
        rcnt[(size_t)g.cell_row[v] * w + k] += d;
        ccnt[(size_t)g.cell_col[v] * w + k] += d;
    };
    struct Frame {
        int zeros, pick, ki, applied;
        int stage;  // 0 = enter, 1 = colours, 2 = zero branch done
    };
    std::vector<Frame> st;
    st.push_back({0, -1, 0, 0, 0});
    while (!st.empty()) {
        Frame& fr = st.back();
        if (fr.stage == 0) {
            if (exhausted || ++nodes > node_budget) {
                exhausted = true;
                st.pop_back();
                continue;
            }
            int pick = -1, pick_feasible = 0, forced = 0;
            for (int v = 0; v < nv; ++v) {
                if (assign[v] != -1) continue;
                int feasible = 0;
                for (int a = g.dom_off[v]; a < g.dom_off[v + 1]; ++a)
                    if (g.dom[a] != 0 && used(v, g.dom[a]) == 0) ++feasible;
                if (feasible == 0) {
                    ++forced;
                    continue;
                }
                if (pick < 0 || feasible < pick_feasible) {
                    pick = v;
                    pick_feasible = feasible;
                }
            }
            if (fr.zeros + forced >= best_f) {  // prune (solve_exact sets prune)
                st.pop_back();
                continue;
            }
            if (pick < 0) {
                best_f = fr.zeros + forced;
                for (int v = 0; v < nv; ++v) best[v] = assign[v] == -1 ? 0 : assign[v];
                st.pop_back();
                continue;
            }
            fr.pick = pick;
            fr.ki = g.dom_off[pick];
            fr.stage = 1;
        }
        if (fr.stage == 1) {
            if (fr.applied) {
                adjust(fr.pick, fr.applied, -1);
                fr.applied = 0;
                if (exhausted) fr.ki = g.dom_off[fr.pick + 1];
            }
            while (fr.ki < g.dom_off[fr.pick + 1]) {
                const int k = g.dom[fr.ki++];
                if (k == 0 || used(fr.pick, k) != 0) continue;
                assign[fr.pick] = (int16_t)k;
                adjust(fr.pick, k, +1);
                fr.applied = k;
                break;
            }
            if (fr.applied) {
                const int z = fr.zeros;
                st.push_back({z, -1, 0, 0, 0});
                continue;
            }
            fr.stage = 2;
            if (!exhausted) {
                assign[fr.pick] = 0;
                const int z = fr.zeros + 1;
                st.push_back({z, -1, 0, 0, 0});
                continue;
            }
        }
        assign[fr.pick] = -1;
        st.pop_back();
    }
    res.optimum_f = best_f;
    res.exact = !exhausted;
    res.nodes = nodes;
    res.certificate.assign(best.begin(), best.end());
    return res;
}

}  // namespace plse_host
