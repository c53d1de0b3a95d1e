// Probe of the C++ host API (include/plse_b200.hpp) driven by tests/test_cpp_host.py: each mode
// prints what the test compares against the Python front-end and the compiled reference.
#include <cstdio>
#include <iostream>

#include "plse_b200.hpp"

using namespace plse_b200;

int main(int argc, char** argv) {
    const std::string mode = argc > 1 ? argv[1] : "";
    try {
        if (mode == "instance") {  // generate -> serialize -> parse round trip, derive_seed
            const PlsInstance g = generate_instance(std::atoi(argv[2]), std::atof(argv[3]), std::strtoull(argv[4], 0, 10));
            const std::string text = serialize_instance(g);
            std::cout << text << (parse_instance(text) == g ? "roundtrip ok\n" : "roundtrip FAIL\n");
            std::cout << derive_seed(88, stream_tag::kInstanceGen, 3) << '\n';
            const ReducedGraph r = preprocess(g);
            const InstanceBounds b = compute_bounds(r);
            std::cout << r.vertex_count() << ' ' << b.l << ' ' << b.upper_bound << '\n';
            return 0;
        }
        if (mode == "exact") {  // solve_exact + to_grid + verify_certificate on an instance file
            const PlsInstance g = load_instance(argv[2]);
            const ReducedGraph r = preprocess(g);
            const OracleResult o = solve_exact(r, std::strtoll(argv[3], 0, 10));
            std::cout << o.optimum_f << ' ' << o.exact << ' ' << o.nodes << '\n';
            for (uint16_t c : o.certificate) std::cout << c << ' ';
            std::cout << '\n';
            const PlsInstance cert = to_grid(g, r, o.certificate);
            const VerifyReport v = verify_certificate(g, cert);
            std::cout << v.legal << ' ' << v.score << ' ' << v.problems.size() << '\n';
            return 0;
        }
        if (mode == "verify") {  // problems of a certificate file against an instance file
            const VerifyReport v = verify_certificate(load_instance(argv[2]), load_instance(argv[3]));
            std::cout << v.legal << ' ' << v.score << '\n';
            for (const auto& p : v.problems) std::cout << p << '\n';
            return 0;
        }
        if (mode == "json") {  // result_to_json for fixed fields + a config from argv
            RunResult res;
            res.best_f = 3;
            res.best_score = 80;
            res.proven_optimal = std::atoi(argv[2]) != 0;
            res.stop_reason = argv[3];
            res.l = 2;
            res.upper_bound = 83;
            res.vertex_count = 50;
            res.generations = 5;
            res.total_iterations = 12345;
            res.elapsed_seconds = std::atof(argv[4]);
            SolverConfig c;
            c.p = std::atoi(argv[5]);
            c.alpha = std::atof(argv[6]);
            c.crossover.mode = parse_crossover(argv[7]);
            c.master_seed = std::strtoull(argv[8], 0, 10);
            c.limits.time_seconds = std::atof(argv[9]);
            c.variant = parse_variant(argv[10]);
            c.workers = 2;
            std::cout << result_to_json("instance.txt", 12, res, c, std::atoi(argv[11]) != 0) << '\n';
            return 0;
        }
        if (mode == "errors") {  // the reference's exception types
            try {
                parse_instance("2\n1 1\n0 0\n");
            } catch (const std::runtime_error& e) {
                std::cout << "runtime_error: " << e.what() << '\n';
            }
            try {
                SolverConfig c;
                c.p = 1;
                c.validate();
            } catch (const std::invalid_argument& e) {
                std::cout << "invalid_argument: " << e.what() << '\n';
            }
            try {
                run(generate_instance(6, 0.5, 1), SolverConfig{});
            } catch (const CudaError& e) {
                std::cout << "CudaError\n";
            } catch (const std::exception& e) {
                std::cout << "other: " << e.what() << '\n';
            }
            return 0;
        }
    } catch (const std::exception& e) {
        std::cout << "exception: " << e.what() << '\n';
        return 1;
    }
    return 2;
}
