// shim_acceptance.cpp -- drives the drop-in shim girih::gpu::run with the REFERENCE'S OWN signature
// (include/girih_gpu.hpp: girih::gpu::run(state, T, dw, wf, shape, variant, groups, opts)) on the
// reference's own ProblemState, the way a maintainer swaps the call site, and
// checks it against the reference's own oracle girih::naive_sweep (proj/src/stencil.cpp:115-127):
//
//  1. acceptance #1 (proj/tests/acceptance.cpp:37-66): 4 stencils x 48^3 x T = 16 x 5 thread-group
//     shapes x {relaxed, FED} x groups {1, 2}, bitwise in u AND v;
//  2. the invalid configurations of proj/tests/test_engine.cpp:223-238 throw
//     std::invalid_argument (incl. resolve_block_size's bs_z % T_z, engine.cpp:270-283);
//  3. T = 0 is a no-op with zero work; a second run continues from the previous level with a
//     padded leading dimension (test_engine.cpp:149-168);
//  4. RunOptions (test_engine.cpp:170-215): the ledger sees every point updated exactly once and
//     the trace CSV carries the reference's columns.
//
// Built by oracle/Makefile against the unmodified reference core (test infrastructure); run by
// tests/test_shim.py on a GPU. Prints PASS/FAIL lines, exits 1 on any failure.
#include <cstdio>
#include <sstream>
#include <stdexcept>
#include <string>

#include "girih/engine.hpp"
#include "girih/stencil.hpp"
#include "girih_gpu.hpp"

using namespace girih;

namespace {

int g_fail = 0;

void report(bool ok, const std::string& what) {
    std::printf("%s  %s\n", ok ? "PASS" : "FAIL", what.c_str());
    if (!ok) ++g_fail;
}

bool same(const ProblemState& a, const ProblemState& b) {
    return a.t_current == b.t_current && a.u.bitwise_equal(b.u) && a.v.bitwise_equal(b.v);
}

template <class F>
bool throws_invalid(F&& f) {
    try {
        f();
    } catch (const std::invalid_argument&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

}  // namespace

int main() {
    // ---- 1. acceptance #1 through the reference-signature shim ----
    {
        const GridSpec grid{48, 48, 48, 0};
        const long T = 16;
        const ThreadGroupShape shapes[] = {
            {1, 1, 1, 1}, {2, 1, 1, 1}, {1, 2, 1, 1}, {2, 1, 2, 1}, {1, 2, 3, 1}};
        for (int k = 0; k < 4; ++k) {
            const StencilKind kind = static_cast<StencilKind>(k);
            const int dw = traits(kind).radius == 1 ? 8 : 16;
            ProblemState oracle = init_state(kind, grid, 1234);
            naive_sweep(oracle, T);
            int cases = 0, bad = 0;
            for (const ThreadGroupShape& shape : shapes)
                for (WavefrontVariant variant :
                     {WavefrontVariant::RelaxedPipelined, WavefrontVariant::FixedExecutionToData})
                    for (int groups : {1, 2}) {
                        ProblemState tiled = init_state(kind, grid, 1234);
                        const PerfReport rep =
                            gpu::run(tiled, T, dw, WavefrontSpec{4, 0}, shape, variant, groups);
                        ++cases;
                        if (!same(tiled, oracle) || rep.lups != 48LL * 48 * 48 * T) ++bad;
                    }
            report(bad == 0, std::string("acceptance #1 ") + traits(kind).name + ": " +
                                 std::to_string(cases - bad) + "/" + std::to_string(cases) +
                                 " shim runs bitwise identical to naive_sweep (u and v)");
        }
    }
    // ---- 2. invalid configurations are rejected up front (test_engine.cpp:223-238) ----
    {
        const GridSpec g{16, 16, 16, 0};
        ProblemState s = init_state(StencilKind::Const7pt, g, 2);
        const WavefrontSpec wf{2, 0};
        const ProblemState fresh = s;
        bool ok = true;
        ok &= throws_invalid([&] {
            gpu::run(s, 4, 7, wf, {1, 1, 1, 1}, WavefrontVariant::RelaxedPipelined, 1);
        });  // D_w not a multiple of 2R
        ok &= throws_invalid([&] {
            gpu::run(s, 4, 8, wf, {1, 3, 1, 1}, WavefrontVariant::RelaxedPipelined, 1);
        });  // T_y > 2
        ok &= throws_invalid([&] {
            gpu::run(s, 4, 8, wf, {1, 1, 1, 1}, WavefrontVariant::RelaxedPipelined, 0);
        });  // no thread group
        ok &= throws_invalid([&] {
            gpu::run(s, -1, 8, wf, {1, 1, 1, 1}, WavefrontVariant::RelaxedPipelined, 1);
        });  // negative steps
        ok &= throws_invalid([&] {
            gpu::run(s, 4, 8, WavefrontSpec{2, 7}, {1, 1, 2, 1},
                     WavefrontVariant::RelaxedPipelined, 1);
        });  // block size not a multiple of T_z
        report(ok && same(s, fresh), "invalid configurations throw std::invalid_argument, state untouched");
    }
    // ---- 3. T = 0; continuation from an odd level with pad_x = 2 ----
    {
        const GridSpec g{16, 16, 16, 0};
        ProblemState s = init_state(StencilKind::Const7pt, g, 2);
        const ProblemState fresh = init_state(StencilKind::Const7pt, g, 2);
        const PerfReport rep =
            gpu::run(s, 0, 8, WavefrontSpec{1, 0}, {1, 1, 1, 1}, WavefrontVariant::RelaxedPipelined, 1);
        report(rep.lups == 0 && rep.glups == 0.0 && same(s, fresh), "T = 0 is a no-op with zero work");

        const GridSpec gp{16, 16, 16, 2};
        for (int k = 0; k < 4; ++k) {
            const StencilKind kind = static_cast<StencilKind>(k);
            const int dw = traits(kind).radius == 1 ? 8 : 16;
            ProblemState want = init_state(kind, gp, 9);
            naive_sweep(want, 7);
            ProblemState t = init_state(kind, gp, 9);
            gpu::run(t, 3, dw, WavefrontSpec{2, 0}, {2, 1, 1, 1}, WavefrontVariant::FixedExecutionToData, 1);
            gpu::run(t, 4, dw, WavefrontSpec{2, 0}, {1, 1, 2, 1}, WavefrontVariant::RelaxedPipelined, 1);
            report(t.t_current == 7 && same(t, want),
                   std::string("continuation 3 + 4 steps, pad_x = 2: ") + traits(kind).name);
        }
    }
    // ---- 4. RunOptions: exactly-once ledger and the execution trace ----
    {
        const GridSpec g{16, 16, 16, 0};
        for (int k = 0; k < 4; ++k) {
            const StencilKind kind = static_cast<StencilKind>(k);
            const int dw = traits(kind).radius == 1 ? 8 : 16;
            ProblemState s = init_state(kind, g, 3);
            ProblemState want = init_state(kind, g, 3);
            naive_sweep(want, 8);
            UpdateLedger ledger(g, 8);
            RunOptions opts;
            opts.ledger = &ledger;
            gpu::run(s, 8, dw, WavefrontSpec{2, 0}, {2, 1, 2, 1}, WavefrontVariant::RelaxedPipelined, 2,
                     opts);
            report(ledger.all_exactly_once() && same(s, want),
                   std::string("ledger: every point updated exactly once, bitwise: ") + traits(kind).name);
        }
        // fused passes, forced z chunks and an odd step count: the tiles and z chunks of every
        // pass must partition every step's updates
        {
            ProblemState s = init_state(StencilKind::Var7pt, GridSpec{37, 32, 41, 1}, 5);
            UpdateLedger ledger(GridSpec{37, 32, 41, 1}, 9);
            RunOptions opts;
            opts.ledger = &ledger;
            gpu::GpuConfig cfg;
            cfg.tb = 2;
            cfg.zchunks = 3;
            gpu::run(s, 9, 8, WavefrontSpec{2, 0}, {1, 1, 1, 1}, WavefrontVariant::RelaxedPipelined, 1,
                     opts, cfg);
            report(ledger.all_exactly_once(), "ledger: var7pt 37x32x41, TB = 2, 3 z chunks, odd T");
        }
        ProblemState s = init_state(StencilKind::Const7pt, g, 8);
        std::ostringstream trace;
        RunOptions opts;
        opts.trace_out = &trace;
        const PerfReport rep =
            gpu::run(s, 8, 8, WavefrontSpec{2, 0}, {1, 1, 2, 1}, WavefrontVariant::RelaxedPipelined, 2, opts);
        std::istringstream is(trace.str());
        std::string header;
        std::getline(is, header);
        long long rows = 0;
        bool ordered = true;
        for (std::string line; std::getline(is, line); ++rows) {
            unsigned long long a = 0, b = 0;
            int tile = -1, group = -1;
            if (std::sscanf(line.c_str(), "%d,%d,%llu,%llu", &tile, &group, &a, &b) != 4 ||
                tile != rows || group < 0 || b < a)
                ordered = false;
        }
        report(header == "tile,group,start_ns,end_ns" && rows > 0 && rows == rep.tiles && ordered,
               "trace CSV: reference columns, one row per work unit (" + std::to_string(rows) + ")");
    }
    std::printf("%s: %d failure(s)\n", g_fail ? "FAIL" : "PASS", g_fail);
    return g_fail ? 1 : 0;
}
