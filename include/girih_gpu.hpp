// girih_gpu.hpp -- header-only C++ shim over the C ABI (girih_gpu.h) shaped like the reference's
// engine entry point, so the reference's own host code switches to the GPU with a one-line change:
//
//     #include "girih/engine.hpp"      // reference: ProblemState, PerfReport, WavefrontSpec, ...
//     #include "girih_gpu.hpp"         // this shim
//     girih::run(state, T, dw, wf, shape, variant, groups);          // before (engine.cpp:332-418)
//     girih::gpu::run(state, T, dw, wf, shape, variant, groups);     // after: same signature
//
// Errors are rethrown with the reference's exception classes: std::invalid_argument for
// inadmissible input (engine.cpp:335-337, geometry.cpp:39-43), std::logic_error for handle misuse,
// std::runtime_error for CUDA / NCCL / out-of-memory failures.
#pragma once

#include <algorithm>
#include <ostream>
#include <stdexcept>
#include <string>
#include <vector>

#include "girih/engine.hpp"
#include "girih/geometry.hpp"
#include "girih/stencil.hpp"
#include "girih_gpu.h"

namespace girih {
namespace gpu {

// GPU execution parameters (girih_gpu_config): they replace (dw, wf, shape, variant, n_groups).
struct GpuConfig {
    int tb = 0;        // time steps fused per HBM pass; 0 = default for the kind
    int variant = -1;  // compiled tile variant; -1 = default for tb
    int zchunks = 0;   // z chunks per tile column; 0 = model
    int ngpus = 1;     // z-slab decomposition across devices [device, device + ngpus)
    int device = 0;
    int graphs = 0;
    int chain = 0;     // 1 = chain same-depth passes into one dependency-driven launch; -1 = off;
                       // 0 = auto (small grids)
    int tile_order = 0;  // W > 0 = column strips of W tiles per z-chunk row; -1 = row-major; 0 = auto
};

// PerfReport (engine.hpp:93-98) plus the GPU-side timings.
struct GpuReport : PerfReport {
    double kernel_seconds = 0, h2d_seconds = 0, d2h_seconds = 0, mlups = 0;
    double model_bytes_per_lup = 0;
    int tb_used = 0, n_launches = 0;
};

inline void check(int rc) {
    if (rc == GIRIH_OK) return;
    const std::string msg = girih_gpu_last_error();
    if (rc == GIRIH_EINVAL) throw std::invalid_argument(msg);
    if (rc == GIRIH_ESTATE) throw std::logic_error(msg);
    throw std::runtime_error(msg);
}

inline girih_gpu_config to_c(const GpuConfig& c) {
    girih_gpu_config o{};
    o.tb = c.tb;
    o.variant = c.variant;
    o.zchunks = c.zchunks;
    o.ngpus = c.ngpus;
    o.exact = 1;
    o.device = c.device;
    o.graphs = c.graphs;
    o.chain = c.chain;
    o.tile_order = c.tile_order;
    return o;
}

// Non-owning view of a reference ProblemState (stencil.hpp:83-98).
struct StateView {
    girih_state_view v{};
    std::vector<const double*> coeffs;
    explicit StateView(ProblemState& s) {
        for (auto& f : s.coeffs) coeffs.push_back(f.data());
        v.kind = static_cast<int>(s.kind);
        v.nx = s.grid.nx;
        v.ny = s.grid.ny;
        v.nz = s.grid.nz;
        v.pad_x = s.grid.pad_x;
        v.t_current = s.t_current;
        v.u = s.u.data();
        v.v = s.v.data();
        v.coeffs = coeffs.data();
        v.n_coeffs = static_cast<int>(coeffs.size());
        for (int c = 0; c < 5; ++c) v.cc[c] = s.cc[c];
    }
};

// Advances the state by `steps` on the GPU (upload, fused passes, download of u and v).
inline GpuReport run(ProblemState& state, long steps, const GpuConfig& cfg) {
    StateView sv(state);
    girih_gpu_config c = to_c(cfg);
    girih_gpu_report r{};
    check(girih_gpu_run(&sv.v, steps, &c, &r));
    state.t_current = static_cast<long>(sv.v.t_current);
    GpuReport out;
    out.wall_seconds = r.wall_s;
    out.lups = r.lups;
    out.glups = r.wall_s > 0 ? r.lups / r.wall_s / 1e9 : 0.0;
    out.tiles = r.units;  // work units (tile column x z chunk per pass)
    out.kernel_seconds = r.kernel_s;
    out.h2d_seconds = r.h2d_s;
    out.d2h_seconds = r.d2h_s;
    out.mlups = r.kernel_s > 0 ? r.lups / r.kernel_s / 1e6 : 0.0;
    out.model_bytes_per_lup = r.model_bytes_per_lup;
    out.tb_used = r.tb_used;
    out.n_launches = r.n_launches;
    return out;
}

namespace detail {
inline void write_trace_csv(void* ctx, const girih_gpu_trace_record* r, long long n) {
    // the reference's TileScheduler::dump_trace_csv columns (scheduler.cpp:96-101): a GPU
    // "tile" is a work unit (pass, tile column x z chunk), its "group" the CTA that ran it
    std::ostream& os = *static_cast<std::ostream*>(ctx);
    os << "tile,group,start_ns,end_ns\n";
    for (long long i = 0; i < n; ++i)
        os << i << ',' << r[i].cta << ',' << r[i].start_ns << ',' << r[i].end_ns << '\n';
}
}  // namespace detail

// Signature-compatible drop-in for girih::run (engine.hpp:113-115). The CPU-engine parameters
// are validated exactly as the reference validates them (so inadmissible configurations still
// throw std::invalid_argument; engine.cpp:270-290, 333-337, geometry.cpp:9-15, 39-43) and are
// otherwise not used by the GPU path. RunOptions (engine.hpp:100-103) are honoured: trace_out
// receives the per-unit execution trace CSV and ledger the exactly-once update counts of the
// GPU run (girih_gpu_run_ex).
inline PerfReport run(ProblemState& state, long steps, int dw, const WavefrontSpec& wf,
                      const ThreadGroupShape& shape, WavefrontVariant variant, int n_groups,
                      const RunOptions& opts = {}, const GpuConfig& cfg = {}) {
    (void)variant;
    // engine.cpp:285-290, 333-335
    if (shape.tx < 1 || shape.ty < 1 || shape.tz < 1)
        throw std::invalid_argument("thread group axes must be positive");
    if (shape.ty > 2) throw std::invalid_argument("T_y must be 1 or 2");
    if (shape.tc != 1) throw std::invalid_argument("T_c must be 1 for scalar stencils");
    if (n_groups < 1) throw std::invalid_argument("need at least one thread group");
    if (steps < 0) throw std::invalid_argument("negative step count");
    if (steps > 0) {
        // geometry admissibility the CPU engine enforces (geometry.cpp:9-15, 39-43)
        const int R = state.radius;
        if (R < 1 || dw < 2 * R || dw % (2 * R) != 0)
            throw std::invalid_argument("build_tessellation: D_w must be a multiple of 2R");
        if (state.grid.ny < dw || state.grid.ny % dw != 0)
            throw std::invalid_argument("build_tessellation: Ny must be a multiple of D_w");
        if (wf.nf < 1) throw std::invalid_argument("wavefront_width: need R >= 1, N_F >= 1, D_w >= 2R");
        // resolve_block_size (engine.cpp:270-283): the wavefront block must split over T_z
        const int ww = wavefront_width(dw, wf.nf, R);
        int bs = wf.bs_z > 0 ? wf.bs_z : default_block_size(ww, shape.tz);
        if (wf.bs_z <= 0) {
            const int unit = default_block_size(1, shape.tz);
            const int cap = std::max(unit, (state.grid.nz + unit - 1) / unit * unit);
            bs = std::min(bs, cap);
        }
        if (bs < shape.tz || bs % shape.tz != 0)
            throw std::invalid_argument("wavefront block size must be a positive multiple of T_z");
    }
    if (!opts.trace_out && !opts.ledger) return run(state, steps, cfg);
    // instrumented run
    StateView sv(state);
    girih_gpu_config c = to_c(cfg);
    girih_gpu_report r{};
    girih_gpu_run_options o{};
    if (opts.trace_out) {
        o.trace_cb = &detail::write_trace_csv;
        o.trace_ctx = opts.trace_out;
    }
    std::vector<unsigned> counts;
    if (opts.ledger) {
        counts.assign(static_cast<size_t>(steps) * state.grid.nx * state.grid.ny * state.grid.nz, 0u);
        o.ledger = counts.data();
    }
    check(girih_gpu_run_ex(&sv.v, steps, &c, &r, &o));
    state.t_current = static_cast<long>(sv.v.t_current);
    if (opts.ledger) {
        const size_t cells = static_cast<size_t>(state.grid.nx) * state.grid.ny * state.grid.nz;
        for (long t = 0; t < steps; ++t)
            for (int z = 0; z < state.grid.nz; ++z)
                for (int y = 0; y < state.grid.ny; ++y)
                    for (int x = 0; x < state.grid.nx; ++x) {
                        const unsigned n = counts[t * cells +
                                                  (static_cast<size_t>(z) * state.grid.ny + y) *
                                                      state.grid.nx + x];
                        for (unsigned k = 0; k < n; ++k) opts.ledger->record(t, z, y, x, 0);
                    }
    }
    PerfReport out;
    out.wall_seconds = r.wall_s;
    out.lups = r.lups;
    out.glups = r.wall_s > 0 ? r.lups / r.wall_s / 1e9 : 0.0;
    out.tiles = o.trace_total;
    return out;
}

}  // namespace gpu
}  // namespace girih
