// girih_gpu_cli.cpp -- the reference CLI's verify / run / tune flows (proj/tools/main.cpp) driven
// through the drop-in shim girih::gpu::run (include/girih_gpu.hpp). It is what a maintainer of the
// reference gets by swapping girih::run for girih::gpu::run; it links the reference core for
// init_state / naive_sweep (the oracle) and libgirih_gpu.so for the sweep. Built by oracle/Makefile
// into oracle/_ref/girih_gpu (only where the reference sources exist).
//
//   girih_gpu verify [--stencil S | --all] [--nx N --ny N --nz N] [--nt T] [--seed S] [--pad P]
//                    [--tb K] [--variant V] [--inject-fault]                 (main.cpp:144-186)
//   girih_gpu run    [--stencil S] [--nx ..] [--nt T] [--seed S] [--tb K] [--remap]
//                    [--out FILE] [--format csv|json] [--use-tuned FILE]   (main.cpp:260-328)
//   girih_gpu tune   [--stencil S] [--nx ..] [--max-tb K] [--out FILE] [--force]
//                                                                         (main.cpp:395-469)
//   girih_gpu model  [--stencil S | --all] [--nx ..] [--tb K] [--variant V] [--hbm GBS]
//                    [--fp64 OPS]   GPU analogue of the analytic models (models.cpp:12-84),
//                    printed beside the reference's CPU code balance / spatial balance
// Exit codes follow main.cpp:185, 524-527: 0 pass, 1 verification failure, 2 error.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "girih/engine.hpp"
#include "girih/models.hpp"
#include "girih/stencil.hpp"
#include "girih_gpu.hpp"

using namespace girih;

namespace {

constexpr int kSchemaVersion = 1;

// measured HBM copy bandwidth: --hbm, else "hbm_gbs" of MEASURED_PEAKS.json (driver-written; in
// $GIRIH_PEAKS or the working directory), else 0 = the library's own fallback
double measured_hbm_gbs(double flag) {
    if (flag > 0) return flag;
    const char* env = std::getenv("GIRIH_PEAKS");
    std::ifstream in(env ? env : "MEASURED_PEAKS.json");
    std::stringstream ss;
    ss << in.rdbuf();
    const std::string s = ss.str();
    const size_t k = s.find("\"hbm_gbs\"");
    if (k == std::string::npos) return 0.0;
    const size_t c = s.find(':', k);
    return c == std::string::npos ? 0.0 : std::atof(s.c_str() + c + 1);
}

struct Options {
    std::string cmd;
    std::string stencil = "const7pt";
    int nx = 32, ny = 32, nz = 32, pad = 0;
    long nt = 8;
    unsigned long long seed = 42;
    bool all = false, inject_fault = false, remap = false, force = false;
    int tb = 0, variant = -1, max_tb = 0;
    double hbm = 0, fp64 = 0;
    std::string out, format = "csv", use_tuned;
};

Options parse(int argc, char** argv) {
    Options o;
    if (argc < 2) throw std::invalid_argument("usage: girih_gpu verify|run|tune [options]");
    o.cmd = argv[1];
    for (int i = 2; i < argc; ++i) {
        const std::string a = argv[i];
        auto next = [&]() -> std::string {
            if (i + 1 >= argc) throw std::invalid_argument("missing value for " + a);
            return argv[++i];
        };
        if (a == "--stencil") o.stencil = next();
        else if (a == "--nx") o.nx = std::stoi(next());
        else if (a == "--ny") o.ny = std::stoi(next());
        else if (a == "--nz") o.nz = std::stoi(next());
        else if (a == "--n") o.nx = o.ny = o.nz = std::stoi(next());
        else if (a == "--pad") o.pad = std::stoi(next());
        else if (a == "--nt") o.nt = std::stol(next());
        else if (a == "--seed") o.seed = std::stoull(next());
        else if (a == "--tb") o.tb = std::stoi(next());
        else if (a == "--variant") o.variant = std::stoi(next());
        else if (a == "--max-tb") o.max_tb = std::stoi(next());
        else if (a == "--out") o.out = next();
        else if (a == "--format") o.format = next();
        else if (a == "--use-tuned") o.use_tuned = next();
        else if (a == "--hbm") o.hbm = std::stod(next());
        else if (a == "--fp64") o.fp64 = std::stod(next());
        else if (a == "--all") o.all = true;
        else if (a == "--inject-fault") o.inject_fault = true;
        else if (a == "--remap") o.remap = true;
        else if (a == "--force") o.force = true;
        else throw std::invalid_argument("unknown option " + a);
    }
    return o;
}

// SURVEY.md 8(d) BASELINE input remap, applied to a reference init_state
void apply_remap(ProblemState& s) {
    auto shift = [](Field& f, double scale) {
        for (std::size_t q = 0; q < f.size(); ++q) f.data()[q] = (f.data()[q] + 0.5) * scale;
    };
    shift(s.u, 1.0);
    shift(s.v, 1.0);
    switch (s.kind) {
    case StencilKind::Const7pt:
        s.cc[0] = (s.cc[0] + 0.5) * 0.2;
        s.cc[1] = (s.cc[1] + 0.5) * 0.2;
        break;
    case StencilKind::Var7pt:
        for (auto& c : s.coeffs) shift(c, 0.14);
        break;
    case StencilKind::Const25pt: {
        shift(s.coeffs[0], 1.0);
        double r[5];
        for (int c = 0; c < 5; ++c) r[c] = s.cc[c] + 0.5;
        const double sc = 0.99 / (r[0] + 6 * (r[1] + r[2] + r[3] + r[4]));
        for (int c = 0; c < 5; ++c) s.cc[c] = r[c] * sc;
        break;
    }
    case StencilKind::Var25pt:
        for (auto& c : s.coeffs) shift(c, 1.0 / 26);
        break;
    }
}

struct VerifyOutcome {
    bool pass = true;
    std::string field;
    int i = 0, j = 0, k = 0;
    double expected = 0, actual = 0;
};

// compare_states (main.cpp:105-127): u and v, every cell including ghosts and pad
VerifyOutcome compare_states(const ProblemState& a_, const ProblemState& b_) {
    VerifyOutcome out;
    const Field* fields[2][2] = {{&a_.u, &b_.u}, {&a_.v, &b_.v}};
    const char* names[2] = {"u", "v"};
    for (int f = 0; f < 2; ++f) {
        const Field& a = *fields[f][0];
        const Field& b = *fields[f][1];
        for (int k = 0; k < a.z(); ++k)
            for (int j = 0; j < a.y(); ++j)
                for (int i = 0; i < a.x(); ++i)
                {
                    const double x = a.at(i, j, k), y = b.at(i, j, k);
                    if (std::memcmp(&x, &y, sizeof(double)) != 0) {  // bitwise, like == on data
                        out = {false, names[f], i, j, k, x, y};
                        return out;
                    }
                }
    }
    return out;
}

std::vector<int> tbs_for(int kind) {
    std::vector<int> out;
    const int n = girih_gpu_variant_count();
    for (int i = 0; i < n; ++i) {
        girih_gpu_variant v{};
        gpu::check(girih_gpu_variant_info(i, &v));
        if (v.kind != kind) continue;
        bool seen = false;
        for (int t : out) seen |= (t == v.tb);
        if (!seen) out.push_back(v.tb);
    }
    return out;
}

int cmd_verify(const Options& o) {
    struct Case {
        StencilKind kind;
        int tb;
    };
    std::vector<Case> cases;
    if (o.all) {
        for (int s = 0; s < 4; ++s)
            for (int tb : tbs_for(s)) cases.push_back({static_cast<StencilKind>(s), tb});
    } else {
        cases.push_back({stencil_from_name(o.stencil), o.tb});
    }
    int failures = 0;
    for (const Case& c : cases) {
        const GridSpec grid{o.nx, o.ny, o.nz, o.pad};
        std::ostringstream label;
        label << traits(c.kind).name << ' ' << o.nx << 'x' << o.ny << 'x' << o.nz
              << " nt=" << o.nt << " tb=" << c.tb << " gpu";
        try {
            ProblemState oracle = init_state(c.kind, grid, o.seed);
            ProblemState tiled = init_state(c.kind, grid, o.seed);
            if (o.remap) {
                apply_remap(oracle);
                apply_remap(tiled);
            }
            naive_sweep(oracle, o.nt);
            gpu::GpuConfig cfg;
            cfg.tb = c.tb;
            cfg.variant = o.all ? -1 : o.variant;
            gpu::run(tiled, o.nt, cfg);
            if (o.inject_fault) {  // main.cpp:137-140
                const int R = tiled.radius;
                tiled.current().at(R + grid.nx / 2, R + grid.ny / 2, R + grid.nz / 2) += 1.0;
            }
            const VerifyOutcome v = compare_states(oracle, tiled);
            if (v.pass) {
                std::cout << "PASS " << label.str() << '\n';
            } else {
                ++failures;
                std::cout << "FAIL " << label.str() << " first-diff field=" << v.field << " cell=("
                          << v.i << ',' << v.j << ',' << v.k << ") oracle=" << std::hexfloat
                          << v.expected << " tiled=" << v.actual << std::defaultfloat << '\n';
            }
        } catch (const std::exception& e) {
            ++failures;
            std::cout << "ERROR " << label.str() << ": " << e.what() << '\n';
        }
    }
    return failures == 0 ? 0 : 1;
}

const char* kCsvHeader =
    "schema_version,stencil,nx,ny,nz,nt,dw,nf,tgs,variant,groups,seed,"
    "wall_seconds,glups,model_cs_bytes,model_bc,verified,"
    "mlups,hbm_gbs,code_balance,roofline_frac,tb,ngpus";

// minimal flat-JSON helpers for the tuned-config cache (one object per line)
std::string tuned_key(const Options& o) {
    std::ostringstream k;
    k << "{\"stencil\":\"" << o.stencil << "\",\"nx\":" << o.nx << ",\"ny\":" << o.ny
      << ",\"nz\":" << o.nz << ",\"machine\":\"b200\",\"ngpus\":1,\"variant\":\"zwave\"}";
    return k.str();
}

bool find_tuned(const std::string& path, const std::string& key, int* tb, int* variant,
                int* zchunks, int* chain = nullptr, int* tile_order = nullptr) {
    std::ifstream in(path);
    std::string line;
    while (std::getline(in, line)) {
        if (line.find(key) == std::string::npos) continue;
        auto field = [&](const char* name) {
            const std::string pat = std::string("\"") + name + "\":";
            const auto p = line.find(pat, line.find("\"best\""));
            return p == std::string::npos ? 0 : std::atoi(line.c_str() + p + pat.size());
        };
        *tb = field("tb");
        *variant = field("variant_index");
        *zchunks = field("zchunks");
        if (chain) *chain = field("chain");  // absent in older records: 0 = auto
        if (tile_order) *tile_order = field("tile_order");  // likewise
        return true;
    }
    return false;
}

int cmd_run(const Options& o) {
    const StencilKind kind = stencil_from_name(o.stencil);
    const GridSpec grid{o.nx, o.ny, o.nz, o.pad};
    gpu::GpuConfig cfg;
    cfg.tb = o.tb;
    cfg.variant = o.variant;
    if (!o.use_tuned.empty()) {
        if (!find_tuned(o.use_tuned, tuned_key(o), &cfg.tb, &cfg.variant, &cfg.zchunks,
                        &cfg.chain, &cfg.tile_order))
            throw std::runtime_error("no tuned configuration for this case in " + o.use_tuned +
                                     "; run `girih_gpu tune` first");
    }
    // run twice, report the faster (main.cpp:291-297); the device-resident kernel time is the
    // MLUP/s the GPU record reports, wall includes the copies
    double wall = 0, ksec = 0;
    gpu::GpuReport best;
    for (int rep = 0; rep < 2; ++rep) {
        ProblemState state = init_state(kind, grid, o.seed);
        if (o.remap) apply_remap(state);
        const gpu::GpuReport r = gpu::run(state, o.nt, cfg);
        if (rep == 0 || r.kernel_seconds < ksec) {
            ksec = r.kernel_seconds;
            best = r;
        }
        wall = rep == 0 ? r.wall_seconds : std::min(wall, r.wall_seconds);
    }
    const StencilTraits& tr = traits(kind);
    const double b1[4] = {16, 72, 32, 120};
    const long long lups = static_cast<long long>(grid.nx) * grid.ny * grid.nz * o.nt;
    const double mlups = ksec > 0 ? lups / ksec / 1e6 : 0.0;
    const double cb = best.model_bytes_per_lup;
    const double hbm_gbs = mlups * 1e6 * cb / 1e9;
    const double hbm_flag = measured_hbm_gbs(o.hbm);
    const double hbm_peak = hbm_flag > 0 ? hbm_flag : 6548.8;  // fallback: the round-1 pool
    const double roof = cb > 0 ? hbm_peak * 1e9 / cb / 1e6 : 0.0;
    std::ostringstream rec;
    const double glups = (wall > 0 && lups > 0) ? lups / wall / 1e9 : 0.0;
    if (o.format == "json") {
        rec << "{\"schema_version\":" << kSchemaVersion << ",\"stencil\":\"" << tr.name
            << "\",\"nx\":" << grid.nx << ",\"ny\":" << grid.ny << ",\"nz\":" << grid.nz
            << ",\"nt\":" << o.nt << ",\"dw\":0,\"nf\":0,\"tgs\":\"gpu\",\"variant\":\"zwave\""
            << ",\"groups\":1,\"seed\":" << o.seed << ",\"wall_seconds\":" << wall
            << ",\"glups\":" << glups << ",\"model_cs_bytes\":0,\"model_bc\":" << cb
            << ",\"verified\":\"na\",\"mlups\":" << mlups << ",\"hbm_gbs\":" << hbm_gbs
            << ",\"code_balance\":" << cb << ",\"roofline_frac\":" << (roof > 0 ? mlups / roof : 0)
            << ",\"tb\":" << best.tb_used << ",\"ngpus\":1}\n";
    } else {
        rec << kSchemaVersion << ',' << tr.name << ',' << grid.nx << ',' << grid.ny << ','
            << grid.nz << ',' << o.nt << ",0,0,gpu,zwave,1," << o.seed << ',' << wall << ','
            << glups << ",0," << cb << ",na," << mlups << ',' << hbm_gbs << ',' << cb << ','
            << (roof > 0 ? mlups / roof : 0) << ',' << best.tb_used << ",1\n";
    }
    if (o.out.empty()) {
        if (o.format != "json") std::cout << kCsvHeader << '\n';
        std::cout << rec.str();
    } else {
        std::ifstream probe(o.out);
        const bool fresh = !probe.good() || probe.peek() == std::ifstream::traits_type::eof();
        probe.close();
        std::ofstream os(o.out, std::ios::app);
        if (!os) throw std::runtime_error("cannot open output file: " + o.out);
        if (fresh && o.format != "json") os << kCsvHeader << '\n';
        os << rec.str();
    }
    return 0;
}

int cmd_tune(const Options& o) {
    const std::string out = o.out.empty() ? "girih_gpu_tuned.jsonl" : o.out;
    const std::string key = tuned_key(o);
    int tb, var, zc;
    if (!o.force && find_tuned(out, key, &tb, &var, &zc)) {
        std::cout << "cached " << key << " tb=" << tb << " variant=" << var << '\n';
        return 0;
    }
    const StencilKind kind = stencil_from_name(o.stencil);
    girih_gpu_config cfg{};
    cfg.variant = -1;
    cfg.ngpus = 1;
    cfg.exact = 1;
    void* h = nullptr;
    gpu::check(girih_gpu_open_seeded(static_cast<int>(kind), o.nx, o.ny, o.nz, o.pad, o.seed, 1,
                                     &cfg, &h));
    girih_gpu_config best{};
    double mlups = 0;
    int measured = 0;
    const int rc = girih_gpu_tune(h, o.max_tb, &best, &mlups, &measured);
    girih_gpu_close(h);
    gpu::check(rc);
    std::ofstream os(out, std::ios::app);
    os << "{\"key\":" << key << ",\"best\":{\"tb\":" << best.tb << ",\"variant_index\":"
       << best.variant << ",\"zchunks\":" << best.zchunks << ",\"chain\":" << best.chain
       << ",\"tile_order\":" << best.tile_order << ",\"mlups\":" << mlups
       << ",\"measured\":" << measured << "}}\n";
    std::cout << "tuned " << key << " tb=" << best.tb << " variant=" << best.variant
              << " zchunks=" << best.zchunks << " chain=" << best.chain
              << " tile_order=" << best.tile_order << " mlups=" << mlups
              << '\n';
    return 0;
}

// GPU model per fused depth next to the reference's CPU models (code_balance Eq. 4 at the
// default diamond width, spatial_balance), one line per (stencil, tb)
int cmd_model(const Options& o) {
    std::vector<std::string> names = {o.stencil};
    if (o.all) names = {"const7pt", "var7pt", "const25pt", "var25pt"};
    std::cout << "stencil,tb,variant,tile,out_tile,threads,smem_bytes,ctas_per_sm,zchunks,"
                 "redundancy,gpu_code_balance,gpu_code_balance_no_l2,hbm_mlups,fp64_mlups,"
                 "roofline_mlups,cpu_code_balance_dw,cpu_spatial_balance\n";
    for (const auto& name : names) {
        const StencilKind kind = stencil_from_name(name);
        const StencilTraits tr = traits(kind);
        const int dw = tr.radius == 1 ? 8 : 16;  // main.cpp:67 defaults
        std::vector<int> tbs = o.tb > 0 ? std::vector<int>{o.tb} : tbs_for(int(kind));
        for (int tb : tbs) {
            girih_gpu_model_out m{};
            gpu::check(girih_gpu_model(int(kind), o.nx, o.ny, o.nz, tb, o.tb > 0 ? o.variant : -1,
                                       measured_hbm_gbs(o.hbm), o.fp64, &m));
            std::printf("%s,%d,%d,%dx%d,%dx%d,%d,%d,%d,%d,%.4f,%.3f,%.3f,%.0f,%.0f,%.0f,%.3f,%.1f\n",
                        name.c_str(), m.tb, m.variant, m.lx, m.ly, m.ox, m.oy, m.threads,
                        m.smem_bytes, m.ctas_per_sm, m.zchunks, m.redundancy, m.code_balance,
                        m.code_balance_no_l2, m.hbm_mlups, m.fp64_mlups, m.roofline_mlups,
                        code_balance(dw, tr.domain_streams, tr.radius), spatial_balance(kind));
        }
    }
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    try {
        const Options o = parse(argc, argv);
        if (o.cmd == "verify") return cmd_verify(o);
        if (o.cmd == "run") return cmd_run(o);
        if (o.cmd == "tune") return cmd_tune(o);
        if (o.cmd == "model") return cmd_model(o);
        throw std::invalid_argument("unknown subcommand " + o.cmd);
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << '\n';
        return 2;
    }
}
