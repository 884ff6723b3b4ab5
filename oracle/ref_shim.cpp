// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" wrapper around the UNMODIFIED reference core library
// (/root/reference/proj/src/*.cpp, compiled in place by oracle/Makefile with the
// reference's own Release flags, proj/CMakeLists.txt:15-25). It lets the Python
// tests, the golden-fixture generator and bench.py's reference arm drive the
// reference's own init_state / naive_sweep / run / interior_checksum.
// No reference source is copied into this repository; this file only includes
// the reference's public headers.
#include "girih/engine.hpp"
#include "girih/geometry.hpp"
#include "girih/stencil.hpp"

#include <cstdint>
#include <stdexcept>
#include <cstring>
#include <exception>
#include <string>
#include <thread>

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return -1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -2;
    }
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

unsigned ref_hardware_concurrency() { return std::thread::hardware_concurrency(); }

// girih::init_state (proj/src/stencil.cpp:58-85)
void* ref_state_new(int kind, int nx, int ny, int nz, int pad_x, unsigned long long seed) {
    girih::ProblemState* out = nullptr;
    const int rc = guarded([&] {
        out = new girih::ProblemState(girih::init_state(static_cast<girih::StencilKind>(kind),
                                                        girih::GridSpec{nx, ny, nz, pad_x}, seed));
    });
    return rc == 0 ? out : nullptr;
}

// A ProblemState with the reference's allocation (init_state's shapes, stencil.cpp:70-80) but
// zero-filled fields, for callers that fill the arrays themselves (the bench's CPU baseline
// fills them with the oracle's multi-threaded copy of the same generator).
void* ref_state_alloc(int kind, int nx, int ny, int nz, int pad_x) {
    girih::ProblemState* out = nullptr;
    const int rc = guarded([&] {
        const girih::StencilKind k = static_cast<girih::StencilKind>(kind);
        const girih::StencilTraits& tr = girih::traits(k);
        const girih::GridSpec grid{nx, ny, nz, pad_x};
        const int R = tr.radius;
        if (nx < 2 * R + 1 || ny < 2 * R + 1 || nz < 2 * R + 1 || pad_x < 0)
            throw std::invalid_argument("grid extent below 2R+1 for stencil radius");
        auto* s = new girih::ProblemState();
        s->kind = k;
        s->grid = grid;
        s->radius = R;
        const int X = grid.x_alloc(R), Y = ny + 2 * R, Z = nz + 2 * R;
        s->u = girih::Field(X, Y, Z);
        s->v = girih::Field(X, Y, Z);
        for (int c = 0; c < tr.coeff_arrays; ++c) s->coeffs.emplace_back(X, Y, Z);
        out = s;
    });
    return rc == 0 ? out : nullptr;
}

void ref_state_free(void* s) { delete static_cast<girih::ProblemState*>(s); }

int ref_state_dims(void* s, int* X, int* Y, int* Z, int* R, int* ncoeff) {
    auto* st = static_cast<girih::ProblemState*>(s);
    *X = st->u.x();
    *Y = st->u.y();
    *Z = st->u.z();
    *R = st->radius;
    *ncoeff = static_cast<int>(st->coeffs.size());
    return 0;
}

// which: 0 = u, 1 = v, 2 + c = coefficient field c
double* ref_state_field(void* s, int which) {
    auto* st = static_cast<girih::ProblemState*>(s);
    if (which == 0) return st->u.data();
    if (which == 1) return st->v.data();
    const int c = which - 2;
    if (c < 0 || c >= static_cast<int>(st->coeffs.size())) return nullptr;
    return st->coeffs[c].data();
}

double* ref_state_cc(void* s) { return static_cast<girih::ProblemState*>(s)->cc.data(); }

long ref_state_t(void* s) { return static_cast<girih::ProblemState*>(s)->t_current; }

void ref_state_set_t(void* s, long t) { static_cast<girih::ProblemState*>(s)->t_current = t; }

// girih::naive_sweep (proj/src/stencil.cpp:115-127)
int ref_naive_sweep(void* s, long steps) {
    return guarded([&] { girih::naive_sweep(*static_cast<girih::ProblemState*>(s), steps); });
}

// girih::run (proj/src/engine.cpp:332-418); variant 0 = relaxed, 1 = fed
int ref_run(void* s, long steps, int dw, int nf, int tx, int ty, int tz, int variant, int groups,
            double* wall_s, double* glups) {
    return guarded([&] {
        const girih::PerfReport r =
            girih::run(*static_cast<girih::ProblemState*>(s), steps, dw, girih::WavefrontSpec{nf, 0},
                       girih::ThreadGroupShape{tx, ty, tz, 1},
                       variant == 0 ? girih::WavefrontVariant::RelaxedPipelined
                                    : girih::WavefrontVariant::FixedExecutionToData,
                       groups);
        if (wall_s) *wall_s = r.wall_seconds;
        if (glups) *glups = r.glups;
    });
}

// girih::interior_checksum (proj/src/stencil.cpp:129-146)
unsigned long long ref_checksum(void* s) {
    return girih::interior_checksum(*static_cast<girih::ProblemState*>(s));
}

// girih::apply_point (proj/src/stencil.cpp:99-113)
double ref_apply_point(void* s, int i, int j, int k) {
    return girih::apply_point(*static_cast<girih::ProblemState*>(s), i, j, k);
}

}  // extern "C"
