// Host-side primitives of the B200 CF-operator engine.
//
// Mirrors the reference vocabulary (Vec3, complex fp64, the five error kinds of
// /root/reference/proj/include/ifgf/common.hpp:40-66) so the C++ operator class can rethrow
// exactly what the reference throws. Arithmetic helpers keep the reference's left-to-right
// evaluation order (dot = (x*x + y*y) + z*z) because every discrete decision of the setup
// (octree cells, cone segments, proximity) must come out bit-identical to the reference
// (SURVEY.md §7 H1, Appendix D). This translation unit family is compiled with -O2
// -ffp-contract=off and no -march, like the reference.
#pragma once

#include <cmath>
#include <complex>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <memory>
#include <utility>
#include <vector>

namespace ifgfb200 {

// Allocator that leaves elements default-initialised (no zero fill): the multi-GB setup
// tables (parent templates, parent work items) are then first touched by the parallel loops
// that fill them instead of by one thread's memset.
template <class T>
struct default_init_allocator : std::allocator<T> {
    template <class U>
    struct rebind {
        using other = default_init_allocator<U>;
    };
    using std::allocator<T>::allocator;
    template <class U, class... Args>
    void construct(U* p, Args&&... args) {
        if constexpr (sizeof...(Args) == 0)
            ::new (static_cast<void*>(p)) U;
        else
            ::new (static_cast<void*>(p)) U(std::forward<Args>(args)...);
    }
};
template <class T>
using uninit_vector = std::vector<T, default_init_allocator<T>>;

using cplx = std::complex<double>;

struct Vec3 {
    double x = 0, y = 0, z = 0;
    constexpr Vec3() = default;
    constexpr Vec3(double a, double b, double c) : x(a), y(b), z(c) {}
    Vec3 operator+(const Vec3& o) const { return {x + o.x, y + o.y, z + o.z}; }
    Vec3 operator-(const Vec3& o) const { return {x - o.x, y - o.y, z - o.z}; }
    Vec3 operator*(double s) const { return {x * s, y * s, z * s}; }
    Vec3 operator/(double s) const { return {x / s, y / s, z / s}; }
    double operator[](int i) const { return i == 0 ? x : (i == 1 ? y : z); }
};
inline Vec3 operator*(double s, const Vec3& v) { return v * s; }
inline double dot3(const Vec3& a, const Vec3& b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
inline double len2(const Vec3& v) { return dot3(v, v); }
inline double len(const Vec3& v) { return std::sqrt(len2(v)); }
inline Vec3 cross3(const Vec3& a, const Vec3& b) {
    return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}

// ---- error kinds (status codes of the C-ABI map 1:1 onto these) ----
enum Status : int {
    kOk = 0,
    kInvalidArgument = 1,
    kParseError = 2,
    kDegenerateGeometry = 3,
    kConvergenceFailure = 4,
    kInternalError = 5,
    kCudaError = 6,
    kNcclError = 7,
};

struct EngineError : std::runtime_error {
    int status;
    EngineError(int st, const std::string& m) : std::runtime_error(m), status(st) {}
};
struct InvalidArgument : EngineError {
    explicit InvalidArgument(const std::string& m) : EngineError(kInvalidArgument, m) {}
};
struct DegenerateGeometry : EngineError {
    explicit DegenerateGeometry(const std::string& m) : EngineError(kDegenerateGeometry, m) {}
};
struct ConvergenceFailure : EngineError {
    std::vector<double> history;
    ConvergenceFailure(const std::string& m, std::vector<double> h)
        : EngineError(kConvergenceFailure, m), history(std::move(h)) {}
};
struct InternalError : EngineError {
    explicit InternalError(const std::string& m) : EngineError(kInternalError, m) {}
};
struct DeviceError : EngineError {
    explicit DeviceError(const std::string& m) : EngineError(kCudaError, m) {}
};

inline constexpr double kPi = 3.141592653589793;
inline constexpr double kConeEtaC = 0.5773502691896258;  // sqrt(3)/3, kernels.hpp:7
inline constexpr double kHalfDiag = 0.8660254037844386;   // h = kHalfDiag * H, kernels.hpp:14

int worker_count(int requested);  // <= 0: all hardware threads

}  // namespace ifgfb200
