// host_compat.h -- TEST INFRASTRUCTURE: lets g++ compile the generated
// per-game rules (struct Game + lx_core.cuh + lx_rules.cuh) for the CPU test
// suite.  Device intrinsics are replaced by exact host equivalents.
#pragma once
#include <cstdint>
#include <cmath>

#define __device__
#define __forceinline__ inline
#define __host__
#define __shared__ static
struct HostThreadIdx { unsigned x = 0, y = 0, z = 0; };
static const HostThreadIdx threadIdx;

static inline int __popc(unsigned x) { return __builtin_popcount(x); }
static inline int __ffs(int x) { return __builtin_ffs(x); }
static inline unsigned __funnelshift_r(unsigned lo, unsigned hi, unsigned s) {
    s &= 31u;
    unsigned long long v = ((unsigned long long)hi << 32) | lo;
    return (unsigned)(v >> s);
}
static inline unsigned __funnelshift_l(unsigned lo, unsigned hi, unsigned s) {
    s &= 31u;
    unsigned long long v = ((unsigned long long)hi << 32) | lo;
    return (unsigned)((v << s) >> 32);
}
// strict IEEE double multiply (compiled with -ffp-contract=off)
static inline double __dmul_rn(double a, double b) { volatile double r = a * b; return r; }
static inline long long __double2ll_rz(double x) { return (long long)x; }
static inline int __double2int_rz(double x) { return (int)x; }
static inline int __clzll(long long x) { return x ? __builtin_clzll((unsigned long long)x) : 64; }
template <class T> static inline T __ldg(const T* p) { return *p; }
