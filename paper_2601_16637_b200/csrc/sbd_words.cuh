// Occupation strings as one or two 64-bit words.
//
// The product path stores a spin string as one u64 (norb <= 64, the
// reference's limit for integrals, integrals.py:67-68).  Configuration
// processing and excitation generation also take 128-bit strings (norb <= 128):
// the reference's table builder works on Python ints of any width
// (basis.py:62-103, 362-403).  These helpers give both word types the same
// interface so the radix sort (sbd_strings.cu) and the enumeration kernel
// (sbd_excite.cu) are written once.
#pragma once

#include <cstdint>

struct U128 {
    uint64_t lo, hi;
};

__host__ __device__ __forceinline__ bool operator==(U128 a, U128 b) { return a.lo == b.lo && a.hi == b.hi; }
__host__ __device__ __forceinline__ bool operator<(U128 a, U128 b) {
    return a.hi < b.hi || (a.hi == b.hi && a.lo < b.lo);
}
__host__ __device__ __forceinline__ bool operator<=(U128 a, U128 b) { return !(b < a); }

namespace words {

// mask of bits [0, b), b in [0, 64]
__host__ __device__ __forceinline__ uint64_t low_mask(int b) { return b >= 64 ? ~0ull : (1ull << b) - 1; }

__device__ __forceinline__ bool test(uint64_t w, int p) { return (w >> p) & 1; }
__device__ __forceinline__ bool test(U128 w, int p) { return p < 64 ? (w.lo >> p) & 1 : (w.hi >> (p - 64)) & 1; }

// w with bit p cleared and bit r set (p occupied, r empty)
__device__ __forceinline__ uint64_t move(uint64_t w, int p, int r) { return (w & ~(1ull << p)) | (1ull << r); }
__device__ __forceinline__ U128 move(U128 w, int p, int r) {
    if (p < 64) w.lo &= ~(1ull << p);
    else w.hi &= ~(1ull << (p - 64));
    if (r < 64) w.lo |= 1ull << r;
    else w.hi |= 1ull << (r - 64);
    return w;
}

// occupied orbitals below b, b in [0, 64] for u64 and [0, 128] for U128
__device__ __forceinline__ int popc_below(uint64_t w, int b) { return __popcll(w & low_mask(b)); }
__device__ __forceinline__ int popc_below(U128 w, int b) {
    return b <= 64 ? __popcll(w.lo & low_mask(b)) : __popcll(w.lo) + __popcll(w.hi & low_mask(b - 64));
}

// (-1)^(occupied orbitals strictly between p and r), basis.py:62-69
template <class W>
__device__ __forceinline__ int sign_between(W w, int p, int r) {
    int lo = min(p, r), hi = max(p, r);
    return ((popc_below(w, hi) - popc_below(w, lo + 1)) & 1) ? -1 : 1;
}

// 8-bit radix digit at bit offset `shift` (a multiple of 8)
__device__ __forceinline__ int digit(uint64_t w, int shift) { return (int)((w >> shift) & 0xFF); }
__device__ __forceinline__ int digit(U128 w, int shift) {
    return (int)(((shift < 64) ? (w.lo >> shift) : (w.hi >> (shift - 64))) & 0xFF);
}

__device__ __forceinline__ uint64_t ldg(const uint64_t *p) { return __ldg(p); }
__device__ __forceinline__ U128 ldg(const U128 *p) {
    ulonglong2 v = __ldg(reinterpret_cast<const ulonglong2 *>(p));
    return U128{v.x, v.y};
}

}  // namespace words
