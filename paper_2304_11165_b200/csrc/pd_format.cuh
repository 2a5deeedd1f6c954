// Exact "%.*g" formatting of IEEE doubles on the device (and host), the text
// the reference's format_scalar produces (scalar_text.hpp:20-28: "%.17g" for
// double, "%.9g" for float widened to double, "nan" for every NaN). glibc
// prints the exactly rounded decimal expansion (round-half-even on the exact
// binary value); so does this: the P significant digits come from an exact
// integer evaluation of |v|·10^p (128-bit for the common exponent range, a
// small bignum otherwise) and the rounding compares the exact remainder with
// one half. Verified against snprintf on random bit patterns and edge sets
// (tests/test_vtk.py).
#pragma once

#include <cstdint>
#include <cstring>

#ifdef __CUDACC__
#define PD_HD __host__ __device__ __forceinline__
#define PD_HDN __host__ __device__ __noinline__
#else
#define PD_HD inline
#define PD_HDN inline
#endif

namespace pdb {
namespace fmt {

constexpr int kMaxText = 25;  // longest "%.17g" text + '\n' ("-1.2345678901234567e-308\n")

struct Big {
    static constexpr int kLimbs = 40;  // 1280 bits: m·5^340 and (5^292·2^q)·2^64 fit
    uint32_t w[kLimbs];
    int n;  // limbs in use (w[n-1] != 0 unless n == 0)
};

PD_HD void big_set(Big& b, uint64_t v) {
    b.w[0] = (uint32_t)v;
    b.w[1] = (uint32_t)(v >> 32);
    b.n = b.w[1] ? 2 : (b.w[0] ? 1 : 0);
}

PD_HD bool big_mul(Big& b, uint32_t m) {
    uint64_t carry = 0;
    for (int i = 0; i < b.n; ++i) {
        const uint64_t t = (uint64_t)b.w[i] * m + carry;
        b.w[i] = (uint32_t)t;
        carry = t >> 32;
    }
    if (carry) {
        if (b.n == Big::kLimbs) return false;
        b.w[b.n++] = (uint32_t)carry;
    }
    return true;
}

PD_HD bool big_mul_pow5(Big& b, int p) {
    for (; p >= 13; p -= 13)
        if (!big_mul(b, 1220703125u)) return false;  // 5^13
    uint32_t r = 1;
    for (; p > 0; --p) r *= 5u;
    return big_mul(b, r);
}

PD_HD bool big_shl(Big& b, int s) {
    if (b.n == 0 || s == 0) return true;
    const int limbs = s >> 5, bits = s & 31;
    int nn = b.n + limbs + 1;
    if (nn > Big::kLimbs) {
        // only legal when the top limb does not spill
        if (nn - 1 > Big::kLimbs) return false;
        if (bits && (b.w[b.n - 1] >> (32 - bits))) return false;
        nn = Big::kLimbs;
    }
    for (int i = nn - 1; i >= 0; --i) {
        const int src = i - limbs;
        uint32_t hi = (src >= 0 && src < b.n) ? b.w[src] : 0u;
        uint32_t lo = (src - 1 >= 0 && src - 1 < b.n) ? b.w[src - 1] : 0u;
        b.w[i] = bits ? (hi << bits) | (lo >> (32 - bits)) : hi;
    }
    b.n = nn;
    while (b.n > 0 && b.w[b.n - 1] == 0) --b.n;
    return true;
}

PD_HD void big_shr1(Big& b) {
    for (int i = 0; i < b.n; ++i) b.w[i] = (b.w[i] >> 1) | (i + 1 < b.n ? (b.w[i + 1] << 31) : 0u);
    while (b.n > 0 && b.w[b.n - 1] == 0) --b.n;
}

PD_HD int big_cmp(const Big& a, const Big& b) {
    if (a.n != b.n) return a.n < b.n ? -1 : 1;
    for (int i = a.n - 1; i >= 0; --i)
        if (a.w[i] != b.w[i]) return a.w[i] < b.w[i] ? -1 : 1;
    return 0;
}

PD_HD void big_sub(Big& a, const Big& b) {  // a >= b
    int64_t borrow = 0;
    for (int i = 0; i < a.n; ++i) {
        int64_t t = (int64_t)a.w[i] - (i < b.n ? (int64_t)b.w[i] : 0) - borrow;
        borrow = t < 0;
        a.w[i] = (uint32_t)(t + (borrow << 32));
    }
    while (a.n > 0 && a.w[a.n - 1] == 0) --a.n;
}

// bit s of b
PD_HD uint32_t big_bit(const Big& b, int s) {
    const int l = s >> 5;
    return l < b.n ? (b.w[l] >> (s & 31)) & 1u : 0u;
}

// Scaled value: N = floor(m·2^e·10^p) and the sign of (fraction − 1/2).
// ok = false when N does not fit 64 bits (the caller raises the exponent).
struct Scaled {
    uint64_t N;
    int half;  // -1 below one half, 0 exactly one half, +1 above
    bool ok;
};

// Exact path for every (m, e, p) a double can produce.
PD_HDN Scaled scaled_big(uint64_t m, int e, int p) {
    Scaled r{0, -1, true};
    Big A;
    big_set(A, m);
    if (p >= 0) {
        if (!big_mul_pow5(A, p)) return Scaled{0, 0, false};
        const int sh = e + p;
        if (sh >= 0) {
            if (!big_shl(A, sh) || A.n > 2) return Scaled{0, 0, false};
            r.N = (uint64_t)A.w[0] | (A.n > 1 ? (uint64_t)A.w[1] << 32 : 0ull);
            return r;
        }
        const int s = -sh;
        // N = A >> s must fit 64 bits
        if ((A.n * 32) > s + 64) {
            for (int k = s + 64; k < A.n * 32; ++k)
                if (big_bit(A, k)) return Scaled{0, 0, false};
        }
        uint64_t N = 0;
        for (int k = 63; k >= 0; --k) N = (N << 1) | big_bit(A, s + k);
        r.N = N;
        if (!big_bit(A, s - 1)) {
            r.half = -1;
        } else {
            bool low = false;
            for (int k = 0; k < s - 1 && !low; ++k) low = big_bit(A, k) != 0;
            r.half = low ? 1 : 0;
        }
        return r;
    }
    const int q = -p;
    Big B;
    big_set(B, 1);
    if (!big_mul_pow5(B, q)) return Scaled{0, 0, false};
    if (e >= q) {
        if (!big_shl(A, e - q)) return Scaled{0, 0, false};
    } else {
        if (!big_shl(B, q - e)) return Scaled{0, 0, false};
    }
    Big Bk = B;  // B·2^64 must exceed A
    if (!big_shl(Bk, 64)) return Scaled{0, 0, false};
    if (big_cmp(A, Bk) >= 0) return Scaled{0, 0, false};
    big_shr1(Bk);  // B·2^63
    uint64_t N = 0;
    for (int k = 63; k >= 0; --k) {
        if (big_cmp(A, Bk) >= 0) {
            big_sub(A, Bk);
            N |= 1ull << k;
        }
        big_shr1(Bk);
    }
    r.N = N;
    if (!big_shl(A, 1)) return Scaled{0, 0, false};
    r.half = big_cmp(A, B);
    return r;
}

// 128-bit path: 0 <= p <= 32 (|v| in about [1e-16, 1e17) for P = 17).
PD_HD Scaled scaled(uint64_t m, int e, int p) {
    if (p < 0 || p > 32) return scaled_big(m, e, p);
    unsigned __int128 A = m;
    const int p1 = p < 27 ? p : 27;
    uint64_t f = 1;
    for (int i = 0; i < p1; ++i) f *= 5u;
    A *= f;
    for (int i = p1; i < p; ++i) A *= 5u;  // m·5^32 < 2^128
    const int sh = e + p;
    Scaled r{0, -1, true};
    if (sh >= 0) {
        if (sh >= 64 || (A >> (64 - sh)) != 0) return Scaled{0, 0, false};
        r.N = (uint64_t)(A << sh);
        return r;
    }
    const int s = -sh;
    if (s >= 128) return Scaled{0, -1, true};  // N = 0: exponent estimate too high
    const unsigned __int128 Nq = A >> s;
    if ((Nq >> 64) != 0) return Scaled{0, 0, false};
    r.N = (uint64_t)Nq;
    const unsigned __int128 R = A - (Nq << s);
    const unsigned __int128 h = (unsigned __int128)1 << (s - 1);
    r.half = R > h ? 1 : (R == h ? 0 : -1);
    return r;
}

PD_HD int clz64(uint64_t x) {
#ifdef __CUDA_ARCH__
    return __clzll((long long)x);
#else
    return __builtin_clzll(x);
#endif
}

PD_HD uint64_t pow10u(int k) {
    uint64_t r = 1;
    for (int i = 0; i < k; ++i) r *= 10u;
    return r;
}

// floor(log10(2^x)) for |x| <= 1100 (exact for that range)
PD_HD int floor_log10_pow2(int x) { return (int)(((int64_t)x * 78913) >> 18); }

// "%.{P}g" of v into out (no terminator); returns the length. NaN prints
// "nan" (format_scalar's rule, any sign or payload).
PD_HDN int format_g(double v, int P, char* out) {
    uint64_t bits;
    std::memcpy(&bits, &v, 8);
    int n = 0;
    const bool neg = bits >> 63;
    const int be = (int)((bits >> 52) & 0x7FF);
    const uint64_t frac = bits & ((1ull << 52) - 1);
    if (be == 0x7FF) {
        if (frac) {
            out[0] = 'n', out[1] = 'a', out[2] = 'n';
            return 3;
        }
        if (neg) out[n++] = '-';
        out[n++] = 'i', out[n++] = 'n', out[n++] = 'f';
        return n;
    }
    if (neg) out[n++] = '-';
    if (be == 0 && frac == 0) {
        out[n++] = '0';
        return n;
    }
    uint64_t m;
    int e;
    if (be == 0) {
        m = frac;
        e = -1074;
    } else {
        m = frac | (1ull << 52);
        e = be - 1075;
    }
    // decimal exponent estimate from the binary one (within one of the truth)
    const int msb = 63 - clz64(m);
    int X = floor_log10_pow2(e + msb);
    const uint64_t lo = pow10u(P - 1), hi = pow10u(P);
    Scaled s{};
    for (int guard = 0; guard < 6; ++guard) {
        s = scaled(m, e, P - 1 - X);
        if (!s.ok || s.N >= hi) {
            ++X;
            continue;
        }
        if (s.N < lo) {
            --X;
            continue;
        }
        break;
    }
    uint64_t N = s.N;
    if (s.half > 0 || (s.half == 0 && (N & 1u))) ++N;
    if (N == hi) {
        N = lo;
        ++X;
    }
    char d[20];
    for (int i = P - 1; i >= 0; --i) {
        d[i] = (char)('0' + (int)(N % 10u));
        N /= 10u;
    }
    if (X < P && X >= -4) {
        // fixed notation, P-1-X digits after the point, trailing zeros dropped
        if (X >= 0) {
            for (int i = 0; i <= X; ++i) out[n++] = d[i];
            int last = P - 1;
            while (last > X && d[last] == '0') --last;
            if (last > X) {
                out[n++] = '.';
                for (int i = X + 1; i <= last; ++i) out[n++] = d[i];
            }
        } else {
            int last = P - 1;
            while (last > 0 && d[last] == '0') --last;
            out[n++] = '0';
            out[n++] = '.';
            for (int i = 0; i < -X - 1; ++i) out[n++] = '0';
            for (int i = 0; i <= last; ++i) out[n++] = d[i];
        }
        return n;
    }
    out[n++] = d[0];
    int last = P - 1;
    while (last > 0 && d[last] == '0') --last;
    if (last > 0) {
        out[n++] = '.';
        for (int i = 1; i <= last; ++i) out[n++] = d[i];
    }
    out[n++] = 'e';
    int x = X;
    if (x < 0) {
        out[n++] = '-';
        x = -x;
    } else {
        out[n++] = '+';
    }
    if (x >= 100) {
        out[n++] = (char)('0' + x / 100);
        x %= 100;
        out[n++] = (char)('0' + x / 10);
        out[n++] = (char)('0' + x % 10);
    } else {
        out[n++] = (char)('0' + x / 10);
        out[n++] = (char)('0' + x % 10);
    }
    return n;
}

// decimal int32 ("%d")
PD_HD int format_int(int32_t v, char* out) {
    int n = 0;
    uint32_t u = (uint32_t)v;
    if (v < 0) {
        out[n++] = '-';
        u = 0u - u;
    }
    char t[10];
    int k = 0;
    do {
        t[k++] = (char)('0' + u % 10u);
        u /= 10u;
    } while (u);
    while (k) out[n++] = t[--k];
    return n;
}

}  // namespace fmt
}  // namespace pdb
