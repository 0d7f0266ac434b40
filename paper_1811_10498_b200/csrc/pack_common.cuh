// ASCII -> 2-bit code helpers shared by the pack kernel (pack.cu) and the text-input match kernel
// (match.cu, TXT mode), which packs its own slices in shared memory.  pack16 is also compiled for
// the host by tests/test_pack_arith.py (exhaustive check of the byte arithmetic).
#pragma once
#include <cstdint>

#if defined(__CUDACC__)
#define PFAC_HD __host__ __device__ __forceinline__
#else
#define PFAC_HD inline
#endif

namespace pfac {

PFAC_HD uint32_t umulhi32(uint32_t a, uint32_t b) {
#if defined(__CUDA_ARCH__)
    return __umulhi(a, b);
#else
    return (uint32_t)(((uint64_t)a * b) >> 32);
#endif
}
// x >> k (1 <= k <= 31) as IMAD.HI on the FMA pipe: the integer ALU pipe (LOP3/SHF/PRMT) is the busier
// of the two half-rate pipes in these kernels (ncu: math_pipe_throttle), so shifts move across.
#ifndef PFAC_FMA_SHR
#define PFAC_FMA_SHR 1
#endif
#ifndef PFAC_FMA_PACK
#define PFAC_FMA_PACK 0  // measured: pack16's shifts stay on the ALU pipe (pack kernel and text kernel)
#endif
PFAC_HD uint32_t shr_fma(uint32_t x, uint32_t k) {
#if defined(__CUDA_ARCH__) && PFAC_FMA_SHR
    uint32_t r;
    asm("mul.hi.u32 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(1u << (32 - k)));
    return r;
#else
    return x >> k;
#endif
}
PFAC_HD uint32_t byte_perm(uint32_t a, uint32_t b, uint32_t s) {  // PRMT, selectors < 8 only
#if defined(__CUDA_ARCH__)
    return __byte_perm(a, b, s);
#else
    const uint64_t v = ((uint64_t)b << 32) | a;
    uint32_t r = 0;
    for (int i = 0; i < 4; ++i) r |= (uint32_t)((v >> (8 * ((s >> (4 * i)) & 7))) & 0xFF) << (8 * i);
    return r;
#endif
}

// ASCII -> 2-bit codes (A0 C1 G2 T3), 16 bases per uint32, base j at bits 2(j mod 16).
// Four bytes at a time (one 32-bit word x), every step byte-local (no carry crosses a byte):
//   code*2 = (x ^ x>>1) & 6: bit 1 = x1^x2, bit 2 = x2^x3 -- A0 C1 G2 T3 for both cases (x3 = 0 in
//     every ACGTacgt byte); codes of other bytes are unspecified (include/pfac.h);
//   gather: umulhi(code*2, 2^31+2^25+2^19+2^13) has c0 | c1<<2 | c2<<4 | c3<<6 in its low byte
//     (the other partial products fall in bits >= 8 or, disjoint and carry-free, in the low word);
//   validity residue: ((x|0x20) ^ 'a') is 0, 2, 6 for a, c, g outside bits 1-2 and 0x15 for t, and
//     t is the only valid byte whose code bits (x>>1)&3 read 2 (e, u, ... also do: they fail the
//     0x11 term); so a byte is in ACGTacgt iff its byte of ((x|0x20) ^ 'a' ^ 0x11*isT) & 0xF9 is 0.
// pack4f returns the gathered byte in bits 0-7 (garbage above) and ORs the residue into acc.
PFAC_HD uint32_t pack4f(uint32_t x, uint32_t &acc) {
#if PFAC_FMA_PACK
    const uint32_t s1 = shr_fma(x, 1);
    const uint32_t is_t = shr_fma(x, 2) & ~s1 & 0x01010101u;
#else
    const uint32_t s1 = x >> 1;
    const uint32_t is_t = (x >> 2) & ~s1 & 0x01010101u;
#endif
    const uint32_t c2 = (x ^ s1) & 0x06060606u;
    acc |= ((x | 0x20202020u) ^ 0x61616161u) ^ (is_t * 0x11u);
    return umulhi32(c2, 0x82082000u);
}
// 16 bytes -> one packed word; acc & kBadMask != 0 iff one of the bytes is outside ACGTacgt.
constexpr uint32_t kBadMask = 0xF9F9F9F9u;
// pack4f with the residue returned instead of accumulated (the text kernel keeps the four residues
// of a word to derive its exact barrier bits when one is nonzero).
PFAC_HD uint32_t pack4r(uint32_t x, uint32_t &res) {
    res = 0;
    return pack4f(x, res);
}
// 4-bit mask (bit b = byte b) of the bytes whose residue is nonzero in its kBadMask bits: bit 7 of
// ((y & 0x7F) + 0x7F) | y is set iff the byte y is nonzero (no carry leaves a byte), and one
// multiply gathers the four bit-7s (partial products land on distinct bits, only the four wanted
// ones in 24..27).
PFAC_HD uint32_t badmask4(uint32_t r) {
    const uint32_t y = r & kBadMask;
    const uint32_t h = (((y & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | y) & 0x80808080u;
    return ((h >> 7) * 0x01020408u) >> 24;
}
PFAC_HD uint32_t badmask16(uint32_t r0, uint32_t r1, uint32_t r2, uint32_t r3) {
    return badmask4(r0) | (badmask4(r1) << 4) | (badmask4(r2) << 8) | (badmask4(r3) << 12);
}
PFAC_HD uint32_t pack16(uint32_t x, uint32_t y, uint32_t z, uint32_t w, uint32_t &acc) {
    const uint32_t h0 = pack4f(x, acc), h1 = pack4f(y, acc), h2 = pack4f(z, acc), h3 = pack4f(w, acc);
    return byte_perm(byte_perm(h0, h1, 0x0040u), byte_perm(h2, h3, 0x0040u), 0x5410u);
}

#if defined(__CUDACC__)
// Exact per-byte validity (the rare path: words that hold a barrier).  expect4: "acgt"[t] with
// t = (x >> 1) & 3 (A0 C1 T2 G3) built by one PRMT, XORed with the case-folded byte.
__device__ __forceinline__ uint32_t expect4(uint32_t x, uint32_t t) {  // nonzero bytes = bad bytes
    uint32_t sel = t | (t >> 4);                    // nibble selectors at bits 0, 4, 16, 20
    sel = (sel & 0xFFu) | ((sel >> 8) & 0xFF00u);   // -> bits 0, 4, 8, 12
    return __byte_perm(0x67746361u, 0u, sel) ^ (x | 0x20202020u);  // "acgt"[t] vs the byte
}
// 4-bit mask of the bad bytes of x (bit b = byte b): the 0x01 bits of the nonzero-byte mask gathered
// by one multiply (partial products land on distinct bits, none in 24..27 but the wanted four).
__device__ __forceinline__ uint32_t bad4(uint32_t x) {
    const uint32_t m = __vcmpne4(expect4(x, (x >> 1) & 0x03030303u), 0u) & 0x01010101u;
    return (m * 0x01020408u) >> 24;
}
__device__ __forceinline__ uint32_t bad16(uint4 v) {
    return bad4(v.x) | (bad4(v.y) << 4) | (bad4(v.z) << 8) | (bad4(v.w) << 12);
}
#endif
PFAC_HD bool valid_byte(uint8_t b) {
    const uint8_t y = b | 0x20;
    return y == 'a' || y == 'c' || y == 'g' || y == 't';
}

}  // namespace pfac
