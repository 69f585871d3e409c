/* Minimal SHA-256 (FIPS 180-4) for lower-triangle digests.
 *
 * TEST INFRASTRUCTURE ONLY (oracle/): used by the reference driver and the
 * C oracle to fingerprint Low(C) as little-endian uint64, row by row
 * (i = 0..n-1, j = 0..i).  The GPU side hashes the same byte stream with
 * Python's hashlib, so digests from either side are directly comparable.
 */
#ifndef FSYRK_ORACLE_SHA256_H
#define FSYRK_ORACLE_SHA256_H

#include <stddef.h>
#include <stdint.h>
#include <string.h>

typedef struct {
    uint32_t h[8];
    uint64_t nbytes;
    uint8_t buf[64];
    size_t nbuf;
} sha256_ctx;

static const uint32_t sha256_k[64] = {
    0x428a2f98u, 0x71374491u, 0xb5c0fbcfu, 0xe9b5dba5u, 0x3956c25bu, 0x59f111f1u, 0x923f82a4u,
    0xab1c5ed5u, 0xd807aa98u, 0x12835b01u, 0x243185beu, 0x550c7dc3u, 0x72be5d74u, 0x80deb1feu,
    0x9bdc06a7u, 0xc19bf174u, 0xe49b69c1u, 0xefbe4786u, 0x0fc19dc6u, 0x240ca1ccu, 0x2de92c6fu,
    0x4a7484aau, 0x5cb0a9dcu, 0x76f988dau, 0x983e5152u, 0xa831c66du, 0xb00327c8u, 0xbf597fc7u,
    0xc6e00bf3u, 0xd5a79147u, 0x06ca6351u, 0x14292967u, 0x27b70a85u, 0x2e1b2138u, 0x4d2c6dfcu,
    0x53380d13u, 0x650a7354u, 0x766a0abbu, 0x81c2c92eu, 0x92722c85u, 0xa2bfe8a1u, 0xa81a664bu,
    0xc24b8b70u, 0xc76c51a3u, 0xd192e819u, 0xd6990624u, 0xf40e3585u, 0x106aa070u, 0x19a4c116u,
    0x1e376c08u, 0x2748774cu, 0x34b0bcb5u, 0x391c0cb3u, 0x4ed8aa4au, 0x5b9cca4fu, 0x682e6ff3u,
    0x748f82eeu, 0x78a5636fu, 0x84c87814u, 0x8cc70208u, 0x90befffau, 0xa4506cebu, 0xbef9a3f7u,
    0xc67178f2u};

static inline uint32_t sha256_ror(uint32_t x, int r) { return (x >> r) | (x << (32 - r)); }

static inline void sha256_block(sha256_ctx* c, const uint8_t* p) {
    uint32_t w[64];
    for (int i = 0; i < 16; ++i)
        w[i] = (uint32_t)p[4 * i] << 24 | (uint32_t)p[4 * i + 1] << 16 | (uint32_t)p[4 * i + 2] << 8 |
               (uint32_t)p[4 * i + 3];
    for (int i = 16; i < 64; ++i) {
        uint32_t s0 = sha256_ror(w[i - 15], 7) ^ sha256_ror(w[i - 15], 18) ^ (w[i - 15] >> 3);
        uint32_t s1 = sha256_ror(w[i - 2], 17) ^ sha256_ror(w[i - 2], 19) ^ (w[i - 2] >> 10);
        w[i] = w[i - 16] + s0 + w[i - 7] + s1;
    }
    uint32_t a = c->h[0], b = c->h[1], cc = c->h[2], d = c->h[3];
    uint32_t e = c->h[4], f = c->h[5], g = c->h[6], h = c->h[7];
    for (int i = 0; i < 64; ++i) {
        uint32_t s1 = sha256_ror(e, 6) ^ sha256_ror(e, 11) ^ sha256_ror(e, 25);
        uint32_t ch = (e & f) ^ (~e & g);
        uint32_t t1 = h + s1 + ch + sha256_k[i] + w[i];
        uint32_t s0 = sha256_ror(a, 2) ^ sha256_ror(a, 13) ^ sha256_ror(a, 22);
        uint32_t mj = (a & b) ^ (a & cc) ^ (b & cc);
        uint32_t t2 = s0 + mj;
        h = g; g = f; f = e; e = d + t1;
        d = cc; cc = b; b = a; a = t1 + t2;
    }
    c->h[0] += a; c->h[1] += b; c->h[2] += cc; c->h[3] += d;
    c->h[4] += e; c->h[5] += f; c->h[6] += g; c->h[7] += h;
}

static inline void sha256_init(sha256_ctx* c) {
    static const uint32_t iv[8] = {0x6a09e667u, 0xbb67ae85u, 0x3c6ef372u, 0xa54ff53au,
                                   0x510e527fu, 0x9b05688cu, 0x1f83d9abu, 0x5be0cd19u};
    memcpy(c->h, iv, sizeof(iv));
    c->nbytes = 0;
    c->nbuf = 0;
}

static inline void sha256_update(sha256_ctx* c, const void* data, size_t len) {
    const uint8_t* p = (const uint8_t*)data;
    c->nbytes += len;
    if (c->nbuf) {
        while (len && c->nbuf < 64) { c->buf[c->nbuf++] = *p++; --len; }
        if (c->nbuf == 64) { sha256_block(c, c->buf); c->nbuf = 0; }
    }
    while (len >= 64) { sha256_block(c, p); p += 64; len -= 64; }
    while (len) { c->buf[c->nbuf++] = *p++; --len; }
}

static inline void sha256_final(sha256_ctx* c, char hex[65]) {
    uint64_t bits = c->nbytes * 8;
    uint8_t pad = 0x80;
    sha256_update(c, &pad, 1);
    uint8_t zero = 0;
    while (c->nbuf != 56) sha256_update(c, &zero, 1);
    uint8_t len[8];
    for (int i = 0; i < 8; ++i) len[i] = (uint8_t)(bits >> (56 - 8 * i));
    sha256_update(c, len, 8);
    static const char* dig = "0123456789abcdef";
    for (int i = 0; i < 8; ++i)
        for (int j = 0; j < 4; ++j) {
            uint8_t byte = (uint8_t)(c->h[i] >> (24 - 8 * j));
            hex[8 * i + 2 * j] = dig[byte >> 4];
            hex[8 * i + 2 * j + 1] = dig[byte & 15];
        }
    hex[64] = 0;
}

/* Digest of Low(C) for a row-major uint64 matrix with the given stride. */
static inline void lower_digest_u64(const uint64_t* c, size_t n, size_t ldc, char hex[65]) {
    sha256_ctx ctx;
    sha256_init(&ctx);
    for (size_t i = 0; i < n; ++i) sha256_update(&ctx, c + i * ldc, (i + 1) * sizeof(uint64_t));
    sha256_final(&ctx, hex);
}

#endif
