/*
 * oracle/amaze_oracle.c -- TEST INFRASTRUCTURE ONLY (the parity checker and the
 * CPU baseline).  Nothing in the product package may link, load or call this file;
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg use it.
 *
 * A plain-C restatement of the random-stream arithmetic the reference relies on,
 * plus the level generator and the ACCEL mutator built on it.
 *
 *   reference call sites (read-only tree /root/reference/pkg/src/autocurricula):
 *     rng.py:43-50            RngStream.generator() = Generator(Philox(SeedSequence(entropy, spawn_key)))
 *     amaze/generator.py:36-52  sample_random_level
 *     amaze/generator.py:55-84  mutate_level
 *
 *   third-party algorithm restated: numpy.random (unpinned in the reference,
 *   pkg/pyproject.toml:11 "numpy>=1.24"; pinned here to the behaviour of numpy
 *   2.3.5, against which tests/test_oracle_rng.py checks this file):
 *     SeedSequence pool mixing + generate_state (numpy/random/bit_generator.pyx),
 *     Philox4x64-10 with a 4-word output buffer and a pending upper 32-bit half
 *     (numpy/random/src/philox), Generator.integers for ranges < 2^32 (32-bit
 *     Lemire rejection), Generator.random (53-bit), Generator.permutation
 *     (Fisher-Yates with masked rejection random_interval).
 *
 * Level layout used by every implementation in this repo (oracle, CUDA, Python):
 *   interior cell (r, c), 1 <= r <= H-2, 1 <= c <= W-2, has bit index
 *   (r-1)*(W-2) + (c-1) in a 128-bit little-endian mask words[4].
 */
#include <stdint.h>
#include <string.h>

/* ----------------------------------------------------------------------------
 * SeedSequence
 * ------------------------------------------------------------------------- */
#define SS_INIT_A 0x43b0d7e5u
#define SS_MULT_A 0x931e8875u
#define SS_INIT_B 0x8b51f9ddu
#define SS_MULT_B 0x58f38dedu
#define SS_MIX_L 0xca01f9ddu
#define SS_MIX_R 0x4973f715u

static uint32_t ss_hashmix(uint32_t v, uint32_t *hc) {
    v ^= *hc;
    *hc *= SS_MULT_A;
    v *= *hc;
    v ^= v >> 16;
    return v;
}

static uint32_t ss_mix(uint32_t x, uint32_t y) {
    uint32_t r = SS_MIX_L * x - SS_MIX_R * y;
    r ^= r >> 16;
    return r;
}

/* words = the assembled entropy array (run entropy, zero-padded to 4 words when
 * a spawn key is present, followed by the spawn-key words).  Writes the Philox key. */
void orc_seedseq_key(const uint32_t *words, int n, uint64_t key[2]) {
    uint32_t pool[4];
    uint32_t hc = SS_INIT_A;
    for (int i = 0; i < 4; i++) pool[i] = ss_hashmix(i < n ? words[i] : 0u, &hc);
    for (int s = 0; s < 4; s++)
        for (int d = 0; d < 4; d++)
            if (s != d) pool[d] = ss_mix(pool[d], ss_hashmix(pool[s], &hc));
    for (int s = 4; s < n; s++)
        for (int d = 0; d < 4; d++) pool[d] = ss_mix(pool[d], ss_hashmix(words[s], &hc));
    uint32_t out[4];
    uint32_t hb = SS_INIT_B;
    for (int i = 0; i < 4; i++) {
        uint32_t v = pool[i] ^ hb;
        hb *= SS_MULT_B;
        v *= hb;
        v ^= v >> 16;
        out[i] = v;
    }
    key[0] = (uint64_t)out[0] | ((uint64_t)out[1] << 32);
    key[1] = (uint64_t)out[2] | ((uint64_t)out[3] << 32);
}

/* ----------------------------------------------------------------------------
 * Philox4x64-10 bit generator with numpy's buffering
 * ------------------------------------------------------------------------- */
typedef struct {
    uint64_t ctr[4];
    uint64_t key[2];
    uint64_t buf[4];
    int pos;          /* 4 = buffer empty */
    int has32;
    uint32_t half;
} orc_philox;

static uint64_t mulhilo(uint64_t a, uint64_t b, uint64_t *hi) {
    __uint128_t p = (__uint128_t)a * b;
    *hi = (uint64_t)(p >> 64);
    return (uint64_t)p;
}

static void philox_block(const uint64_t in[4], const uint64_t key_in[2], uint64_t out[4]) {
    uint64_t c0 = in[0], c1 = in[1], c2 = in[2], c3 = in[3];
    uint64_t k0 = key_in[0], k1 = key_in[1];
    for (int r = 0; r < 10; r++) {
        if (r > 0) {
            k0 += 0x9E3779B97F4A7C15ull;
            k1 += 0xBB67AE8584CAA73Bull;
        }
        uint64_t h0, h1;
        uint64_t l0 = mulhilo(0xD2E7470EE14C6C93ull, c0, &h0);
        uint64_t l1 = mulhilo(0xCA5A826395121157ull, c2, &h1);
        uint64_t n0 = h1 ^ c1 ^ k0, n2 = h0 ^ c3 ^ k1;
        c0 = n0; c1 = l1; c2 = n2; c3 = l0;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

void orc_philox_init(orc_philox *g, const uint64_t key[2]) {
    memset(g, 0, sizeof(*g));
    g->key[0] = key[0];
    g->key[1] = key[1];
    g->pos = 4;
}

uint64_t orc_next64(orc_philox *g) {
    if (g->pos < 4) return g->buf[g->pos++];
    if (++g->ctr[0] == 0)
        if (++g->ctr[1] == 0)
            if (++g->ctr[2] == 0) ++g->ctr[3];
    philox_block(g->ctr, g->key, g->buf);
    g->pos = 1;
    return g->buf[0];
}

uint32_t orc_next32(orc_philox *g) {
    if (g->has32) {
        g->has32 = 0;
        return g->half;
    }
    uint64_t v = orc_next64(g);
    g->has32 = 1;
    g->half = (uint32_t)(v >> 32);
    return (uint32_t)v;
}

double orc_random(orc_philox *g) {
    return (double)(orc_next64(g) >> 11) * (1.0 / 9007199254740992.0);
}

/* Generator.integers(0, n) for 1 <= n <= 2^32 - 1: 32-bit Lemire rejection. */
uint32_t orc_below(orc_philox *g, uint32_t n) {
    uint32_t rng = n - 1u;
    if (rng == 0) return 0;
    uint64_t m = (uint64_t)orc_next32(g) * n;
    uint32_t left = (uint32_t)m;
    if (left < n) {
        uint32_t thresh = (0xFFFFFFFFu - rng) % n;
        while (left < thresh) {
            m = (uint64_t)orc_next32(g) * n;
            left = (uint32_t)m;
        }
    }
    return (uint32_t)(m >> 32);
}

/* random_interval(max) with max < 2^32: masked rejection. */
uint32_t orc_interval(orc_philox *g, uint32_t max) {
    if (max == 0) return 0;
    uint32_t mask = max;
    mask |= mask >> 1; mask |= mask >> 2; mask |= mask >> 4;
    mask |= mask >> 8; mask |= mask >> 16;
    uint32_t v;
    while ((v = orc_next32(g) & mask) > max) {
    }
    return v;
}

/* Generator.permutation(n) on an int64 arange. */
void orc_permutation(orc_philox *g, int n, int32_t *out) {
    for (int i = 0; i < n; i++) out[i] = i;
    for (int i = n - 1; i >= 1; i--) {
        uint32_t j = orc_interval(g, (uint32_t)i);
        int32_t t = out[i];
        out[i] = out[j];
        out[j] = t;
    }
}

/* ----------------------------------------------------------------------------
 * Levels
 * ------------------------------------------------------------------------- */
typedef struct {
    uint32_t walls[4];
    uint8_t agent_r, agent_c, agent_dir, goal_r, goal_c, pad0, pad1, pad2;
    uint32_t pad3, pad4;
} orc_level; /* 32 bytes, identical to amz_level_t in include/amaze_b200.h */

static int bit_get(const uint32_t w[4], int i) { return (w[i >> 5] >> (i & 31)) & 1; }
static void bit_flip(uint32_t w[4], int i) { w[i >> 5] ^= 1u << (i & 31); }

/* amaze/generator.py:36-52. ``words``/``n`` = the lane's assembled entropy. */
void orc_sample_level(const uint32_t *words, int n, int H, int W, int budget, orc_level *out) {
    uint64_t key[2];
    orc_seedseq_key(words, n, key);
    orc_philox g;
    orc_philox_init(&g, key);
    const int iw = W - 2, ni = (H - 2) * (W - 2);
    int32_t order[256];
    memset(out, 0, sizeof(*out));
    uint32_t n_walls = orc_below(&g, (uint32_t)budget + 1u);
    orc_permutation(&g, ni, order);
    for (uint32_t k = 0; k < n_walls; k++) {
        int i = order[k];
        out->walls[i >> 5] |= 1u << (i & 31);
    }
    /* free cells in permutation order */
    int nfree = ni - (int)n_walls;
    const int32_t *fr = order + n_walls;
    uint32_t gk = orc_below(&g, (uint32_t)nfree);
    int goal = fr[gk];
    /* drop the goal, keep order, pick the agent */
    uint32_t ak = orc_below(&g, (uint32_t)(nfree - 1));
    int agent = fr[ak < gk ? ak : ak + 1];
    uint32_t dir = orc_below(&g, 4u);
    out->goal_r = (uint8_t)(goal / iw + 1);
    out->goal_c = (uint8_t)(goal % iw + 1);
    out->agent_r = (uint8_t)(agent / iw + 1);
    out->agent_c = (uint8_t)(agent % iw + 1);
    out->agent_dir = (uint8_t)dir;
}

/* amaze/generator.py:55-84. Cells are enumerated row-major over the interior. */
void orc_mutate_level(const uint32_t *words, int n, int H, int W, int n_edits,
                      const orc_level *in, orc_level *out) {
    uint64_t key[2];
    orc_seedseq_key(words, n, key);
    orc_philox g;
    orc_philox_init(&g, key);
    const int iw = W - 2, ni = (H - 2) * (W - 2);
    *out = *in;
    int agent = (in->agent_r - 1) * iw + (in->agent_c - 1);
    int goal = (in->goal_r - 1) * iw + (in->goal_c - 1);
    for (int e = 0; e < n_edits; e++) {
        if (orc_random(&g) < 0.05) {
            /* goal := uniform cell among interior, not wall, not agent (may be the current goal) */
            int nfree = 0;
            for (int i = 0; i < ni; i++) nfree += (!bit_get(out->walls, i) && i != agent);
            uint32_t k = orc_below(&g, (uint32_t)nfree);
            for (int i = 0; i < ni; i++) {
                if (!bit_get(out->walls, i) && i != agent) {
                    if (k == 0) { goal = i; break; }
                    k--;
                }
            }
        } else {
            /* toggle a uniform interior cell that is neither agent nor goal */
            int ncand = ni - 1 - (agent != goal);
            uint32_t k = orc_below(&g, (uint32_t)ncand);
            for (int i = 0; i < ni; i++) {
                if (i != agent && i != goal) {
                    if (k == 0) { bit_flip(out->walls, i); break; }
                    k--;
                }
            }
        }
    }
    out->goal_r = (uint8_t)(goal / iw + 1);
    out->goal_c = (uint8_t)(goal % iw + 1);
}

/* Batch helpers used by the CPU baseline: lane i's entropy = prefix ++ [i] (++ suffix). */
void orc_sample_levels_batch(const uint32_t *prefix, int n_prefix, uint32_t lane0, int count,
                             int H, int W, int budget, orc_level *out) {
    uint32_t words[64];
    memcpy(words, prefix, sizeof(uint32_t) * (size_t)n_prefix);
    for (int i = 0; i < count; i++) {
        words[n_prefix] = lane0 + (uint32_t)i;
        orc_sample_level(words, n_prefix + 1, H, W, budget, &out[i]);
    }
}

void orc_mutate_levels_batch(const uint32_t *prefix, int n_prefix, uint32_t lane0, int count,
                             int H, int W, int n_edits, const orc_level *in, orc_level *out) {
    uint32_t words[64];
    memcpy(words, prefix, sizeof(uint32_t) * (size_t)n_prefix);
    for (int i = 0; i < count; i++) {
        words[n_prefix] = lane0 + (uint32_t)i;
        orc_mutate_level(words, n_prefix + 1, H, W, n_edits, &in[i], &out[i]);
    }
}

/* Raw-stream probes for the RNG tests. */
void orc_probe_stream(const uint32_t *words, int n, int kind, uint32_t arg, int count, uint64_t *out) {
    uint64_t key[2];
    orc_seedseq_key(words, n, key);
    orc_philox g;
    orc_philox_init(&g, key);
    for (int i = 0; i < count; i++) {
        switch (kind) {
        case 0: out[i] = orc_next64(&g); break;
        case 1: out[i] = orc_next32(&g); break;
        case 2: out[i] = orc_below(&g, arg); break;
        case 3: { double d = orc_random(&g); memcpy(&out[i], &d, 8); } break;
        default: out[i] = orc_interval(&g, arg); break;
        }
    }
}
