/*
 * oracle/mickey_oracle.c -- CPU restatement of the reference's MICKEY 2.0 path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing under paper_1909_04750_b200/ may import,
 * link or call this file.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs use it, and there only as the checker
 * (or as the CPU arm that is timed beside the GPU path), never as the product.
 *
 * Parity status: PINNED.  tests/test_oracle.py checks this file against
 *   - the three eSTREAM known-answer vectors the reference embeds
 *     (pkg/src/slicerng/vectors.py:41-60), and
 *   - tests/golden/mickey_golden.json, produced by oracle/gen_golden.py by
 *     importing the reference package itself (scalar, packed, sliced and numba
 *     engines) in the build container.
 *
 * Every function cites the reference lines (relative to /root/reference/) it
 * restates.  The reference is pure Python + numba; this is a from-scratch C
 * restatement of the same algorithm, not a translation of its source text.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <unistd.h>

#define NB 100 /* bits per register: pkg/src/slicerng/mickey.py:31 */

/* Cipher tables, bit i of the table = word i/32 bit i%32
 * (pkg/src/slicerng/mickey.py:35-39, expanded by _expand at :49-50). */
static const uint32_t T_RTAPS[4] = {0x1279327Bu, 0xB5546660u, 0xDF87818Fu, 0x00000003u};
static const uint32_t T_COMP0[4] = {0x6AA97A30u, 0x7942A809u, 0x057EBFEAu, 0x00000006u};
static const uint32_t T_COMP1[4] = {0xDD629E9Au, 0xE3A21D63u, 0x91C23DD7u, 0x00000001u};
static const uint32_t T_FB0[4] = {0x9FFA7FAFu, 0xAF4A9381u, 0x9CEC5802u, 0x00000001u};
static const uint32_t T_FB1[4] = {0x4C8CB877u, 0x4911B063u, 0x40FBC52Bu, 0x00000008u};

static inline int tb(const uint32_t *t, int i) { return (int)((t[i >> 5] >> (i & 31)) & 1u); }

/* export the tables so tests can compare them with the golden file */
void mk2o_tables(uint8_t out[5][NB])
{
    const uint32_t *all[5] = {T_RTAPS, T_COMP0, T_COMP1, T_FB0, T_FB1};
    for (int k = 0; k < 5; ++k)
        for (int i = 0; i < NB; ++i)
            out[k][i] = (uint8_t)tb(all[k], i);
}

/* ------------------------------------------------------------------------
 * Bit-serial engine: one instance, one byte per state bit.
 * Normative clock: pkg/src/slicerng/mickey.py:110-139 (MickeyScalar).
 * ---------------------------------------------------------------------- */
typedef struct {
    uint8_t r[NB];
    uint8_t s[NB];
} mk2o_scalar;

void mk2o_scalar_reset(mk2o_scalar *st) { memset(st, 0, sizeof *st); }

/* mickey.py:110-117 clock_kg; :119-129 _clock_r; :131-139 _clock_s */
void mk2o_scalar_clock(mk2o_scalar *st, int mixing, int in)
{
    const uint8_t *r = st->r, *s = st->s;
    int ctrl_r = s[34] ^ r[67];
    int ctrl_s = s[67] ^ r[33];
    int in_r = mixing ? (in ^ s[50]) : in;
    uint8_t nr[NB], ns[NB];

    int fbr = r[99] ^ in_r;
    nr[0] = 0;
    for (int i = 1; i < NB; ++i) nr[i] = r[i - 1];
    if (fbr)
        for (int i = 0; i < NB; ++i) nr[i] ^= (uint8_t)tb(T_RTAPS, i);
    if (ctrl_r)
        for (int i = 0; i < NB; ++i) nr[i] ^= r[i];

    int fbs = s[99] ^ in;
    ns[0] = 0;
    for (int i = 1; i < 99; ++i)
        ns[i] = (uint8_t)(s[i - 1] ^ ((s[i] ^ tb(T_COMP0, i)) & (s[i + 1] ^ tb(T_COMP1, i))));
    ns[99] = s[98];
    if (fbs) {
        const uint32_t *fb = ctrl_s ? T_FB1 : T_FB0;
        for (int i = 0; i < NB; ++i) ns[i] ^= (uint8_t)tb(fb, i);
    }
    memcpy(st->r, nr, NB);
    memcpy(st->s, ns, NB);
}

/* key/IV bit c is the (7 - c%8)-th bit of byte c/8: bitops.py:33-36 */
static inline int msb_bit(const uint8_t *bytes, int c) { return (bytes[c >> 3] >> (7 - (c & 7))) & 1; }

/* mickey.py:141-151 from_key_iv: IV bits, 80 key bits, 100 pre-clocks, all mixing */
void mk2o_scalar_init(mk2o_scalar *st, const uint8_t key[10], const uint8_t *iv, int iv_nbits)
{
    mk2o_scalar_reset(st);
    for (int c = 0; c < iv_nbits; ++c) mk2o_scalar_clock(st, 1, msb_bit(iv, c));
    for (int c = 0; c < 80; ++c) mk2o_scalar_clock(st, 1, msb_bit(key, c));
    for (int c = 0; c < 100; ++c) mk2o_scalar_clock(st, 1, 0);
}

/* mickey.py:153-161: z = r0 ^ s0 sampled before the clock; MSB-first bytes
 * (bitops.py:20-23). */
void mk2o_scalar_keystream_bytes(mk2o_scalar *st, uint64_t nbytes, uint8_t *out)
{
    for (uint64_t b = 0; b < nbytes; ++b) {
        unsigned v = 0;
        for (int k = 0; k < 8; ++k) {
            v = (v << 1) | (unsigned)(st->r[0] ^ st->s[0]);
            mk2o_scalar_clock(st, 0, 0);
        }
        out[b] = (uint8_t)v;
    }
}

void mk2o_scalar_keystream_bits(mk2o_scalar *st, uint64_t nbits, uint8_t *out)
{
    for (uint64_t t = 0; t < nbits; ++t) {
        out[t] = (uint8_t)(st->r[0] ^ st->s[0]);
        mk2o_scalar_clock(st, 0, 0);
    }
}

/* ------------------------------------------------------------------------
 * Column-major ("sliced") engine, 64 lanes per word.
 * Word clock: pkg/src/slicerng/mickey.py:329-360 (MickeySliced.clock_kg).
 * ---------------------------------------------------------------------- */
typedef struct {
    uint64_t r[NB];
    uint64_t s[NB];
} mk2o_sliced;

void mk2o_sliced_reset(mk2o_sliced *st) { memset(st, 0, sizeof *st); }

void mk2o_sliced_clock(mk2o_sliced *st, int mixing, uint64_t in)
{
    const uint64_t *r = st->r, *s = st->s;
    uint64_t ctrl_r = s[34] ^ r[67];
    uint64_t ctrl_s = s[67] ^ r[33];
    uint64_t in_r = mixing ? (in ^ s[50]) : in;
    uint64_t fbr = r[99] ^ in_r;
    uint64_t fbs = s[99] ^ in;
    uint64_t fb1 = fbs & ctrl_s, fb0 = fbs & ~ctrl_s;
    uint64_t nr[NB], ns[NB];

    nr[0] = ctrl_r & r[0];
    for (int i = 1; i < NB; ++i) nr[i] = r[i - 1] ^ (ctrl_r & r[i]);
    for (int i = 0; i < NB; ++i)
        if (tb(T_RTAPS, i)) nr[i] ^= fbr;

    ns[0] = 0;
    for (int i = 1; i < 99; ++i) {
        uint64_t c0 = tb(T_COMP0, i) ? ~0ull : 0ull;
        uint64_t c1 = tb(T_COMP1, i) ? ~0ull : 0ull;
        ns[i] = s[i - 1] ^ ((s[i] ^ c0) & (s[i + 1] ^ c1));
    }
    ns[99] = s[98];
    for (int i = 0; i < NB; ++i) {
        int f0 = tb(T_FB0, i), f1 = tb(T_FB1, i);
        if (f0 && f1) ns[i] ^= fbs;
        else if (f0) ns[i] ^= fb0;
        else if (f1) ns[i] ^= fb1;
    }
    memcpy(st->r, nr, sizeof nr);
    memcpy(st->s, ns, sizeof ns);
}

/* mickey.py:258-304 from_key_ivs.  keys: n x 10 bytes; ivs: n x iv_stride
 * bytes (MSB-first bits); iv_nbits: per-lane IV bit lengths (n entries).
 * Uniform lengths take the word-wide route (:291-303); ragged lengths take the
 * per-lane scalar route + transpose (:287-289, :306-316).  Lanes >= n stay
 * all-zero material (they behave as zero key / empty-or-zero IV lanes of the
 * same clock count, exactly as the reference's unused lanes do).
 * Returns 0, or -(lane+1) when a lane's IV is longer than 80 bits. */
int mk2o_sliced_init2(mk2o_sliced *st, const uint8_t *keys, const uint8_t *ivs, int iv_stride,
                      const uint8_t *iv_nbits, int n, int force_ragged)
{
    if (n < 1 || n > 64) return -1000;
    int uniform = !force_ragged;
    for (int j = 0; j < n; ++j) {
        if (iv_nbits[j] > 80) return -(j + 1);
        if (iv_nbits[j] != iv_nbits[0]) uniform = 0;
    }
    mk2o_sliced_reset(st);
    if (!uniform) {
        for (int j = 0; j < n; ++j) {
            mk2o_scalar sc;
            mk2o_scalar_init(&sc, keys + 10 * j, ivs + (size_t)iv_stride * j, iv_nbits[j]);
            for (int i = 0; i < NB; ++i) {
                st->r[i] |= (uint64_t)sc.r[i] << j;
                st->s[i] |= (uint64_t)sc.s[i] << j;
            }
        }
        return 0;
    }
    for (int c = 0; c < iv_nbits[0]; ++c) {
        uint64_t w = 0;
        for (int j = 0; j < n; ++j) w |= (uint64_t)msb_bit(ivs + (size_t)iv_stride * j, c) << j;
        mk2o_sliced_clock(st, 1, w);
    }
    for (int c = 0; c < 80; ++c) {
        uint64_t w = 0;
        for (int j = 0; j < n; ++j) w |= (uint64_t)msb_bit(keys + 10 * j, c) << j;
        mk2o_sliced_clock(st, 1, w);
    }
    for (int c = 0; c < 100; ++c) mk2o_sliced_clock(st, 1, 0);
    return 0;
}

int mk2o_sliced_init(mk2o_sliced *st, const uint8_t *keys, const uint8_t *ivs, int iv_stride,
                     const uint8_t *iv_nbits, int n)
{
    return mk2o_sliced_init2(st, keys, ivs, iv_stride, iv_nbits, n, 0);
}

/* mickey.py:362-368 keystream_words (resumable, state advances) */
void mk2o_sliced_keystream_words(mk2o_sliced *st, uint64_t n, uint64_t *out)
{
    for (uint64_t t = 0; t < n; ++t) {
        out[t] = st->r[0] ^ st->s[0];
        mk2o_sliced_clock(st, 0, 0);
    }
}

/* ------------------------------------------------------------------------
 * The compiled keystream loop the reference times:
 * pkg/src/slicerng/kernels.py:46-95 (_mickey_sliced_loop).  Same structure:
 * runtime all-ones/zero mask arrays (kernels.py:32-43), ping-pong buffers,
 * body written for two clocks, no state write-back.  n must be even.
 * ---------------------------------------------------------------------- */
static uint64_t M_RT[NB], M_C0[NB], M_C1[NB], M_FB0[NB], M_FB1[NB];
static int masks_ready = 0;

static void build_masks(void)
{
    if (masks_ready) return;
    for (int i = 0; i < NB; ++i) {
        M_RT[i] = tb(T_RTAPS, i) ? ~0ull : 0;
        M_C0[i] = tb(T_COMP0, i) ? ~0ull : 0;
        M_C1[i] = tb(T_COMP1, i) ? ~0ull : 0;
        M_FB0[i] = tb(T_FB0, i) ? ~0ull : 0;
        M_FB1[i] = tb(T_FB1, i) ? ~0ull : 0;
    }
    masks_ready = 1;
}

static inline void loop_half(const uint64_t *restrict ra, const uint64_t *restrict sa,
                             uint64_t *restrict rb, uint64_t *restrict sb, uint64_t *zout)
{
    *zout = ra[0] ^ sa[0];
    uint64_t ctrl_r = sa[34] ^ ra[67];
    uint64_t ctrl_s = sa[67] ^ ra[33];
    uint64_t fb_r = ra[99], fb_s = sa[99];
    uint64_t a_sel = fb_s & ~ctrl_s, b_sel = fb_s & ctrl_s;
    rb[0] = (ctrl_r & ra[0]) ^ (fb_r & M_RT[0]);
    for (int i = 1; i < NB; ++i) rb[i] = ra[i - 1] ^ (ctrl_r & ra[i]) ^ (fb_r & M_RT[i]);
    sb[0] = (M_FB0[0] & a_sel) | (M_FB1[0] & b_sel);
    for (int i = 1; i < 99; ++i)
        sb[i] = sa[i - 1] ^ ((sa[i] ^ M_C0[i]) & (sa[i + 1] ^ M_C1[i])) ^
                ((M_FB0[i] & a_sel) | (M_FB1[i] & b_sel));
    sb[99] = sa[98] ^ ((M_FB0[99] & a_sel) | (M_FB1[99] & b_sel));
}

void mk2o_sliced_loop(const uint64_t r_io[NB], const uint64_t s_io[NB], uint64_t *out, uint64_t n)
{
    uint64_t ra[NB], sa[NB], rb[NB], sb[NB];
    build_masks();
    memcpy(ra, r_io, sizeof ra);
    memcpy(sa, s_io, sizeof sa);
    for (uint64_t it = 0; it < n / 2; ++it) {
        loop_half(ra, sa, rb, sb, &out[2 * it]);
        loop_half(rb, sb, ra, sa, &out[2 * it + 1]);
    }
}

/* ------------------------------------------------------------------------
 * Bulk generator over N instances, in the layouts the GPU boundary emits
 * (SURVEY.md section 8(b)):
 *   column-major: uint32 out[T][G], G = ceil(N/32), bit j of out[t][g] =
 *                 keystream bit t of instance 32 g + j; lanes >= N inside the
 *                 last group are the reference's "unused lanes" (zero
 *                 material when IV lengths are uniform, zero state when
 *                 ragged) and are NOT masked, as at width 64 in the reference.
 *   row-major:    uint8 out[N][T/8], MSB-first bytes (kernels.py:604-621).
 * Built from kernels.py:189-200 (mickey_sliced_words = init + loop + width
 * mask) applied to consecutive batches of 64 lanes, the way the reference's
 * callers batch (cli.py:219-231).  iv_nbits_uniform < 0 means per-lane
 * lengths are given in iv_nbits[].  Threads: pthreads pulling 64-lane batches from a shared counter.
 * ---------------------------------------------------------------------- */
static void batch_words(const uint8_t *keys, const uint8_t *ivs, int iv_stride, const uint8_t *iv_nbits,
                        int iv_uniform, uint64_t first, uint64_t N, uint64_t T, uint64_t *words)
{
    int n = (int)((N - first) < 64 ? (N - first) : 64);
    uint8_t lens[64];
    for (int j = 0; j < n; ++j) lens[j] = iv_uniform >= 0 ? (uint8_t)iv_uniform : iv_nbits[first + j];
    mk2o_sliced st;
    /* uniform call (one IV length for the whole set): word-wide route, unused
     * lanes load zero bits for the same clock count; per-lane lengths: always
     * the scalar route, unused lanes stay in the zero state -- the two routes of
     * mickey.py:287-303, chosen per CALL so padding does not depend on how a
     * ragged set happens to fall into 64-lane batches. */
    mk2o_sliced_init2(&st, keys + 10 * first, ivs + (size_t)iv_stride * first, iv_stride, lens, n, iv_uniform < 0);
    /* no lane mask at width 64 (kernels.py:196-200): unused lanes keep the
     * keystream of their padding material, exactly as in the reference */
    mk2o_sliced_loop(st.r, st.s, words, T + (T & 1));
}

/* minimal pthread pool: workers pull batch indices from an atomic counter */
typedef struct {
    const uint8_t *keys, *ivs, *iv_nbits;
    int iv_stride, iv_uniform, rowmajor;
    uint64_t N, T, G, nb;
    void *out;
    uint64_t next; /* atomic */
    int fail;
} bulk_job;

static void *bulk_worker(void *arg)
{
    bulk_job *jb = (bulk_job *)arg;
    uint64_t T = jb->T, G = jb->G, rowb = T / 8;
    uint64_t *words = (uint64_t *)malloc((T + 2) * sizeof(uint64_t));
    if (!words) {
        __atomic_store_n(&jb->fail, 1, __ATOMIC_RELAXED);
        return NULL;
    }
    for (;;) {
        uint64_t b = __atomic_fetch_add(&jb->next, 1, __ATOMIC_RELAXED);
        if (b >= jb->nb) break;
        uint64_t first = b * 64;
        batch_words(jb->keys, jb->ivs, jb->iv_stride, jb->iv_nbits, jb->iv_uniform, first, jb->N, T, words);
        if (!jb->rowmajor) {
            uint32_t *out = (uint32_t *)jb->out;
            uint64_t g0 = b * 2;
            for (uint64_t t = 0; t < T; ++t) {
                out[t * G + g0] = (uint32_t)words[t];
                if (g0 + 1 < G) out[t * G + g0 + 1] = (uint32_t)(words[t] >> 32);
            }
        } else {
            uint8_t *out = (uint8_t *)jb->out;
            int n = (int)((jb->N - first) < 64 ? (jb->N - first) : 64);
            for (int j = 0; j < n; ++j) { /* kernels.py:604-612, msb packing */
                uint8_t *row = out + (first + (uint64_t)j) * rowb;
                for (uint64_t q = 0; q < rowb; ++q) {
                    unsigned v = 0;
                    for (int k = 0; k < 8; ++k) v = (v << 1) | (unsigned)((words[8 * q + k] >> j) & 1);
                    row[q] = (uint8_t)v;
                }
            }
        }
    }
    free(words);
    return NULL;
}

int mk2o_max_threads(void)
{
    long n = sysconf(_SC_NPROCESSORS_ONLN);
    return n < 1 ? 1 : (int)n;
}

static int run_bulk(bulk_job *jb, int nthreads)
{
    build_masks();
    if (nthreads < 1) nthreads = mk2o_max_threads();
    if ((uint64_t)nthreads > jb->nb) nthreads = (int)(jb->nb ? jb->nb : 1);
    if (nthreads > 1024) nthreads = 1024;
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)nthreads);
    if (!th) return -1;
    int started = 0;
    for (int i = 0; i < nthreads; ++i) {
        if (pthread_create(&th[i], NULL, bulk_worker, jb) != 0) break;
        ++started;
    }
    if (started == 0) bulk_worker(jb); /* degrade to the calling thread */
    for (int i = 0; i < started; ++i) pthread_join(th[i], NULL);
    free(th);
    return jb->fail ? -1 : 0;
}

int mk2o_bulk_colmajor(const uint8_t *keys, const uint8_t *ivs, int iv_stride, const uint8_t *iv_nbits,
                       int iv_uniform, uint64_t N, uint64_t T, uint32_t *out, int nthreads)
{
    bulk_job jb = {keys, ivs, iv_nbits, iv_stride, iv_uniform, 0, N, T, (N + 31) / 32, (N + 63) / 64, out, 0, 0};
    return run_bulk(&jb, nthreads);
}

int mk2o_bulk_rowmajor(const uint8_t *keys, const uint8_t *ivs, int iv_stride, const uint8_t *iv_nbits,
                       int iv_uniform, uint64_t N, uint64_t T, uint8_t *out, int nthreads)
{
    if (T % 8) return -2; /* bitops.py:17-18 */
    bulk_job jb = {keys, ivs, iv_nbits, iv_stride, iv_uniform, 1, N, T, (N + 31) / 32, (N + 63) / 64, out, 0, 0};
    return run_bulk(&jb, nthreads);
}

/* Timing arm for bench.py: exactly what the reference's bench times
 * (pkg/src/slicerng/bench.py:169-183): W=64, keystream loop only, init and
 * transposition outside the timed region.  Each worker thread runs an
 * independent generator (bench.py:265-282).  Caller passes one initial state
 * per worker (r/s: nworkers x 100 words) and a scratch of nworkers x nclocks
 * words; returns an XOR of the last words so the work cannot be elided. */
typedef struct {
    const uint64_t *r, *s;
    uint64_t *o;
    uint64_t nclocks;
    int ncalls;
} loop_job;

static void *loop_worker(void *arg)
{
    loop_job *lj = (loop_job *)arg;
    for (int c = 0; c < lj->ncalls; ++c) mk2o_sliced_loop(lj->r, lj->s, lj->o, lj->nclocks);
    return NULL;
}

/* ncalls back-to-back runs of the loop per worker over the same scratch (the
 * reference's `repeats`), so the sample size is not bounded by memory. */
uint64_t mk2o_timed_loops(const uint64_t *r, const uint64_t *s, uint64_t *scratch, uint64_t nclocks,
                          int ncalls, int nworkers)
{
    build_masks();
    if (nworkers < 1) nworkers = 1;
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)nworkers);
    loop_job *jobs = (loop_job *)malloc(sizeof(loop_job) * (size_t)nworkers);
    uint64_t sink = 0;
    if (!th || !jobs) {
        free(th);
        free(jobs);
        return 0;
    }
    for (int w = 0; w < nworkers; ++w) {
        jobs[w] = (loop_job){r + (size_t)w * NB, s + (size_t)w * NB, scratch + (size_t)w * nclocks, nclocks, ncalls};
        if (w > 0 && pthread_create(&th[w], NULL, loop_worker, &jobs[w]) != 0) loop_worker(&jobs[w]), th[w] = 0;
    }
    loop_worker(&jobs[0]);
    for (int w = 1; w < nworkers; ++w)
        if (th[w]) pthread_join(th[w], NULL);
    for (int w = 0; w < nworkers; ++w) sink ^= jobs[w].o[nclocks - 1];
    free(th);
    free(jobs);
    return sink;
}

/* Checksum both sides agree on: the column-major buffer read
 * as little-endian uint64 words, summed mod 2^64.  Written per group so it is
 * layout independent: word of group g counts with weight 2^(32 (g & 1)). */
uint64_t mk2o_checksum_colmajor(const uint32_t *out, uint64_t T, uint64_t G, uint64_t g_offset)
{
    uint64_t acc = 0;
    for (uint64_t t = 0; t < T; ++t)
        for (uint64_t g = 0; g < G; ++g) acc += (uint64_t)out[t * G + g] << (32 * ((g + g_offset) & 1));
    return acc;
}

/* ------------------------------------------------------------------------
 * The same checksum for a whole job, WITHOUT materialising the keystream, so
 * that BASELINE-size geometries (2^20 instances, every chain) can be checked
 * instance by instance: mk2o_checksum_colmajor(mk2o_bulk_colmajor(...)) computed
 * batch by batch (64 lanes = one call of kernels.mickey_sliced_words,
 * kernels.py:189-200, as the reference's callers batch, cli.py:219-231).
 *   counter != 0: the synthetic set of SURVEY.md 8(d) -- every lane uses
 *       keys[0..9], lane n gets the 80-bit big-endian IV (first + n); ivs is
 *       ignored and first must be a multiple of 64;
 *   counter == 0: explicit material, arguments as mk2o_bulk_colmajor.
 * g_offset: global group index of group 0 (the weight 2^(32 ((g+g_offset)&1))).
 * *rc: 0, or -1 (allocation / thread failure).
 * ---------------------------------------------------------------------- */
typedef struct {
    const uint8_t *keys, *ivs, *iv_nbits;
    int iv_stride, iv_uniform, counter;
    uint64_t first, N, T, G, nb, g_offset;
    uint64_t next; /* atomic */
    uint64_t sum;  /* atomic */
    int fail;
} csum_job;

static void *csum_worker(void *arg)
{
    csum_job *jb = (csum_job *)arg;
    const uint64_t T = jb->T;
    uint64_t *words = (uint64_t *)malloc((T + 2) * sizeof(uint64_t));
    if (!words) {
        __atomic_store_n(&jb->fail, 1, __ATOMIC_RELAXED);
        return NULL;
    }
    uint64_t local = 0;
    for (;;) {
        const uint64_t b = __atomic_fetch_add(&jb->next, 1, __ATOMIC_RELAXED);
        if (b >= jb->nb) break;
        const uint64_t lane0 = b * 64;
        if (jb->counter) {
            /* all 64 lanes of the batch continue the counter, also past N: mk2_init_counter_iv synthesises
             * whole 32-lane groups (groups past G are dropped from the sum below) */
            const int n = 64;
            uint8_t k64[64 * 10], v64[64 * 10];
            for (int j = 0; j < n; ++j) {
                const uint64_t idx = jb->first + lane0 + (uint64_t)j;
                memcpy(k64 + 10 * j, jb->keys, 10);
                v64[10 * j] = v64[10 * j + 1] = 0;
                for (int q = 0; q < 8; ++q) v64[10 * j + 2 + q] = (uint8_t)(idx >> (8 * (7 - q)));
            }
            batch_words(k64, v64, 10, NULL, 80, 0, (uint64_t)n, T, words);
        } else {
            batch_words(jb->keys, jb->ivs, jb->iv_stride, jb->iv_nbits, jb->iv_uniform, lane0, jb->N, T, words);
        }
        const uint64_t g0 = 2 * b;
        const int has_hi = g0 + 1 < jb->G;
        const int odd = (int)((g0 + jb->g_offset) & 1);
        uint64_t lo = 0, hi = 0;
        for (uint64_t t = 0; t < T; ++t) {
            lo += (uint32_t)words[t];
            hi += words[t] >> 32;
        }
        if (!has_hi) hi = 0;
        local += odd ? (lo << 32) + hi : lo + (hi << 32);
    }
    free(words);
    __atomic_fetch_add(&jb->sum, local, __ATOMIC_RELAXED);
    return NULL;
}

uint64_t mk2o_checksum_job(const uint8_t *keys, const uint8_t *ivs, int iv_stride, const uint8_t *iv_nbits,
                           int iv_uniform, int counter, uint64_t first, uint64_t N, uint64_t T, uint64_t g_offset,
                           int nthreads, int *rc)
{
    csum_job jb = {keys, ivs, iv_nbits, iv_stride, iv_uniform, counter, first, N, T, (N + 31) / 32, (N + 63) / 64,
                   g_offset, 0, 0, 0};
    build_masks();
    if (nthreads < 1) nthreads = mk2o_max_threads();
    if ((uint64_t)nthreads > jb.nb) nthreads = (int)(jb.nb ? jb.nb : 1);
    if (nthreads > 1024) nthreads = 1024;
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)nthreads);
    int started = 0;
    if (th)
        for (int i = 0; i < nthreads; ++i) {
            if (pthread_create(&th[i], NULL, csum_worker, &jb) != 0) break;
            ++started;
        }
    if (started == 0) csum_worker(&jb); /* degrade to the calling thread */
    for (int i = 0; i < started; ++i) pthread_join(th[i], NULL);
    free(th);
    if (rc) *rc = jb.fail ? -1 : 0;
    return jb.sum;
}

/* ------------------------------------------------------------------------
 * Seed derivation: pkg/src/slicerng/seedgen.py:57-86.
 * AES-128 is the standard FIPS-197 cipher the reference implements as
 * AesScalarTable (pkg/src/slicerng/aes_ctr.py:193-219); restated here with a
 * computed S-box (GF(2^8) inverse + affine map) instead of a table literal.
 *   dk      = AES_{seed[0:16]}(seed[16:32])                       seedgen.py:57-60
 *   block_c = tag || lane (4 bytes BE) || c (4 bytes BE) || 0^7   seedgen.py:72-78
 *   stream  = AES_dk(block_0) || AES_dk(block_1);  key = stream[0:10], iv = stream[10:20]
 * tag: 1 = aes-ctr, 2 = grain, 3 = mickey (sorted names, seedgen.py:31).
 * ---------------------------------------------------------------------- */
static uint8_t AES_SBOX[256];
static int aes_ready = 0;

static uint8_t gf_mul(uint8_t a, uint8_t b)
{
    uint8_t p = 0;
    for (int i = 0; i < 8; ++i) {
        if (b & 1) p ^= a;
        uint8_t hi = a & 0x80;
        a = (uint8_t)(a << 1);
        if (hi) a ^= 0x1B;
        b >>= 1;
    }
    return p;
}

static void aes_build(void)
{
    if (aes_ready) return;
    for (int x = 0; x < 256; ++x) {
        uint8_t inv = 0;
        if (x)
            for (int y = 1; y < 256; ++y)
                if (gf_mul((uint8_t)x, (uint8_t)y) == 1) { inv = (uint8_t)y; break; }
        uint8_t r = inv, v = inv;
        for (int k = 0; k < 4; ++k) { r = (uint8_t)((r << 1) | (r >> 7)); v ^= r; }
        AES_SBOX[x] = v ^ 0x63;
    }
    aes_ready = 1;
}

static void aes_expand(const uint8_t key[16], uint8_t rk[11][16])
{
    memcpy(rk[0], key, 16);
    uint8_t rcon = 1;
    for (int r = 1; r <= 10; ++r) {
        const uint8_t *p = rk[r - 1];
        uint8_t t[4] = {AES_SBOX[p[13]], AES_SBOX[p[14]], AES_SBOX[p[15]], AES_SBOX[p[12]]};
        t[0] ^= rcon;
        rcon = gf_mul(rcon, 2);
        for (int c = 0; c < 4; ++c)
            for (int b = 0; b < 4; ++b) {
                uint8_t prev = c ? rk[r][4 * (c - 1) + b] : t[b];
                rk[r][4 * c + b] = p[4 * c + b] ^ prev;
            }
    }
}

static void aes_encrypt(const uint8_t rk[11][16], const uint8_t in[16], uint8_t out[16])
{
    uint8_t st[16], t[16];
    for (int i = 0; i < 16; ++i) st[i] = in[i] ^ rk[0][i];
    for (int r = 1; r <= 10; ++r) {
        for (int i = 0; i < 16; ++i) t[i] = AES_SBOX[st[i]];
        /* ShiftRows: byte i = row i%4, column i/4; row k rotates left by k */
        for (int c = 0; c < 4; ++c)
            for (int k = 0; k < 4; ++k) st[4 * c + k] = t[4 * ((c + k) & 3) + k];
        if (r < 10)
            for (int c = 0; c < 4; ++c) {
                uint8_t *a = st + 4 * c, b0 = a[0], b1 = a[1], b2 = a[2], b3 = a[3], all = b0 ^ b1 ^ b2 ^ b3;
                a[0] = b0 ^ all ^ gf_mul(b0 ^ b1, 2);
                a[1] = b1 ^ all ^ gf_mul(b1 ^ b2, 2);
                a[2] = b2 ^ all ^ gf_mul(b2 ^ b3, 2);
                a[3] = b3 ^ all ^ gf_mul(b3 ^ b0, 2);
            }
        for (int i = 0; i < 16; ++i) st[i] ^= rk[r][i];
    }
    memcpy(out, st, 16);
}

void mk2o_aes128_encrypt(const uint8_t key[16], const uint8_t in[16], uint8_t out[16])
{
    uint8_t rk[11][16];
    aes_build();
    aes_expand(key, rk);
    aes_encrypt(rk, in, out);
}

void mk2o_derive_material(const uint8_t seed[32], uint32_t tag, uint64_t first_lane, uint64_t n, uint8_t *keys,
                          uint8_t *ivs)
{
    uint8_t rk[11][16], dk[16];
    aes_build();
    aes_expand(seed, rk);
    aes_encrypt(rk, seed + 16, dk);
    aes_expand(dk, rk);
    for (uint64_t j = 0; j < n; ++j) {
        uint64_t lane = first_lane + j;
        uint8_t stream[32];
        for (uint32_t c = 0; c < 2; ++c) {
            uint8_t blk[16] = {(uint8_t)tag, (uint8_t)(lane >> 24), (uint8_t)(lane >> 16), (uint8_t)(lane >> 8),
                               (uint8_t)lane, 0, 0, 0, (uint8_t)c, 0, 0, 0, 0, 0, 0, 0};
            aes_encrypt(rk, blk, stream + 16 * c);
        }
        memcpy(keys + 10 * j, stream, 10);
        memcpy(ivs + 10 * j, stream + 10, 10);
    }
}

/* ========================================================================
 * Grain v1: pkg/src/slicerng/grain.py.
 * 80-bit NFSR b and 80-bit LFSR s shift together every clock.
 *   f(s)  = s62^s51^s38^s23^s13^s0                                  grain.py:33-34, 120-124
 *   g(b)  = 11 linear taps ^ 11 product terms                        grain.py:36-52, 106-117
 *   h     = 5-input filter over s3,s25,s46,s64,b63                   grain.py:54-56, 96-103
 *   z     = h ^ b1^b2^b4^b10^b31^b43^b56                             grain.py:58-59, 127-133
 * init: b = key bits, s = iv bits || 1^16, 160 clocks with z fed back into both
 * registers (grain.py:147-156); key/IV bits LSB-first per byte (grain.py:88-92).
 * ====================================================================== */
#define GB 80
static const int G_LFSR[6] = {62, 51, 38, 23, 13, 0};
static const int G_NLIN[11] = {62, 60, 52, 45, 37, 33, 28, 21, 14, 9, 0};
static const int G_PROD[11][7] = {  /* first entry = length */
    {2, 63, 60}, {2, 37, 33}, {2, 15, 9}, {3, 60, 52, 45}, {3, 33, 28, 21}, {4, 63, 45, 28, 9},
    {4, 60, 52, 37, 33}, {4, 63, 60, 21, 15}, {5, 63, 60, 52, 45, 37}, {5, 33, 28, 21, 15, 9},
    {6, 52, 45, 37, 33, 28, 21}};
static const int G_OUT[7] = {1, 2, 4, 10, 31, 43, 56};

static inline uint64_t grain_h(uint64_t x0, uint64_t x1, uint64_t x2, uint64_t x3, uint64_t x4)
{
    return x1 ^ x4 ^ (x0 & x3) ^ (x2 & x3) ^ (x3 & x4) ^ (x0 & x1 & x2) ^ (x0 & x2 & x3) ^ (x0 & x2 & x4) ^
           (x1 & x2 & x4) ^ (x2 & x3 & x4);
}
static inline uint64_t grain_g(const uint64_t *b)
{
    uint64_t v = 0;
    for (int i = 0; i < 11; ++i) v ^= b[G_NLIN[i]];
    for (int i = 0; i < 11; ++i) {
        uint64_t p = ~0ull;
        for (int k = 1; k <= G_PROD[i][0]; ++k) p &= b[G_PROD[i][k]];
        v ^= p;
    }
    return v;
}
static inline uint64_t grain_f(const uint64_t *s)
{
    uint64_t v = 0;
    for (int i = 0; i < 6; ++i) v ^= s[G_LFSR[i]];
    return v;
}
static inline uint64_t grain_z(const uint64_t *b, const uint64_t *s)
{
    uint64_t z = grain_h(s[3], s[25], s[46], s[64], b[63]);
    for (int i = 0; i < 7; ++i) z ^= b[G_OUT[i]];
    return z;
}

/* word engine: lanes = bits of the words (1 lane => the scalar engine, GrainScalar grain.py:136-173;
 * 64 lanes => GrainSliced grain.py:232-308) */
typedef struct {
    uint64_t b[GB], s[GB];
} mk2o_grain;

static void grain_clock(mk2o_grain *st, int init, uint64_t *zout)
{
    uint64_t z = grain_z(st->b, st->s);
    uint64_t fl = grain_f(st->s), fn = grain_g(st->b) ^ st->s[0];
    if (init) { fl ^= z; fn ^= z; }
    memmove(st->s, st->s + 1, sizeof(uint64_t) * (GB - 1));
    memmove(st->b, st->b + 1, sizeof(uint64_t) * (GB - 1));
    st->s[GB - 1] = fl;
    st->b[GB - 1] = fn;
    if (zout) *zout = z;
}

static inline int lsb_bit(const uint8_t *bytes, int c) { return (bytes[c >> 3] >> (c & 7)) & 1; }

/* GrainSliced.from_key_ivs (grain.py:250-277): keys n x 10, ivs n x 8; the 16 top LFSR words
 * are ones only in the lanes that exist. */
int mk2o_grain_init(mk2o_grain *st, const uint8_t *keys, const uint8_t *ivs, int n)
{
    if (n < 1 || n > 64) return -1000;
    memset(st, 0, sizeof *st);
    for (int j = 0; j < n; ++j) {
        for (int i = 0; i < 80; ++i) st->b[i] |= (uint64_t)lsb_bit(keys + 10 * j, i) << j;
        for (int i = 0; i < 64; ++i) st->s[i] |= (uint64_t)lsb_bit(ivs + 8 * j, i) << j;
    }
    uint64_t full = n == 64 ? ~0ull : ((1ull << n) - 1);
    for (int i = 64; i < 80; ++i) st->s[i] = full;
    for (int c = 0; c < 160; ++c) grain_clock(st, 1, NULL);
    return 0;
}

void mk2o_grain_keystream_words(mk2o_grain *st, uint64_t n, uint64_t *out)
{
    for (uint64_t t = 0; t < n; ++t) grain_clock(st, 0, &out[t]);
}

/* bulk layouts as for MICKEY; rowmajor bytes msb (default) or lsb first (grain.py:171-172) */
typedef struct {
    const uint8_t *keys, *ivs;
    uint64_t N, T, G, nb;
    void *out;
    int rowmajor, lsb;
    uint64_t next;
} grain_job;

static void *grain_worker(void *arg)
{
    grain_job *jb = (grain_job *)arg;
    uint64_t T = jb->T, G = jb->G, rowb = T / 8;
    uint64_t *words = (uint64_t *)malloc((T + 1) * sizeof(uint64_t));
    if (!words) return NULL;
    for (;;) {
        uint64_t b = __atomic_fetch_add(&jb->next, 1, __ATOMIC_RELAXED);
        if (b >= jb->nb) break;
        uint64_t first = b * 64;
        int n = (int)((jb->N - first) < 64 ? (jb->N - first) : 64);
        mk2o_grain st;
        mk2o_grain_init(&st, jb->keys + 10 * first, jb->ivs + 8 * first, n);
        mk2o_grain_keystream_words(&st, T, words);
        if (!jb->rowmajor) {
            uint32_t *out = (uint32_t *)jb->out;
            for (uint64_t t = 0; t < T; ++t) {
                out[t * G + 2 * b] = (uint32_t)words[t];
                if (2 * b + 1 < G) out[t * G + 2 * b + 1] = (uint32_t)(words[t] >> 32);
            }
        } else {
            uint8_t *out = (uint8_t *)jb->out;
            for (int j = 0; j < n; ++j) {
                uint8_t *row = out + (first + (uint64_t)j) * rowb;
                for (uint64_t q = 0; q < rowb; ++q) {
                    unsigned v = 0;
                    for (int k = 0; k < 8; ++k) {
                        unsigned bit = (unsigned)((words[8 * q + k] >> j) & 1);
                        v |= jb->lsb ? bit << k : bit << (7 - k);
                    }
                    row[q] = (uint8_t)v;
                }
            }
        }
    }
    free(words);
    return NULL;
}

int mk2o_grain_bulk(const uint8_t *keys, const uint8_t *ivs, uint64_t N, uint64_t T, void *out, int rowmajor, int lsb,
                    int nthreads)
{
    if (rowmajor && (T % 8)) return -2;
    grain_job jb = {keys, ivs, N, T, (N + 31) / 32, (N + 63) / 64, out, rowmajor, lsb, 0};
    if (nthreads < 1) nthreads = mk2o_max_threads();
    if ((uint64_t)nthreads > jb.nb) nthreads = (int)(jb.nb ? jb.nb : 1);
    pthread_t th[1024];
    if (nthreads > 1024) nthreads = 1024;
    int started = 0;
    for (int i = 0; i < nthreads; ++i) {
        if (pthread_create(&th[i], NULL, grain_worker, &jb) != 0) break;
        ++started;
    }
    if (!started) grain_worker(&jb);
    for (int i = 0; i < started; ++i) pthread_join(th[i], NULL);
    return 0;
}
