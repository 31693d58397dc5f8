/*
 * mk2.h -- C ABI of the B200-native bitsliced MICKEY 2.0 keystream generator.
 *
 * This is the drop-in boundary for ONE path of the reference package
 * `slicerng` (arxiv 1909.04750): bulk MICKEY 2.0 keystream generation.  The
 * reference is pure Python + numba and has no FFI of its own; each entry point
 * below names the reference function (path:line under /root/reference/) whose
 * work it replaces, and INTEGRATION.md shows the ctypes binding a maintainer of
 * the reference would add.  Plain pointers and sizes only; no exceptions, no
 * C++/torch types.  Every function returns 0 on success or a negative
 * MK2_E* code; mk2_last_error() gives the text.  There is NO CPU fallback:
 * without an sm_100 device mk2_create() fails.
 *
 * Geometry: N instances are processed as G = ceil(N/32) groups; one GPU thread
 * owns one group (32 instances, column-major: one 32-bit word per bit of the
 * 100-bit R and S registers -- MickeySliced, pkg/src/slicerng/mickey.py:236).
 * Pointers marked "host or device" are classified with
 * cudaPointerGetAttributes:
 *   device pointers  are used in place (e.g. a torch CUDA tensor's data_ptr());
 *   pinned host      (cudaHostAlloc / cudaHostRegister / mk2_host_alloc /
 *                    torch pin_memory) outputs receive asynchronous D2H copies
 *                    of the device staging tiles directly, at link speed;
 *   pageable host    (malloc, a fresh numpy array) outputs of 64 MiB or more are
 *                    moved by the context's copy lanes (mk2_set_host_threads):
 *                    host threads with their own stream and two page-locked
 *                    slots that each copy sub-chunks (2 or 8 MiB) of the device
 *                    staging tile to a slot and move the previous one into the
 *                    caller's array meanwhile, so several D2H copies are always
 *                    in flight; smaller outputs and pageable inputs (key/IV
 *                    bytes, 20 B per instance) are plain cudaMemcpyAsync calls.
 * Every output call returns with the caller's array complete.
 *
 * Current device: every entry point runs on its context's device and restores
 * the caller's current CUDA device before it returns, so a process that drives
 * other devices (e.g. torch on cuda:0, a context on device 1) is not disturbed.
 *
 * Threading: a context is exclusively owned by one thread at a time
 * (SPEC.md:336-337 gives the reference's engines the same rule); use one
 * context per (thread, device).
 */
#ifndef MK2_H
#define MK2_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct mk2_ctx mk2_ctx;

enum {
    MK2_OK = 0,
    MK2_E_CUDA = -1,     /* a CUDA runtime call failed (text in mk2_last_error) */
    MK2_E_ARG = -2,      /* invalid argument */
    MK2_E_STATE = -3,    /* context not initialised with key/IV material yet */
    MK2_E_NODEVICE = -4, /* no CUDA device / not an sm_100 part */
    MK2_E_NOMEM = -5
};

#define MK2_IV_UNUSED 0xFFu /* mk2_init_ragged: lane stays in the all-zero state */

/* Library / device discovery. */
int mk2_abi_version(void); /* currently 2 */
int mk2_device_count(void);

/* Context = one device, one stream, the state of N instances. */
int mk2_create(int device, mk2_ctx **out);
int mk2_destroy(mk2_ctx *ctx);
/* Launch on the caller's stream (e.g. torch's current stream; NULL/0 is the
 * legacy default stream) instead of the context's own non-blocking stream;
 * mk2_use_own_stream() goes back. */
int mk2_set_stream(mk2_ctx *ctx, void *cuda_stream);
int mk2_use_own_stream(mk2_ctx *ctx);
int mk2_sync(mk2_ctx *ctx);
/* Give scratch memory back to the device: the context keeps its stream-ordered
 * pool (bit-sliced key/IV words, staged inputs) and its host-output staging
 * buffers warm between calls; state, checksum and scheduler arrays stay. */
int mk2_trim(mk2_ctx *ctx);
const char *mk2_last_error(const mk2_ctx *ctx); /* ctx may be NULL: last create error */

/* Shard bookkeeping: this context holds global groups
 * [group_offset, group_offset + G).  Only the checksum weighting uses it. */
int mk2_set_group_offset(mk2_ctx *ctx, uint64_t group_offset);

/*
 * Key/IV load + 100 pre-clocks for N instances with one common IV bit length.
 * Replaces MickeySliced.from_key_ivs, uniform route
 * (pkg/src/slicerng/mickey.py:258-304, word-wide load :291-303).
 *   keys: N x 10 bytes, row-major, bit k_0 = MSB of byte 0 (bitops.py:33-36)
 *   ivs : N rows of iv_stride bytes (>= ceil(iv_bits/8)), MSB-first; may be
 *         NULL when iv_bits == 0
 *   iv_bits: 0..80
 * keys / ivs: host or device.  Lanes N..32*G-1 load zero material, like the
 * reference's unused lanes.
 */
int mk2_init_from_material(mk2_ctx *ctx, const uint8_t *keys, const uint8_t *ivs, uint32_t iv_stride,
                           uint32_t iv_bits, uint64_t N);

/*
 * Same with a per-instance IV bit length (the reference's ragged route,
 * mickey.py:287-289 + from_scalar_states :306-316).  iv_nbits[n] in 0..80, or
 * MK2_IV_UNUSED for a lane that must stay in the all-zero state.
 */
int mk2_init_ragged(mk2_ctx *ctx, const uint8_t *keys, const uint8_t *ivs, uint32_t iv_stride,
                    const uint8_t *iv_nbits, uint64_t N);

/*
 * Synthetic material generated on the device: every instance
 * uses `key`; instance n gets the 80-bit big-endian IV (first_index + n).
 * first_index must be a multiple of 32.  No host->device traffic.
 */
int mk2_init_counter_iv(mk2_ctx *ctx, const uint8_t key[10], uint64_t first_index, uint64_t N);

/*
 * Seed-derived material (pkg/src/slicerng/seedgen.py:57-86, derive_lane_material):
 * AES-128 counter construction under a key derived from the 32-byte master
 * seed; lane n gets key = stream[0:10], iv = stream[10:20].  The reference caps
 * a seed at 64 lanes (seedgen.py:22); here first_lane + N may be up to 2^32
 * (the lane field of the derivation block).  algo_tag (seedgen.py:24-31):
 * 3 = mickey, keys N x 10 and ivs N x 10 bytes; 2 = grain, keys N x 10 and ivs
 * N x 8 bytes (stream[10:18]).  Tag 1 (aes-ctr, 16-byte key + 12-byte nonce) and
 * unknown tags are rejected with MK2_E_ARG: that cipher is not on this library's
 * path.  keys / ivs: host or device.  mk2_init_from_seed derives (tag 3) and
 * initialises in one go without the material ever leaving the device.
 */
int mk2_derive_material(mk2_ctx *ctx, const uint8_t seed[32], uint32_t algo_tag, uint64_t first_lane, uint64_t N,
                        uint8_t *keys, uint8_t *ivs);
int mk2_init_from_seed(mk2_ctx *ctx, const uint8_t seed[32], uint64_t first_lane, uint64_t N);

/*
 * T more keystream clocks, column-major ("bit-interleaved",
 * docs/conventions.md:61-63): out[t * stride_words + g] is a uint32 whose bit j
 * is keystream bit t of instance 32 g + j.  For N = 64 and stride 2 the buffer
 * is byte-identical to the uint64 array kernels.mickey_sliced_words returns
 * (pkg/src/slicerng/kernels.py:189-200).  Replaces the compiled loop
 * kernels._mickey_sliced_loop (kernels.py:46-95) and
 * MickeySliced.keystream_words (mickey.py:362-368); resumable like the latter.
 * out: host or device; stride_words >= G.
 */
int mk2_generate_colmajor(mk2_ctx *ctx, uint64_t T, void *out, uint64_t stride_words);

/*
 * T more keystream clocks (T % 8 == 0, bitops.py:17-18), row-major
 * ("lane-major", docs/conventions.md:58-60): row n = instance n, T/8 bytes,
 * first bit in the MSB of the first byte -- what kernels.words_to_lane_bytes /
 * words_lane_major_bytes (kernels.py:604-621) produce from the words.
 * out points at the first NEW byte of row 0; pitch_bytes is the row stride, so
 * successive calls can fill a longer row chunk by chunk.  out: host or device.
 */
int mk2_generate_rowmajor(mk2_ctx *ctx, uint64_t T, void *out, uint64_t pitch_bytes);
/* The same with the byte packing chosen by the caller: lsb_first != 0 puts the
 * first bit of every byte in its LEAST significant position -- bit_order="lsb"
 * of kernels.words_to_lane_bytes / words_lane_major_bytes (kernels.py:610-611). */
int mk2_generate_rowmajor_order(mk2_ctx *ctx, uint64_t T, void *out, uint64_t pitch_bytes, int lsb_first);

/*
 * n raw CLOCK_KG steps without output: MickeySliced.clock_kg(mixing, word)
 * (pkg/src/slicerng/mickey.py:329-360).  input_words: uint32 [n][G] (bit j of
 * word [c][g] = input bit of instance 32 g + j at step c) or NULL for zero
 * input.  host or device.  Not a throughput path.
 */
int mk2_clock(mk2_ctx *ctx, int mixing, const uint32_t *input_words, uint64_t n);

/*
 * Grain v1, the paper's second bitsliced stream cipher (pkg/src/slicerng/grain.py;
 * compiled loop kernels.py:268-292).  Same context, geometry, layouts, scheduling
 * and checksum as MICKEY; a context holds the state of one cipher at a time.
 *   mk2_grain_init_from_material  = GrainSliced.from_key_ivs (grain.py:250-277):
 *       keys N x 10 bytes, ivs N x 8 bytes, bits LSB-first per byte (grain.py:88-92),
 *       160 init clocks; lanes N..32G-1 are the reference's unused lanes.
 *   mk2_grain_generate_colmajor   = kernels.grain_sliced_words (kernels.py:334-342)
 *   mk2_grain_generate_rowmajor   = lane-major bytes, first bit in the MSB (library
 *       default) or, with lsb_first != 0, in the LSB (the published vectors' order).
 *   mk2_grain_state_export        = uint32 bs[160][G]: NFSR words then LFSR words.
 */
int mk2_grain_init_from_material(mk2_ctx *ctx, const uint8_t *keys, const uint8_t *ivs, uint64_t N);
int mk2_grain_generate_colmajor(mk2_ctx *ctx, uint64_t T, void *out, uint64_t stride_words);
int mk2_grain_generate_rowmajor(mk2_ctx *ctx, uint64_t T, void *out, uint64_t pitch_bytes, int lsb_first);
int mk2_grain_state_export(mk2_ctx *ctx, uint32_t *bs);

/* Number of instances / groups / clocks emitted since init. */
int mk2_query(const mk2_ctx *ctx, uint64_t *N, uint64_t *G, uint64_t *clocks);

/*
 * Raw sliced state, uint32 rs[200][G]: rs[i][g] = R bit i, rs[100+i][g] = S
 * bit i of group g (MickeySliced.rregs/.sregs, mickey.py:250-251).  Import
 * also (re)sizes the context to N instances and clears the checksum.
 * rs: host or device.
 */
int mk2_state_export(mk2_ctx *ctx, uint32_t *rs);
int mk2_state_import(mk2_ctx *ctx, const uint32_t *rs, uint64_t N);

/*
 * Checksum of everything emitted since init: the column-major stream read as
 * little-endian uint64 words (group g + group_offset even = low half) and
 * summed mod 2^64.  Layout independent; additive over disjoint group ranges,
 * so per-GPU values can be combined with one 8-byte ncclSum all-reduce.
 */
int mk2_checksum(mk2_ctx *ctx, uint64_t *sum);

/* Device time (ms, CUDA events on the launch stream) of the kernels launched by
 * the most recent init / generate call, and how many kernels that was. */
float mk2_last_kernel_ms(const mk2_ctx *ctx);
int mk2_last_kernel_launches(const mk2_ctx *ctx);
/* Skip the per-call event synchronisation (for callers that time the stream
 * themselves); mk2_last_kernel_ms is then only valid after mk2_sync. */
int mk2_set_async(mk2_ctx *ctx, int async);

/*
 * One-shot bulk generation, row-major: key/IV load + pre-clocks + T keystream bits
 * of N instances in one call -- kernels.mickey_sliced_words (kernels.py:189-200)
 * followed by words_lane_major_bytes (kernels.py:615-621) in the reference, for
 * any N.  Arguments as mk2_init_from_material / mk2_generate_rowmajor; keys and
 * ivs must both be host or both be device pointers.  With host buffers the
 * instances are processed in blocks (2 x 8 x SMs x 1024) and the upload of block
 * b+1, the init + keystream of block b and the download of block b-1 overlap on
 * three streams.  *checksum (optional) receives what mk2_checksum would return for
 * the whole call.  When N spans more than one block the context holds no
 * resumable state afterwards (mk2_init_* again before mk2_generate_*).
 */
int mk2_bulk_rowmajor(mk2_ctx *ctx, const uint8_t *keys, const uint8_t *ivs, uint32_t iv_stride, uint32_t iv_bits,
                      uint64_t N, uint64_t T, void *out, uint64_t pitch_bytes, uint64_t *checksum);

/* Tuning knob: clocks per scheduling chunk of the persistent keystream kernels
 * (0 = automatic, else >= 128): a chain of 1024 instances runs one chunk, parks
 * its state and goes back to the ready queue.
 * mk2_last_plan reports what the most recent keystream launch used. */
int mk2_set_chunk_clocks(mk2_ctx *ctx, uint32_t clocks);
/* Tuning knob: size of one device staging tile for HOST output buffers (two are
 * in flight: one being generated, one being copied out).  0 = default (32 MiB;
 * row-major tiles, which are 2-D copies, are 16x this). */
int mk2_set_stage_bytes(mk2_ctx *ctx, uint64_t bytes);
/* Number of copy lanes (host threads) that move staging tiles into PAGEABLE
 * output arrays; 0 = automatic (one per hardware thread, 2..16; contiguous
 * column-major tiles use at most 8 of them). */
int mk2_set_host_threads(mk2_ctx *ctx, int threads);
/* Pinned (page-locked, portable) host memory for output arrays that should take
 * the direct D2H path: what the Python front end's fresh result arrays are made
 * of (kernels.py:194-200 returns a fresh array per call; here it comes from a
 * cached pinned pool).  mk2_last_error(NULL) has the text after a failure. */
int mk2_host_alloc(size_t bytes, void **out);
int mk2_host_free(void *p);
/* Tuning knob: where the row-major kernel parks 256 keystream words per thread
 * between two drains: 1 = shared memory (seven worker warps per SM fit),
 * 2 = tensor memory (tcgen05.st / tcgen05.ld; eight fit), 0 = automatic
 * (tensor memory).  Grain v1: 0 and 1 = 256-clock tiles in shared memory;
 * 2 = the experimental 512-clock tiles split between tensor and shared memory
 * (64 contiguous bytes per row and drain; slower overall);
 * 3 = the same 512-clock tiles in global scratch meant to stay in L2 (74 MB;
 * measured: it does not stay, 7.2 Tb/s against 10.4 -- kept as a documented
 * negative result); 4 = the lone-warp experiments: row-major with four warps
 * per SM, in-register bit transposes and the drain of a tile riding on the
 * generation of the next one through a three-block ring (full 256-clock
 * tiles, whole groups of 32 instances and 32-byte aligned rows only, other
 * shapes fall back to 0; 10.5-10.6 Tb/s against 10.6-10.7), and column-major
 * on an 80-word circular buffer with no realignment moves (T a multiple of
 * 16; 12.3 Tb/s against 13.8: the 56 KB loop body is instruction-fetch
 * bound); 5 = row-major with EIGHT warps per SM, 28 of a tile's 32 groups in
 * shared and 4 in tensor memory (whole chains of 1024 instances, full tiles
 * and 32-byte aligned rows only, other shapes fall back to 0; 10.6-10.8 Tb/s
 * against 11.4: with eight warps the open row lines no longer fit L2).
 * Modes 3, 4 and 5 on a MICKEY context behave like 0. */
int mk2_set_row_staging(mk2_ctx *ctx, int mode);
/* Tuning knob: mk2_bulk_rowmajor with key/IV arrays AND output on the device can
 * run as one kernel (csrc/mk2_fused.cuh: records -> input words in tensor memory ->
 * load clocks -> pre-clocks -> keystream -> rows; neither the bitsliced material
 * nor the state passes through HBM) when the IV length is a whole number of bytes,
 * IV records are 10 bytes apart and both arrays are 16-byte aligned.
 *   mode 1 (default): for init-dominated calls, T <= 1024 bits per instance
 *          (BASELINE config 5); longer calls run pack + init + the persistent
 *          keystream kernel over the whole batch, which is quicker there;
 *   mode 2: whenever eligible;   mode 0: never (A/B, tests). */
int mk2_set_bulk_fused(mk2_ctx *ctx, int mode);
/* Tuning knob: small batches (up to 2048 groups = 65536 instances; the reference's
 * own calling unit is 64 lanes, kernels.py:189-200, cli.py:219-231) are initialised
 * and clocked column-major by warp-per-group kernels (csrc/mk2_coop.cuh: the 200
 * state bits of a group spread over the lanes of a warp, neighbours and taps by
 * shuffle), which cut the latency of a call several times.  enable = 0 forces the
 * thread-per-group throughput kernels (A/B, tests).  Same state layout either way. */
int mk2_set_small_batch(mk2_ctx *ctx, int enable);
int mk2_last_plan(const mk2_ctx *ctx, int *block_threads, uint32_t *chunk_clocks);

/* Diagnostics: per-job trace of the column-major persistent kernel.  Records
 * are 48-byte structs {u32 chain, k, smid, warp; u64 t_pop, t_start, t_end
 * (ns, %globaltimer); u64 pad}.  capacity 0 switches tracing off.
 * mk2_read_trace copies out and clears the records gathered so far.
 * mk2_set_max_ctas caps the number of persistent CTAs (0 = no cap). */
int mk2_set_trace(mk2_ctx *ctx, uint64_t capacity);
int mk2_read_trace(mk2_ctx *ctx, void *records, uint64_t max_records, uint64_t *count);
int mk2_set_max_ctas(mk2_ctx *ctx, uint32_t ctas);

/* Tuning knob: threads per persistent CTA of the keystream kernels (0 =
 * automatic; else 32..256 in steps of 32; one CTA per SM, 255 registers per
 * thread, so 128 = one worker warp per SM sub-partition, 256 = two). */
int mk2_set_block_threads(mk2_ctx *ctx, int threads);

/*
 * Roofline probe: sustained LOP3 lane-operations per second of this device,
 * measured with a dependency-free LOP3 kernel.
 */
int mk2_lop3_peak(mk2_ctx *ctx, double *lane_ops_per_s, float *ms);

/* Static facts about the kernels (for DESIGN.md / bench.py): ALU-pipe logic ops
 * per keystream clock per 32-lane word as counted in SURVEY.md 8(d). */
int mk2_lop3_per_clock(void);
/* The kernels run the clock in blocks of mk2_rblock(kernel) clocks with R's
 * feedback reduction deferred to the end of the block (csrc/mk2_clock.cuh);
 * mk2_lop3_per_block(kernel) is the number of LOP3 a keystream block executes,
 * so mk2_lop3_per_block / mk2_rblock < mk2_lop3_per_clock.
 * kernel: 0 = column-major keystream, 1 = row-major keystream, 2 = key/IV load + pre-clock. */
#define MK2_KERNEL_COLMAJOR 0
#define MK2_KERNEL_ROWMAJOR 1
#define MK2_KERNEL_INIT 2
int mk2_rblock(int kernel);
int mk2_lop3_per_block(int kernel);

#ifdef __cplusplus
}
#endif
#endif /* MK2_H */
