/* abi_consumer.c -- a plain C program that uses libmk2.so through include/mk2.h only (no Python, no CUDA headers).
 *
 * What a non-Python host of the reference's MICKEY path would write: the eSTREAM known-answer vector
 * (pkg/src/slicerng/vectors.py:41-47: key 123456789abcdef01234, IV 21436587 -> 9821e10c5ed28d32bbc3d1fb15e93a15)
 * on 70 instances through mk2_init_from_material + mk2_generate_rowmajor with ordinary malloc'ed host buffers,
 * then the same rows from the one-shot mk2_bulk_rowmajor.
 *
 * exit 0: keystream matches; exit 3: no sm_100 device (mk2_create said MK2_E_NODEVICE -- the library has no CPU
 * path, and says so); anything else: failure.  tests/test_host.py builds it with gcc and expects 3 on the CPU box,
 * tests/test_gpu_parity.py expects 0 on the B200.
 */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "mk2.h"

#define N 70
#define T 128 /* keystream bits per instance */

static const uint8_t KEY[10] = {0x12, 0x34, 0x56, 0x78, 0x9a, 0xbc, 0xde, 0xf0, 0x12, 0x34};
static const uint8_t IV[4] = {0x21, 0x43, 0x65, 0x87};
static const uint8_t WANT[16] = {0x98, 0x21, 0xe1, 0x0c, 0x5e, 0xd2, 0x8d, 0x32, 0xbb, 0xc3, 0xd1, 0xfb, 0x15, 0xe9, 0x3a, 0x15};

int main(void)
{
    mk2_ctx *ctx = NULL;
    int rc = mk2_create(0, &ctx);
    if (rc == MK2_E_NODEVICE) {
        fprintf(stderr, "no device: %s\n", mk2_last_error(NULL));
        return 3;
    }
    if (rc != MK2_OK) {
        fprintf(stderr, "mk2_create failed (%d): %s\n", rc, mk2_last_error(NULL));
        return 1;
    }
    uint8_t *keys = malloc(N * 10), *ivs = malloc(N * 4), *rows = malloc(N * (T / 8)), *bulk = malloc(N * (T / 8));
    if (!keys || !ivs || !rows || !bulk) return 1;
    for (int n = 0; n < N; ++n) {
        memcpy(keys + 10 * n, KEY, 10);
        memcpy(ivs + 4 * n, IV, 4);
    }
    if ((rc = mk2_init_from_material(ctx, keys, ivs, 4, 32, N)) != MK2_OK ||
        (rc = mk2_generate_rowmajor(ctx, T, rows, T / 8)) != MK2_OK) {
        fprintf(stderr, "generate failed (%d): %s\n", rc, mk2_last_error(ctx));
        return 1;
    }
    uint64_t sum_two_call = 0, sum_bulk = 0;
    if ((rc = mk2_checksum(ctx, &sum_two_call)) != MK2_OK ||
        (rc = mk2_bulk_rowmajor(ctx, keys, ivs, 4, 32, N, T, bulk, T / 8, &sum_bulk)) != MK2_OK) {
        fprintf(stderr, "bulk failed (%d): %s\n", rc, mk2_last_error(ctx));
        return 1;
    }
    int bad = 0;
    for (int n = 0; n < N; ++n) bad |= memcmp(rows + n * (T / 8), WANT, 16) != 0;
    bad |= memcmp(rows, bulk, N * (T / 8)) != 0 || sum_two_call != sum_bulk;
    /* errors come back as codes, never as a crash */
    bad |= mk2_generate_rowmajor(ctx, 12, rows, 2) != MK2_E_ARG;
    mk2_destroy(ctx);
    free(keys); free(ivs); free(rows); free(bulk);
    printf("%s: %d instances x %d bits, checksum %016llx\n", bad ? "MISMATCH" : "ok", N, T, (unsigned long long)sum_two_call);
    return bad ? 2 : 0;
}
