/* C-ABI known answer, no Python: hom_nand of two reference ciphertexts through
 * libfhegpu.so must equal the reference's result (tests/golden/kat_default_nand.bin, made from
 * the reference-generated scheme_default.npz).  Also exercises hom_not twice (identity).
 * usage: abi_kat <fixture>   exit 0 = pass */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "../../include/fhegpu.h"

int main(int argc, char **argv) {
  if (argc < 2) return 2;
  FILE *f = fopen(argv[1], "rb");
  if (!f) return 2;
  uint32_t hdr[5];
  if (fread(hdr, 4, 5, f) != 5) return 2;
  const uint32_t words = hdr[4];
  uint32_t *buf = malloc(sizeof(uint32_t) * 3 * words), *out = malloc(sizeof(uint32_t) * words),
           *not1 = malloc(sizeof(uint32_t) * words), *not2 = malloc(sizeof(uint32_t) * words);
  if (fread(buf, 4, 3 * words, f) != 3 * words) return 2;
  fclose(f);
  fhegpu_params p = {hdr[0], hdr[1], hdr[2], hdr[3]};
  fhegpu_ctx *ctx = NULL;
  if (fhegpu_ctx_create(&p, 0, &ctx) != FHEGPU_OK) {
    fprintf(stderr, "ctx_create: %s\n", fhegpu_last_error());
    return 1;
  }
  int rc = fhegpu_nand_batch(ctx, buf, buf + words, out, 1);
  rc |= fhegpu_not_batch(ctx, out, not1, 1);
  rc |= fhegpu_not_batch(ctx, not1, not2, 1);
  if (rc != FHEGPU_OK) {
    fprintf(stderr, "call failed: %s\n", fhegpu_last_error());
    return 1;
  }
  const int nand_ok = memcmp(out, buf + 2 * words, 4 * words) == 0;
  const int not_ok = memcmp(not2, out, 4 * words) == 0 && memcmp(not1, out, 4 * words) != 0;
  printf("%s kernel=%d nand %s, not(not(x)) %s\n", fhegpu_version(), fhegpu_ctx_kernel(ctx),
         nand_ok ? "== reference" : "DIFFERS", not_ok ? "== x" : "WRONG");
  fhegpu_ctx_destroy(ctx);
  return nand_ok && not_ok ? 0 : 1;
}
