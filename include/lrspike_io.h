/* Matrix Market ingestion and the reorder pipeline as a C-ABI (liblrspike.so), for FFI
 * callers such as paper_2504_11167_b200/reorder.py.  Host-side structural preprocessing:
 * SPEC.md:39-47 (read_matrix_market), SPEC.md:96-133 (strip_disconnected,
 * diagonal_scale, rcm_ordering, apply_permutation).  The C++ API is
 * include/lrspike/reorder.hpp.  Status codes are lrs_status (lrspike_capi.h). */
#ifndef LRSPIKE_IO_H
#define LRSPIKE_IO_H

#include <stdint.h>

#include "lrspike_capi.h"

#ifdef __cplusplus
extern "C" {
#endif

/* A host CSR (0-based, int64 indices).  Outputs are malloc'd: release with lrs_io_free. */
typedef struct lrs_csr_host {
  int64_t n_rows, n_cols, nnz;
  int64_t* row_ptr;
  int64_t* col_idx;
  double* values;
} lrs_csr_host;

typedef struct lrs_io_error {
  char message[512];
  int64_t line; /* ParseError payload */
  int64_t row;  /* SingularScalingError payload */
} lrs_io_error;

LRS_API int32_t lrs_io_read_mm(const char* path, lrs_csr_host* out);
LRS_API int32_t lrs_io_write_mm(const char* path, const lrs_csr_host* a);
LRS_API void lrs_io_free(lrs_csr_host* a);
/* forward[old] = new (n entries) */
LRS_API int32_t lrs_reorder_rcm(const lrs_csr_host* a, int64_t* forward);
/* removed: capacity n_rows; *n_removed entries written */
LRS_API int32_t lrs_reorder_strip(const lrs_csr_host* a, lrs_csr_host* out, int64_t* removed,
                                  int64_t* n_removed);
/* scale: n entries, D = diag(|a_ii|^-1/2), out = D A D */
LRS_API int32_t lrs_reorder_scale(const lrs_csr_host* a, lrs_csr_host* out, double* scale);
LRS_API int32_t lrs_reorder_permute(const lrs_csr_host* a, const int64_t* row_forward,
                                    const int64_t* col_forward, lrs_csr_host* out);
LRS_API int32_t lrs_io_last_error(lrs_io_error* out);

#ifdef __cplusplus
}
#endif

#endif /* LRSPIKE_IO_H */
