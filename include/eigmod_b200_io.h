/* C ABI of the ingest / egest formats (libeigmod_b200_cxx.so; host code, all
 * threads). Replaces proj/include/eigmod/io.hpp:17-33 for FFI callers:
 *   read_matrix_market / write_matrix_market  (io.cpp:59-131)
 *   read_csv_matrix / write_csv_matrix        (io.cpp:133-194)
 * Same grammar, values and messages; written files are byte-identical to the
 * reference's. Return codes: 0 ok, 3 FormatError (message via
 * eigmod_b200_io_last_error), 4 other failure. Row-major doubles. */
#ifndef EIGMOD_B200_IO_H
#define EIGMOD_B200_IO_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Message of the last failed call on this thread. */
const char* eigmod_b200_io_last_error(void);

/* signs may be NULL (no "# signs:" line). */
int eigmod_b200_io_write_csv(const char* path, const double* m, int64_t rows, int64_t cols,
                             const int* signs, int64_t nsigns);
/* Two-phase read: the file is parsed once and kept per thread; shape3 =
 * (rows, cols, nsigns or -1 without a signs line); then
 * eigmod_b200_io_take_csv copies the values (rows*cols) and signs out. */
int eigmod_b200_io_read_csv(const char* path, int64_t* shape3);
int eigmod_b200_io_take_csv(double* values, int* signs);

int eigmod_b200_io_write_matrix_market(const char* path, const double* a, int64_t n);
/* Two-phase like CSV: n_out, then take the n x n symmetric matrix. */
int eigmod_b200_io_read_matrix_market(const char* path, int64_t* n_out);
int eigmod_b200_io_take_matrix_market(double* a);

#ifdef __cplusplus
}
#endif
#endif
