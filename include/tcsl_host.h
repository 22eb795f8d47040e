/* tcsl_host.h — C entry points of the C++ drop-in host library (libtcsl.so) for
 * bindings that cannot call C++ (ctypes, cgo, JNI). Status: 0 ok, else
 * tcsl::Errc ordinal + 1 (proj/include/tcsl/errors.hpp:10-22). */
#ifndef TCSL_HOST_H
#define TCSL_HOST_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* gen_random_sparse (proj/src/matrix.cpp:35-67), bit for bit, into a caller
 * buffer of rows*cols binary16 bit patterns (row-major). */
int tcsl_host_gen_random_sparse(int rows, int cols, double beta, uint64_t seed, uint16_t* out);

#ifdef __cplusplus
}
#endif
#endif /* TCSL_HOST_H */
