/* sg_oracle.h -- CPU checker for the B200 M4RM path (test infrastructure only). */
#ifndef SG_ORACLE_H
#define SG_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif
enum { SGO_F2 = 0, SGO_F3 = 1, SGO_F5 = 2, SGO_F7 = 3, SGO_GF4 = 4, SGO_GF8 = 5, SGO_Z4 = 6, SGO_Z8 = 7 };
int sgo_planes(int field);
int sgo_order(int field);
int sgo_pack(int field, const uint8_t* dense, int64_t m, int64_t n, uint64_t* planes);
int sgo_unpack(int field, const uint64_t* planes, int64_t m, int64_t n, uint8_t* dense);
void sgo_canonicalize(int field, uint64_t* planes, int64_t rows, int64_t words);
int sgo_word_op(const char* name, const uint64_t* in, uint64_t* out);
int sgo_m4rm(int field, const uint64_t* A, const uint64_t* B, uint64_t* C, int64_t m,
             int64_t l, int64_t n, int k, int threads, int64_t row0, int64_t row1);
#ifdef __cplusplus
}
#endif
#endif
