/* Declaration-only stand-in for <gmp.h>, written for this repo.
 *
 * TEST INFRASTRUCTURE ONLY. The image ships GMP 6.3's runtime
 * (libgmp.so.10) but not its development header. The reference's
 * bigcount.hpp includes <gmp.h>; this file declares exactly the subset of
 * GMP's public, documented ABI that the reference uses so that the
 * reference sources under /root/reference/proj/src compile unmodified into
 * oracle/_ref/.  It is never included by the product.
 */
#ifndef PBB_ORACLE_GMP_SHIM_H
#define PBB_ORACLE_GMP_SHIM_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int _mp_alloc;
  int _mp_size;
  unsigned long* _mp_d;
} __mpz_struct;
typedef __mpz_struct mpz_t[1];
typedef __mpz_struct* mpz_ptr;
typedef const __mpz_struct* mpz_srcptr;

void __gmpz_init(mpz_ptr);
void __gmpz_init_set(mpz_ptr, mpz_srcptr);
void __gmpz_clear(mpz_ptr);
void __gmpz_set(mpz_ptr, mpz_srcptr);
void __gmpz_swap(mpz_ptr, mpz_ptr);
void __gmpz_add(mpz_ptr, mpz_srcptr, mpz_srcptr);
void __gmpz_sub(mpz_ptr, mpz_srcptr, mpz_srcptr);
void __gmpz_mul(mpz_ptr, mpz_srcptr, mpz_srcptr);
void __gmpz_fdiv_q(mpz_ptr, mpz_srcptr, mpz_srcptr);
unsigned long __gmpz_fdiv_q_ui(mpz_ptr, mpz_srcptr, unsigned long);
void __gmpz_fdiv_q_2exp(mpz_ptr, mpz_srcptr, unsigned long);
int __gmpz_cmp(mpz_srcptr, mpz_srcptr);
size_t __gmpz_sizeinbase(mpz_srcptr, int);
void* __gmpz_export(void*, size_t*, int, size_t, int, size_t, mpz_srcptr);
void __gmpz_import(mpz_ptr, size_t, int, size_t, int, size_t, const void*);
char* __gmpz_get_str(char*, int, mpz_srcptr);
int __gmpz_set_str(mpz_ptr, const char*, int);
void __gmpz_fac_ui(mpz_ptr, unsigned long);
void __gmp_get_memory_functions(void* (**)(size_t), void* (**)(void*, size_t, size_t),
                                void (**)(void*, size_t));

#define mpz_init __gmpz_init
#define mpz_init_set __gmpz_init_set
#define mpz_clear __gmpz_clear
#define mpz_set __gmpz_set
#define mpz_swap __gmpz_swap
#define mpz_add __gmpz_add
#define mpz_sub __gmpz_sub
#define mpz_mul __gmpz_mul
#define mpz_fdiv_q __gmpz_fdiv_q
#define mpz_fdiv_q_ui __gmpz_fdiv_q_ui
#define mpz_fdiv_q_2exp __gmpz_fdiv_q_2exp
#define mpz_cmp __gmpz_cmp
#define mpz_sizeinbase __gmpz_sizeinbase
#define mpz_export __gmpz_export
#define mpz_import __gmpz_import
#define mpz_get_str __gmpz_get_str
#define mpz_set_str __gmpz_set_str
#define mpz_fac_ui __gmpz_fac_ui
#define mp_get_memory_functions __gmp_get_memory_functions
#define mpz_sgn(Z) ((Z)->_mp_size < 0 ? -1 : (Z)->_mp_size > 0)

#ifdef __cplusplus
}
#endif

#endif
