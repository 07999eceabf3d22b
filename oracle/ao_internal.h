/* ao_internal.h — shared helpers of the CPU oracle (test infrastructure). */
#ifndef AO_INTERNAL_H
#define AO_INTERNAL_H
#include <stddef.h>

void ao_matmul(int m, int k, int n, const double* a, const double* b, double* c);
void ao_matmul_bt(int m, int k, int n, const double* a, const double* b, double* c);
void ao_matmul_at(int m, int k, int n, const double* a, const double* b, double* c);
void ao_matvec(int m, int n, const double* a, const double* x, double* y);
void ao_matvec_t(int m, int n, const double* a, const double* x, double* y);
void ao_transpose(int m, int n, const double* a, double* at);
void ao_symm(int n, double* a);
int ao_all_zero(int n, const double* a);
void ao_eye(int n, double* a);
void ao_sandwich(int m, int n, const double* a, const double* p, double* out, double* work);

/* broadcast accessors (lgssm.hpp:34-40) */
#define AO_F(m, t) ((m)->F + (size_t)((m)->nF > 1 ? (t) : 0) * (m)->dx * (m)->dx)
#define AO_B(m, t) ((m)->b + (size_t)((m)->nb > 1 ? (t) : 0) * (m)->dx)
#define AO_Q(m, t) ((m)->Q + (size_t)((m)->nQ > 1 ? (t) : 0) * (m)->dx * (m)->dx)
#define AO_H(m, t) ((m)->H + (size_t)((m)->nH > 1 ? (t) : 0) * (m)->dy * (m)->dx)
#define AO_C(m, t) ((m)->c + (size_t)((m)->nc > 1 ? (t) : 0) * (m)->dy)
#define AO_R(m, t) ((m)->R + (size_t)((m)->nR > 1 ? (t) : 0) * (m)->dy * (m)->dy)
#define AO_OBSERVED(m, t) ((m)->mask == NULL || (m)->mask[t] != 0)

#endif
