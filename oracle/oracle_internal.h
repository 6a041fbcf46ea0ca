/* oracle_internal.h -- private structures of the oracle (TEST INFRASTRUCTURE ONLY). */
#ifndef ORACLE_INTERNAL_H
#define ORACLE_INTERNAL_H
#include "oracle.h"

enum { FACE_W = 0, FACE_E = 1, FACE_S = 2, FACE_N = 3 };   /* canonical stencil order */

struct face {
    int present;     /* face exists (not beyond the domain) */
    double c;        /* coupling on the face */
    int64_t g;       /* grid index of the neighbour cell */
    int64_t q;       /* unknown index of the neighbour, -1 if land */
};

struct orc_problem {
    int32_t ni, nj, periodic;
    double *cE, *cN;         /* copies of the inputs, [nj][ni] */
    uint8_t* mask;
    int64_t n, nnz;
    int64_t* unk_of;         /* grid -> unknown (-1 land) */
    int64_t* grid_of;        /* unknown -> grid */
    double* sigma;           /* per unknown */
    int64_t *rowptr, *col;   /* CSR of A, columns ascending */
    double *val, *diag;
};

struct orc_ainv {
    int64_t n, nnz;
    int64_t *colptr, *row;   /* Zhat in CSC, rows ascending within a column */
    double *zhat, *z;        /* unit-diagonal factor and z_kj = fl(s_k zhat_kj) */
    double *p, *s;           /* pivots (Dhat) and Jacobi scale s = 1/sqrt(A_pp) */
    /* row-wise copy of Z (CSR of Z, columns ascending) for s = Z t */
    int64_t *rptr, *rcol;
    double* rval;
};

void orc_faces(const orc_problem* P, int32_t i, int32_t j, struct face f[4]);

#endif
