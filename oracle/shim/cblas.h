/* Declaration-only CBLAS shim (test infrastructure).
 *
 * The reference includes <cblas.h> (/root/reference/proj/src/distances.cpp:3,
 * vectors.cpp:3) but ships no BLAS and pins no version (proj/CMakeLists.txt:5
 * points at an absent vendor/ dir). This header declares the one routine it
 * calls, with the standard CBLAS enum values; the oracle Makefile links the
 * OpenBLAS 0.3.15 build bundled in the image (opencv_python_headless.libs),
 * which exports plain `cblas_sgemm`. */
#ifndef ORACLE_SHIM_CBLAS_H
#define ORACLE_SHIM_CBLAS_H
#ifdef __cplusplus
extern "C" {
#endif
enum CBLAS_ORDER { CblasRowMajor = 101, CblasColMajor = 102 };
enum CBLAS_TRANSPOSE { CblasNoTrans = 111, CblasTrans = 112, CblasConjTrans = 113 };
void cblas_sgemm(enum CBLAS_ORDER order, enum CBLAS_TRANSPOSE ta, enum CBLAS_TRANSPOSE tb, int m, int n, int k,
                 float alpha, const float* a, int lda, const float* b, int ldb, float beta, float* c, int ldc);
#ifdef __cplusplus
}
#endif
#endif
