/*
 * A C host for the B200 path, no Python involved: read a mesh + charges,
 * build the device problem with the reference's default rules
 * (hobi_create_default), solve (hobi_solve: RHS + GMRES + energy) and print
 * the result.  This is what a C/C++ (or cgo / JNI) integrator links against.
 *
 *   cc -std=c99 -I include examples/c_solve.c -L paper_1301_5914_b200 -lhobi \
 *      -Wl,-rpath,$PWD/paper_1301_5914_b200 -o c_solve
 *   ./c_solve problem.bin
 *
 * problem.bin (native endian): int64 nv, nf, nc; double eps1, eps2, kappa;
 * double vertices[3nv], normals[3nv]; int64 faces[3nf]; double qpos[3nc], q[nc].
 * Output: "iterations matvecs residual energy" with the energy as an exact
 * hexadecimal double.
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "hobi.h"

static void* read_n(FILE* f, size_t bytes) {
  void* p = malloc(bytes ? bytes : 1);
  if (!p || fread(p, 1, bytes, f) != bytes) {
    fprintf(stderr, "c_solve: truncated input\n");
    exit(2);
  }
  return p;
}

int main(int argc, char** argv) {
  if (argc != 2) {
    fprintf(stderr, "usage: %s problem.bin\n", argv[0]);
    return 2;
  }
  FILE* f = fopen(argv[1], "rb");
  if (!f) {
    perror(argv[1]);
    return 2;
  }
  int64_t* sizes = (int64_t*)read_n(f, 3 * sizeof(int64_t));
  const int64_t nv = sizes[0], nf = sizes[1], nc = sizes[2];
  double* phys = (double*)read_n(f, 3 * sizeof(double));
  double* v = (double*)read_n(f, 3 * nv * sizeof(double));
  double* n = (double*)read_n(f, 3 * nv * sizeof(double));
  int64_t* faces = (int64_t*)read_n(f, 3 * nf * sizeof(int64_t));
  double* qpos = (double*)read_n(f, 3 * nc * sizeof(double));
  double* q = (double*)read_n(f, nc * sizeof(double));
  fclose(f);

  hobi_ctx* ctx = NULL;
  if (hobi_create_default(0, v, n, nv, faces, nf, phys[0], phys[1], phys[2], 4, &ctx) != HOBI_OK) {
    fprintf(stderr, "c_solve: %s\n", hobi_last_error());
    return 1;
  }
  double* phi = (double*)malloc(nv * sizeof(double));
  double* dphi = (double*)malloc(nv * sizeof(double));
  double energy = 0.0, residual = 0.0;
  int iterations = 0, matvecs = 0;
  /* SolverConfig defaults: tolerance 1e-6, restart 100, max_iterations 1000 */
  int st = hobi_solve(ctx, qpos, q, nc, 1e-6, 100, 1000, phi, dphi, &energy, &iterations, &residual, &matvecs);
  if (st != HOBI_OK) {
    fprintf(stderr, "c_solve: %s\n", hobi_last_error());
    hobi_destroy(ctx);
    return 1;
  }
  printf("%d %d %.17g %a\n", iterations, matvecs, residual, energy);
  hobi_destroy(ctx);
  free(sizes); free(phys); free(v); free(n); free(faces); free(qpos); free(q); free(phi); free(dphi);
  return 0;
}
