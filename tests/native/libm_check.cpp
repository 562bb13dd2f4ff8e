// Host build of the device scalar math (csrc/tabx_math.cuh) for CPU tests:
// reads float64 arguments from argv[2], writes mode-dependent results to argv[3].
//   mode "sincos": (sin, cos) per argument
//   mode "pairwise": argv[4] = row length n; one pairwise sum per row
//   mode "remainder": argv[4] = divisor; np.remainder per argument
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <vector>
#include "tabx_math.cuh"

int main(int argc, char** argv) {
  if (argc < 4) return 2;
  FILE* f = fopen(argv[2], "rb");
  FILE* g = fopen(argv[3], "wb");
  if (!f || !g) return 3;
  std::vector<double> xs;
  double x;
  while (fread(&x, 8, 1, f) == 1) xs.push_back(x);
  if (!strcmp(argv[1], "sincos")) {
    for (double v : xs) {
      double s = tabx::libm_sin(v), c = tabx::libm_cos(v);
      fwrite(&s, 8, 1, g);
      fwrite(&c, 8, 1, g);
    }
  } else if (!strcmp(argv[1], "sincos2")) {
    for (double v : xs) {
      const tabx::sincos_t r = tabx::libm_sincos(v);
      fwrite(&r.s, 8, 1, g);
      fwrite(&r.c, 8, 1, g);
    }
  } else if (!strcmp(argv[1], "pairwise")) {
    int n = atoi(argv[4]);
    for (size_t r = 0; r + n <= xs.size(); r += n) {
      double s = tabx::pairwise_sum(xs.data() + r, n);
      fwrite(&s, 8, 1, g);
    }
  } else if (!strcmp(argv[1], "remainder")) {
    double d = atof(argv[4]);
    for (double v : xs) {
      double m = tabx::np_remainder(v, d);
      fwrite(&m, 8, 1, g);
    }
  } else {
    return 4;
  }
  fclose(f);
  fclose(g);
  return 0;
}
