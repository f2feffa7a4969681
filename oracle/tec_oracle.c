/* oracle/tec_oracle.c -- TEST INFRASTRUCTURE ONLY (see tec_oracle.h).
 *
 * Every loop below follows the reference's evaluation order exactly so that
 * f32 results are bit-identical to evaluate_reference:
 *  - outputs in row-major (n, oc, oh, ow) order        R/src/texpr.cpp:189-199
 *  - per output: facc = 0.0f; odometer over the reduce axes in declaration
 *    order (ic, rh, rw), last axis fastest             R/src/texpr.cpp:205-228
 *    (depthwise drops ic: reduce axes are (rh, rw))    R/src/ops.cpp:138-141
 *  - the body is mul(data, wgt): one float product, then facc = facc + v,
 *    each rounded to float (no FMA; built with -ffp-contract=off)
 *                                                      R/src/expr.cpp:137-145
 *  - padded reads: select(in-bounds, x[clamped], 0)    R/src/ops.cpp:147-155
 *  - integer path: int64 products/sums, i32 range check on store
 *                                                      R/src/expr.cpp:95-127,
 *                                                      R/include/tec/tensor.hpp:63-69
 *  - fused members run one after another, each materialising its full
 *    result (so each epilogue op rounds to float separately)
 *                                                      R/src/graph.cpp:209-222
 * Independent (n, oc) output planes are split over pthreads; each output is
 * still computed by one thread in the reference order, so the thread count
 * never changes a bit of the result.
 */
#include "tec_oracle.h"

#include <pthread.h>
#include <stddef.h>
#include <stdint.h>

enum { ERR_OK = 0, ERR_SHAPE = 2, ERR_OVERFLOW = 3 };

int tec_oracle_out_hw(const tec_oracle_conv* d, int64_t* oh, int64_t* ow) {
  /* R/src/ops.cpp:131-132 and the checks of infer_conv :163-192 */
  if (d->n <= 0 || d->c <= 0 || d->h <= 0 || d->w <= 0 || d->oc <= 0 ||
      d->kh <= 0 || d->kw <= 0 || d->sh <= 0 || d->sw <= 0 || d->ph < 0 ||
      d->pw < 0)
    return ERR_SHAPE;
  if (d->depthwise && d->oc != d->c) return ERR_SHAPE;
  *oh = (d->h + 2 * d->ph - d->kh) / d->sh + 1;
  *ow = (d->w + 2 * d->pw - d->kw) / d->sw + 1;
  if (*oh <= 0 || *ow <= 0) return ERR_SHAPE;
  return ERR_OK;
}

static float relu_f(float x) {
  /* relu = vmax(x, cstf(0)) evaluated with std::max(x, 0.0f)
   * (R/src/ops.cpp:250-258, R/src/expr.cpp:150-152): (x < 0) ? 0 : x */
  return (x < 0.0f) ? 0.0f : x;
}

typedef struct {
  const tec_oracle_conv* d;
  const void* x;
  const void* w;
  const tec_oracle_epi* epi;
  int n_epi;
  void* y;
  int64_t oh, ow;
  int64_t plane_begin, plane_end; /* range over n * oc */
  int is_int;
  int overflow;
} job_t;

static void plane_f32(job_t* j, int64_t n, int64_t oc) {
  const tec_oracle_conv* d = j->d;
  const float* x = (const float*)j->x;
  const float* w = (const float*)j->w;
  float* y = (float*)j->y;
  const int64_t C = d->c, H = d->h, W = d->w, O = d->oc;
  const int64_t KH = d->kh, KW = d->kw;
  const int64_t RC = d->depthwise ? 1 : C;
  const int padded = d->ph != 0 || d->pw != 0;
  for (int64_t oh = 0; oh < j->oh; ++oh) {
    for (int64_t ow = 0; ow < j->ow; ++ow) {
      float facc = 0.0f;
      for (int64_t r = 0; r < RC; ++r) {
        const int64_t ic = d->depthwise ? oc : r;
        for (int64_t rh = 0; rh < KH; ++rh) {
          const int64_t hh = oh * d->sh + rh - d->ph;
          for (int64_t rw = 0; rw < KW; ++rw) {
            const int64_t ww = ow * d->sw + rw - d->pw;
            float data;
            if (!padded || (hh >= 0 && hh < H && ww >= 0 && ww < W))
              data = x[((n * C + ic) * H + hh) * W + ww];
            else
              data = 0.0f;
            const float wgt = d->depthwise
                                  ? w[(oc * KH + rh) * KW + rw]
                                  : w[((oc * C + ic) * KH + rh) * KW + rw];
            const float v = data * wgt;
            facc = facc + v;
          }
        }
      }
      const int64_t o = ((n * O + oc) * j->oh + oh) * j->ow + ow;
      /* Epilogue members, in member order, float rounding per op. */
      for (int e = 0; e < j->n_epi; ++e) {
        switch (j->epi[e].op) {
          case TEC_ORACLE_SCALE:
            facc = facc * (float)j->epi[e].scale;
            break;
          case TEC_ORACLE_BIAS:
            facc = facc + ((const float*)j->epi[e].operand)[oc];
            break;
          case TEC_ORACLE_ADD:
            facc = facc + ((const float*)j->epi[e].operand)[o];
            break;
          case TEC_ORACLE_MUL:
            facc = facc * ((const float*)j->epi[e].operand)[o];
            break;
          case TEC_ORACLE_RELU:
            facc = relu_f(facc);
            break;
        }
      }
      y[o] = facc;
    }
  }
}

static void plane_i8(job_t* j, int64_t n, int64_t oc) {
  const tec_oracle_conv* d = j->d;
  const int8_t* x = (const int8_t*)j->x;
  const int8_t* w = (const int8_t*)j->w;
  int32_t* y = (int32_t*)j->y;
  const int64_t C = d->c, H = d->h, W = d->w, O = d->oc;
  const int64_t KH = d->kh, KW = d->kw;
  const int64_t RC = d->depthwise ? 1 : C;
  for (int64_t oh = 0; oh < j->oh; ++oh) {
    for (int64_t ow = 0; ow < j->ow; ++ow) {
      int64_t iacc = 0;
      for (int64_t r = 0; r < RC; ++r) {
        const int64_t ic = d->depthwise ? oc : r;
        for (int64_t rh = 0; rh < KH; ++rh) {
          const int64_t hh = oh * d->sh + rh - d->ph;
          for (int64_t rw = 0; rw < KW; ++rw) {
            const int64_t ww = ow * d->sw + rw - d->pw;
            int64_t data = 0;
            if (hh >= 0 && hh < H && ww >= 0 && ww < W)
              data = x[((n * C + ic) * H + hh) * W + ww];
            const int64_t wgt = d->depthwise
                                    ? w[(oc * KH + rh) * KW + rw]
                                    : w[((oc * C + ic) * KH + rh) * KW + rw];
            iacc += data * wgt;
          }
        }
      }
      /* set_i range check of the conv result (tensor.hpp:63-69) */
      if (iacc < INT32_MIN || iacc > INT32_MAX) j->overflow = 1;
      const int64_t o = ((n * O + oc) * j->oh + oh) * j->ow + ow;
      for (int e = 0; e < j->n_epi; ++e) {
        switch (j->epi[e].op) {
          case TEC_ORACLE_SCALE:
            iacc = iacc * (int64_t)j->epi[e].scale;
            break;
          case TEC_ORACLE_BIAS:
            iacc = iacc + ((const int32_t*)j->epi[e].operand)[oc];
            break;
          case TEC_ORACLE_ADD:
            iacc = iacc + ((const int32_t*)j->epi[e].operand)[o];
            break;
          case TEC_ORACLE_MUL:
            iacc = iacc * ((const int32_t*)j->epi[e].operand)[o];
            break;
          case TEC_ORACLE_RELU:
            iacc = iacc < 0 ? 0 : iacc;
            break;
        }
        if (iacc < INT32_MIN || iacc > INT32_MAX) j->overflow = 1;
      }
      y[o] = (int32_t)iacc;
    }
  }
}

static void* run_job(void* arg) {
  job_t* j = (job_t*)arg;
  for (int64_t pl = j->plane_begin; pl < j->plane_end; ++pl) {
    const int64_t n = pl / j->d->oc, oc = pl % j->d->oc;
    if (j->is_int)
      plane_i8(j, n, oc);
    else
      plane_f32(j, n, oc);
  }
  return NULL;
}

static int run(const tec_oracle_conv* d, const void* x, const void* w,
               const tec_oracle_epi* epi, int n_epi, void* y, int threads,
               int is_int) {
  int64_t OH, OW;
  int st = tec_oracle_out_hw(d, &OH, &OW);
  if (st) return st;
  if (is_int) {
    for (int e = 0; e < n_epi; ++e) {
      /* "integer scale requires an integral factor" (R/src/ops.cpp:267-270) */
      if (epi[e].op == TEC_ORACLE_SCALE &&
          epi[e].scale != (double)(int64_t)epi[e].scale)
        return ERR_SHAPE;
    }
  }
  const int64_t planes = d->n * d->oc;
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  if (threads > planes) threads = (int)planes;
  job_t jobs[256];
  pthread_t tids[256];
  for (int t = 0; t < threads; ++t) {
    job_t j = {d, x, w, epi, n_epi, y, OH, OW,
               planes * t / threads, planes * (t + 1) / threads, is_int, 0};
    jobs[t] = j;
  }
  for (int t = 1; t < threads; ++t)
    pthread_create(&tids[t], NULL, run_job, &jobs[t]);
  run_job(&jobs[0]);
  int overflow = jobs[0].overflow;
  for (int t = 1; t < threads; ++t) {
    pthread_join(tids[t], NULL);
    overflow |= jobs[t].overflow;
  }
  return overflow ? ERR_OVERFLOW : ERR_OK;
}

int tec_oracle_fused_conv_f32(const tec_oracle_conv* d, const float* x,
                              const float* w, const tec_oracle_epi* epi,
                              int n_epi, float* y, int threads) {
  return run(d, x, w, epi, n_epi, y, threads, 0);
}

int tec_oracle_fused_conv_i8(const tec_oracle_conv* d, const int8_t* x,
                             const int8_t* w, const tec_oracle_epi* epi,
                             int n_epi, int32_t* y, int threads) {
  return run(d, x, w, epi, n_epi, y, threads, 1);
}

/* ---------------------------------------------------------------- pooling
 * New graph operators of the ResNet-18 graph (not in the reference op set;
 * the build defines them, include/tec_sm100.h tec_pool_desc):
 *   max_pool2d: max over the in-image taps of each window (padding taps are
 *     skipped), NCHW, exact.
 *   global_avg_pool: the reference composition
 *     scale(sum(sum(x, axis=3), axis=2), 1/(H*W)):
 *     sum reduces in order from 0 with float rounding (R/src/ops.cpp:111-149,
 *     R/src/texpr.cpp:205-228), scale multiplies by the attr rounded to
 *     float (R/src/ops.cpp:260-281). */
int tec_oracle_max_pool2d_f32(const float* x, int64_t n, int64_t c, int64_t h, int64_t w,
                              int64_t r, int64_t s, int64_t sh, int64_t sw, int64_t ph,
                              int64_t pw, float* y) {
  if (h + 2 * ph < r || w + 2 * pw < s || sh <= 0 || sw <= 0) return ERR_SHAPE;
  const int64_t oh = (h + 2 * ph - r) / sh + 1, ow = (w + 2 * pw - s) / sw + 1;
  for (int64_t p = 0; p < n * c; ++p)
    for (int64_t i = 0; i < oh; ++i)
      for (int64_t j = 0; j < ow; ++j) {
        float best = 0.0f;
        int any = 0;
        for (int64_t a = 0; a < r; ++a) {
          const int64_t ih = i * sh + a - ph;
          if (ih < 0 || ih >= h) continue;
          for (int64_t b = 0; b < s; ++b) {
            const int64_t iw = j * sw + b - pw;
            if (iw < 0 || iw >= w) continue;
            const float v = x[(p * h + ih) * w + iw];
            if (!any || v > best) best = v;
            any = 1;
          }
        }
        y[(p * oh + i) * ow + j] = best;
      }
  return ERR_OK;
}

int tec_oracle_global_avg_pool_f32(const float* x, int64_t n, int64_t c, int64_t h,
                                   int64_t w, float* y) {
  const float f = (float)(1.0 / (double)(h * w));
  for (int64_t p = 0; p < n * c; ++p) {
    float tot = 0.0f;
    for (int64_t i = 0; i < h; ++i) {
      float row = 0.0f;
      for (int64_t j = 0; j < w; ++j) row = row + x[(p * h + i) * w + j];
      tot = tot + row;
    }
    y[p] = tot * f;
  }
  return ERR_OK;
}
