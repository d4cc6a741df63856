/*
 * TEST INFRASTRUCTURE ONLY — CPU oracle for the gridloc belief-filter hot
 * path. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg
 * may load this library, and only as the checker. The product
 * (paper_1910_00572_b200, libgridloc_b200.so) never links or calls it.
 *
 * Parity pinning: this restatement is checked bit-for-bit against the
 * UNMODIFIED reference compiled from /root/reference (oracle/_ref, see
 * oracle/Makefile) and against the known-answer tests of
 * proj/tests/test_belief_engine.cpp and proj/tests/test_observation.cpp
 * (ported in tests/test_oracle_*.py).
 *
 * Layout is the reference's: belief [k][j][i] FP64, idx k*W*H + j*W + i
 * (belief_tensor.hpp:55-60); occupancy uint8 row-major, 1 = occupied
 * (occupancy_map.hpp:50-54,79).
 */
#ifndef GL_ORACLE_H
#define GL_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  GLO_OK = 0,
  GLO_EXTINGUISHED = 1, /* BeliefExtinguishedError */
  GLO_INVALID = 2,      /* std::invalid_argument */
  GLO_MAP_PARSE = 3,    /* MapParseError */
};

/* KernelSet (belief_tensor.hpp:79-89), flattened. */
typedef struct {
  int channels;
  int radius;
  int separable;
  int degenerate_spatial;
  int degenerate_angular;
  double sep[64];      /* 2r+1 taps when separable */
  double* spatial;     /* channels * (2r+1)^2, owned */
  int n_ang;
  int ang_off[4096];
  double ang_w[4096];
} glo_kernels;

int glo_build_kernels(double sigma_x, double sigma_y, double sigma_theta,
                      int channels, double cell, double delta_theta,
                      glo_kernels* out);
void glo_kernels_free(glo_kernels* k);

void glo_motion_vector(double u, double v, int k, double theta_t,
                       double delta_theta, double cell, double* dx,
                       double* dy);

/* Activation::values / inverse, each channels*W*H. */
void glo_make_activation(const uint8_t* occ, int w, int h,
                         const glo_kernels* ks, double* values,
                         double* inverse);

int glo_init_uniform(const uint8_t* occ, int w, int h, int channels,
                     double* out);

/* One Algorithm-1 step in place; *theta_t advances by w. Returns
 * GLO_EXTINGUISHED (tensor and theta_t already updated) like the reference. */
int glo_step(double* belief, int w, int h, int channels, double cell,
             double* theta_t, double u, double v, double dw,
             const uint8_t* occ, const glo_kernels* ks,
             const double* inverse);

/* glo_step with the wall-crossing mask (wall_mask != 0): an EXTENSION the
 * reference does not have (it masks destinations only,
 * belief_tensor.cpp:414-416): a bilinear tap is dropped when the open segment
 * between its source and destination cell centres crosses the interior of
 * an occupied cell. Parity for this mode is against this restatement of the
 * rule only (no reference behaviour exists to pin it to). */
int glo_step_wall(double* belief, int w, int h, int channels, double cell,
                  double* theta_t, double u, double v, double dw,
                  const uint8_t* occ, const glo_kernels* ks,
                  const double* inverse, int wall_mask);
/* cells crossed by the tap offset (ox, oy), relative to the destination;
 * returns the full count, stores at most cap */
int glo_seg_cells(int ox, int oy, int* qx, int* qy, int cap);

void glo_apply_motion(double* belief, int w, int h, int channels, double cell,
                      double* theta_t, double u, double v, double dw);

void glo_belief_map(const double* belief, int w, int h, int channels,
                    double* out);

int glo_argmax(const double* belief, int w, int h, int channels, double cell,
               double ox, double oy, double theta_t, int* ijk, double* pose,
               double* confidence);

/* cells: (i, j) pairs in emission order, at most cap pairs written. */
int glo_dither(const double* bm, int w, int h, int budget, int* cells,
               int cap, int* n, double* source_mass);

void glo_distance_field(const uint8_t* occ, int w, int h, double res,
                        double* out);

int glo_scan_likelihood(const uint8_t* occ, const double* field, int w, int h,
                        double res, double ox, double oy, double px, double py,
                        double pth, const double* angles, const double* ranges,
                        int nb, double max_range, double sigma_hit,
                        double weight_floor, int beam_stride, double* out);

int glo_observation_update(double* belief, int w, int h, int channels,
                           double cell, double ox, double oy, double theta_t,
                           const int* cells, int n, const double* angles,
                           const double* ranges, int nb, double max_range,
                           const uint8_t* occ, const double* field,
                           double sigma_hit, double weight_floor,
                           int beam_stride);

/* load_map: PGM P2/P5 decode + threshold + forced boundary ring. Writes the
 * dims first (call with occ == NULL to size), then the cells. */
int glo_load_map(const uint8_t* bytes, size_t n, int threshold, int* w, int* h,
                 uint8_t* occ);

#ifdef __cplusplus
}
#endif

#endif
