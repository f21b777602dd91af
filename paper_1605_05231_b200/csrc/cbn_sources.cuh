// Node generators of the projector, evaluated per point on the device in
// float64 with the reference's operation order (no FMA contraction):
//
//  * RadialSrc   -- radial-line lattice nodes  (radon_fourier.py:59-72,
//                   geometry.py:162-168), node order rho fastest, then theta,
//                   then phi; wrapped twice as the reference does
//                   (_wrap_nodes, then plan_nufft's wrap_nodes).
//  * UmbrellaSrc -- one umbrella plane per target (geometry.py:190-217),
//                   canonical polar wrap twice (geometry.py:143-159), the
//                   |rho| validity mask and origin pinning
//                   (pipeline.py:96-102), fractional lattice indices with the
//                   +rho_max fold (resampling.py:38-59), the rho padding and
//                   node = -2 pi pos / padded (resampling.py:97-101).
//                   Output axis order is the device grid order (phi, theta, rho).
//  * PolarSrc    -- Grangeat detector-plane polar nodes (grangeat.py:110-117).
#pragma once

#include "cbn_common.cuh"

namespace cbn {

struct RadialSrc {
    const double* om;     // n_rho   radial_omega(spec) * voxel (rad / voxel)
    const double* cphi;   // n_phi
    const double* sphi;
    const double* cth;    // n_theta
    const double* sth;
    int n_rho, n_theta;
    struct Aux {
        double raw[3];    // unwrapped node (for the trilinear transfer)
        double wc[3];     // wrapped once: the centre phase's node (radon_fourier.py:102,106)
        int ir, it;
    };
    CBN_D void node(int64_t i, double (&w)[3], Aux& a) const {
        const int ir = (int)(i % n_rho);
        const int64_t rest = i / n_rho;
        const int it = (int)(rest % n_theta);
        const int ip = (int)(rest / n_theta);
        const double st = sth[it];
        const double o = om[ir];
        a.raw[0] = dmul(o, dmul(cphi[ip], st));
        a.raw[1] = dmul(o, dmul(sphi[ip], st));
        a.raw[2] = dmul(o, cth[it]);
        a.ir = ir;
        a.it = it;
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            a.wc[d] = wrap_pi(a.raw[d]);
            w[d] = wrap_pi(a.wc[d]);      // plan_nufft wraps again (nufft.py:150)
        }
    }
};

// The radial lattice of a real volume is Hermitian: the node at rho index
// n_rho - k is the mirror (-w) of the node at k, and its value is the
// conjugate -- up to rounding whenever both of its node representatives (once-
// and twice-wrapped) are the negations of the partner's and the taps mirror
// (same support after the reference's exact edge test).  That fails at wrap
// ties (a component at an odd multiple of pi, where the reference's wrapping
// is not odd) and where u - J/2 is an integer on one side only.  RadialPairSrc enumerates a plan-time list
// of primary nodes: idx >= 0 -> node idx, whose mirror is written as the
// conjugate; idx < 0 -> node ~idx on its own (k = 0, k = n_rho/2, tie pairs).
struct RadialPairSrc {
    RadialSrc base;
    const int* idx;
    using Aux = RadialSrc::Aux;
    CBN_D void node(int64_t i, double (&w)[3], Aux& a) const {
        const int f = idx[i];
        base.node(f >= 0 ? f : ~f, w, a);
    }
};

// RadialPairSrc after the bin sort: the sorted order holds the packed entries
// themselves (f or ~f), so the gather decodes its index argument directly
struct RadialPackedSrc {
    RadialSrc base;
    using Aux = RadialSrc::Aux;
    CBN_D void node(int64_t i, double (&w)[3], Aux& a) const { base.node(i >= 0 ? i : ~i, w, a); }
};

// plan step: for every line and rho index 0..n/2, the primary entry; a
// lower-half node whose mirror is not exactly its negation is entered
// without mirroring and its mirror is appended (counter `extra`)
__global__ void k_radial_pairs(RadialSrc r, KBSet kb, int J, int64_t lines, int* __restrict__ idx,
                               int* __restrict__ extra, int64_t base_count,
                               int64_t line0 = 0);
// perm[k] = idx[perm[k]] (in place): a bin order over RadialPairSrc -> packed entries
__global__ void k_gather_index(const int* __restrict__ idx, int64_t n, int* __restrict__ perm);

// Centre phase x plan phase of the reference, each on its own node
// representative: the centre phase uses the once-wrapped node, the plan phase
// the twice-wrapped one; a node at +pi can wrap to -pi the second time, and
// for even N the two representatives give opposite signs, so the product is
// not a function of one node value.  Returns the angle of
//   exp(+i wc.(N/2 - 1/2)) * exp(-i wp.(N//2))   (centre * plan phase);
// the adjoint uses its negative.
template <int D>
CBN_D double centre_plan_angle(const double (&wc)[D], const double (&wp)[D], const int (&N)[D]) {
    double a = 0.0;
#pragma unroll
    for (int d = 0; d < D; ++d)
        a += wc[d] * ((double)N[d] / 2.0 - 0.5) - wp[d] * (double)(N[d] / 2);
    return a;
}

struct UmbrellaGeom {
    const double* cos_a;   // per view: cos / sin of the source angle
    const double* sin_a;
    const double* cos_mu;  // per umbrella line angle
    const double* sin_mu;
    double so, dt;
    int n_mu, n_t;
    // radial spec and resample padding
    double rho_max, d_rho;
    int n_rho, n_theta, n_phi;
    int pad;
    double padded[3];      // reference order (rho, theta, phi)
    int n_views;
};

// canonical_polar (geometry.py:143-159)
CBN_D void canonical(double& rho, double& theta, double& phi) {
    const double st = sin(theta);
    double nx = dmul(cos(phi), st);
    double ny = dmul(sin(phi), st);
    double nz = cos(theta);
    if (nz < 0.0) {
        nx = -nx;
        ny = -ny;
        nz = -nz;
        rho = -rho;
    }
    double th = acos(fmin(fmax(nz, -1.0), 1.0));
    double ph = np_mod(atan2(ny, nx), kTwoPi);
    theta = th >= kPi ? 0.0 : th;
    phi = ph;
}

struct UmbrellaSrc {
    UmbrellaGeom g;
    int view0;
    // Optional base-view cache: positions (rho, theta, phi, valid) of view 0's
    // targets.  Rotating the source by 2 pi k / V rotates every umbrella
    // plane normal about z, leaving rho and theta unchanged and adding
    // k n_phi / V to the phi index (mod n_phi), so view k's targets follow
    // from view 0's without the per-target trigonometry.
    //
    // The pole (theta exactly 0: the mu = pi/2, t = 0 plane of every view) is
    // the exception: the reference's canonical wrap sets its phi from the
    // signs of zero components (0 or pi per view, geometry.py:143-159), not
    // by the rotation, so pole targets are always computed directly.  (The
    // lattice rows at theta = 0 coincide for every phi, so the two choices
    // differ only at the level of the J = 3 interpolation error.)
    const double4* cache = nullptr;
    struct Aux {
        bool valid;
        bool pole;     // valid target at theta == 0 (phi from the view's own geometry)
    };
    CBN_D void cached_position(int64_t i, double (&pos)[3], bool& valid) const {
        const int64_t per_view = (int64_t)g.n_mu * g.n_t;
        const int v = view0 + (int)(i / per_view);
        const double4 c = cache[i % per_view];
        valid = c.w != 0.0;
        pos[0] = c.x;
        pos[1] = c.y;
        const double shift = ddiv(dmul((double)v, (double)g.n_phi), (double)g.n_views);
        pos[2] = valid ? np_mod(dadd(c.z, shift), (double)g.n_phi) : c.z;
    }
    // fractional lattice indices (rho incl. padding, theta, phi), reference order
    CBN_D void position(int64_t i, double (&pos)[3], bool& valid) const {
        if (cache) {
            cached_position(i, pos, valid);
            if (!(valid && pos[1] == 0.0)) return;
        }
        const int64_t per_view = (int64_t)g.n_mu * g.n_t;
        const int v = view0 + (int)(i / per_view);
        const int rem = (int)(i % per_view);
        const int im = rem / g.n_t;
        const int jt = rem % g.n_t;
        const double ca = g.cos_a[v], sa = g.sin_a[v];
        const double cm = g.cos_mu[im], sm = g.sin_mu[im];
        const double t = dmul((double)(jt - g.n_t / 2), g.dt);
        // s = SO (cos a, sin a, 0); u_hat = (-sin a, cos a, 0); v_hat = (0, 0, 1)
        const double sx = dmul(g.so, ca), sy = dmul(g.so, sa), sz = dmul(g.so, 0.0);
        const double ux = -sa, uy = ca, uz = 0.0;
        // e = cos mu u_hat + sin mu v_hat ; d = -sin mu u_hat + cos mu v_hat
        const double ex = dadd(dmul(cm, ux), dmul(sm, 0.0));
        const double ey = dadd(dmul(cm, uy), dmul(sm, 0.0));
        const double ez = dadd(dmul(cm, uz), dmul(sm, 1.0));
        const double msm = -sm;
        const double dx = dadd(dmul(msm, ux), dmul(cm, 0.0));
        const double dy = dadd(dmul(msm, uy), dmul(cm, 0.0));
        const double dz = dadd(dmul(msm, uz), dmul(cm, 1.0));
        // a = p0 - s ; n = a x d ; n /= |n|
        const double ax = dsub(dmul(t, ex), sx);
        const double ay = dsub(dmul(t, ey), sy);
        const double az = dsub(dmul(t, ez), sz);
        double nx = dsub(dmul(ay, dz), dmul(az, dy));
        double ny = dsub(dmul(az, dx), dmul(ax, dz));
        double nz = dsub(dmul(ax, dy), dmul(ay, dx));
        const double nn = sqrt(dadd(dadd(dmul(nx, nx), dmul(ny, ny)), dmul(nz, nz)));
        nx = ddiv(nx, nn);
        ny = ddiv(ny, nn);
        nz = ddiv(nz, nn);
        double rho = dadd(dadd(dmul(nx, sx), dmul(ny, sy)), dmul(nz, sz));
        double theta = acos(fmin(fmax(nz, -1.0), 1.0));
        double phi = np_mod(atan2(ny, nx), kTwoPi);
        canonical(rho, theta, phi);
        valid = fabs(rho) <= g.rho_max * (1.0 + 1e-12);
        if (!valid) {
            rho = 0.0;
            theta = 0.0;
            phi = 0.0;
        }
        canonical(rho, theta, phi);   // polar_index_map wraps again
        double ir = dadd(ddiv(rho, g.d_rho), (double)g.n_rho / 2.0);
        double it = ddiv(dmul(theta, (double)g.n_theta), kPi);
        double ip = ddiv(dmul(phi, (double)g.n_phi), kTwoPi);
        if (ir >= (double)g.n_rho - 1e-9) {
            ir = 0.0;
            it = np_mod(dsub((double)g.n_theta, it), (double)g.n_theta);
            ip = np_mod(dadd(ip, (double)g.n_phi / 2.0), (double)g.n_phi);
        }
        pos[0] = dadd(ir, (double)g.pad);
        pos[1] = it;
        pos[2] = ip;
    }
    CBN_D void node(int64_t i, double (&w)[3], Aux& a) const {
        double pos[3];
        position(i, pos, a.valid);
        a.pole = a.valid && pos[1] == 0.0;
        const double m2pi = -kTwoPi;
        // device axis order: (phi, theta, rho)
        w[0] = wrap_pi(ddiv(dmul(m2pi, pos[2]), g.padded[2]));
        w[1] = wrap_pi(ddiv(dmul(m2pi, pos[1]), g.padded[1]));
        w[2] = wrap_pi(ddiv(dmul(m2pi, pos[0]), g.padded[0]));
    }
};

struct PolarSrc {
    const double* omega;   // n_t  rad / mm
    const double* cos_mu;  // n_mu
    const double* sin_mu;
    double pu, pv;
    int n_t;
    struct Aux {
        int jt;
        double wc[2];     // wrapped once: the centre phase's node (grangeat.py:117-119)
    };
    CBN_D void node(int64_t i, double (&w)[2], Aux& a) const {
        const int im = (int)(i / n_t);
        a.jt = (int)(i % n_t);
        const double o = omega[a.jt];
        a.wc[0] = wrap_pi(dmul(dmul(o, cos_mu[im]), pu));
        a.wc[1] = wrap_pi(dmul(dmul(o, sin_mu[im]), pv));
        w[0] = wrap_pi(a.wc[0]);
        w[1] = wrap_pi(a.wc[1]);
    }
};

}  // namespace cbn
