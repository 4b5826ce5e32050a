#!/bin/bash
# mutation check of the oracle pins: each mutation must make some pin fail
mkdir -p /tmp/mut && cd /tmp/mut
muts=(
's/double bb = 2.0 \* Knew\[o + k\] - Kold\[o + k\];/double bb = Knew[o + k];/'
's/an\[o + k\] = a\[o + k\] + tau2 \* bb;/an[o + k] = a[o + k] - tau2 * bb;/'
's/gy\[k\] = (j < ny - 1) ? a\[k\] - a\[k + (size_t)nx\] : 0.0;/gy[k] = (j < ny - 1) ? a[k + (size_t)nx] - a[k] : 0.0;/'
's/for (size_t k = 0; k < N; ++k) gx\[o + k\] = r\[o + k\] + tau1 \* a\[o + k\];/for (size_t k = 0; k < N; ++k) gx[o + k] = r[o + k] - tau1 * a[o + k];/'
's/Knew\[o + k\] = dv\[o + k\] - rn\[o + k\] - x1\[k\] + x0\[k\];/Knew[o + k] = dv[o + k] + rn[o + k] - x1[k] + x0[k];/'
's/double ATa = (a_s ? a_s\[k\] : 0.0) - (a_sm ? a_sm\[k\] : 0.0);/double ATa = (a_sm ? a_sm[k] : 0.0) - (a_s ? a_s[k] : 0.0);/'
's/(MYv(my, nx, ny, i, j) - MYv(my, nx, ny, i, j - 1));/(MYv(my, nx, ny, i, j) - MYv(my, nx, ny, i - 1, j));/'
's/double s = (nrm > sigma) ? (nrm - sigma) \/ nrm : 0.0;/double s = (nrm > sigma) ? (nrm - sigma) : 0.0;/'
's/uot_ref_shrink_l1((int64_t)N, gx + o, alpha \* tau1, rn + o);/uot_ref_shrink_l1((int64_t)N, gx + o, alpha, rn + o);/'
's/rn\[o + k\] = gx\[o + k\] \/ (1.0 + 2.0 \* alpha \* tau1);/rn[o + k] = gx[o + k] \/ (1.0 + alpha * tau1);/'
's/if (s == 0 \&\& prm->fix_first) {/if (s == 1 \&\& prm->fix_first) {/'
's/double v = 0.5 \* (x\[k\] + a\[k\] + z\[k\] + b\[k\]);/double v = x[k] + a[k];/'
's/xn\[k\] = (y\[k\] + prm->rho \* (s\[k\] - a\[k\])) \/ (1.0 + prm->rho);/xn[k] = (y[k] + prm->rho * (s[k] + a[k])) \/ (1.0 + prm->rho);/'
's/s2 += Knew\[o + k\] \* Knew\[o + k\];/s2 += Kold[o + k] * Kold[o + k];/'
's/s3 += dmx \* dmx + dmy \* dmy + dr \* dr;/s3 += dmx * dmx + dmy * dmy;/'
's/s3 += dx \* dx;/s3 += 0.0 * dx;/'
's/res\[2 \* it + 1\] = prm->rho \* sqrt(du);/res[2 * it + 1] = sqrt(du);/'
's/pr += (xn\[q\] - s\[q\]) \* (xn\[q\] - s\[q\])/pr += (x[q] - s[q]) * (x[q] - s[q])/'
)
for m in "${muts[@]}"; do
  rm -rf w; mkdir w; cp -r /root/repo/oracle /root/repo/tests /root/repo/paper_1909_00149_b200 w/; rm -f w/oracle/liboracle.so
  sed -i "$m" w/oracle/uot_oracle.c
  if cmp -s w/oracle/uot_oracle.c /root/repo/oracle/uot_oracle.c; then echo "MUTATION DID NOT APPLY: $m"; continue; fi
  (cd w && timeout 600 python -m pytest tests/test_oracle_pins.py tests/test_oracle_residual_pins.py -x -q -p no:cacheprovider 2>&1 | tail -1) | sed "s|^|[$m] |" | cut -c1-220
done
