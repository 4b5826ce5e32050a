#!/bin/bash
# mutation check of the Algorithm-3 oracle pins (tests/test_rpca_pins.py):
# each plausible mistake in oracle/rpca.py must make some pin fail
mkdir -p /tmp/mutr && cd /tmp/mutr
muts=(
's/sig = 1.0 + wz + ww /sig = 1.0 + wz /'
's/Lnew = np.maximum(0.5 \* (Tm - D + X - Snew + A), 0.0)/Lnew = np.maximum(Tm - D + X - Snew + A, 0.0)/'
's/Lnew = np.maximum(0.5 \* (Tm - D + X - Snew + A), 0.0)/Lnew = np.maximum(0.5 * (Tm + D + X - Snew + A), 0.0)/'
's/Dnew = D + Lnew - Tnew /Dnew = D - Lnew + Tnew /'
's/Bnew = Bd + Znew - Snew\[:-1\]/Bnew = Bd - Znew + Snew[:-1]/'
's/Cnew = Cd + Wnew - Snew\[1:\]/Cnew = Cd + Wnew - Snew[:-1]/'
's/centres = np.stack(\[Snew\[:-1\] - Bd, Snew\[1:\] - Cd\], axis=1)/centres = np.stack([Snew[:-1] + Bd, Snew[1:] + Cd], axis=1)/'
's/Tnew = svt(Mmat, gamma \/ rho)/Tnew = svt(Mmat, gamma)/'
's/thr = lam \/ (rho \* sig\[t\])/thr = lam \/ rho/'
's/iterate(centres, mu, rho \/ kappa,/iterate(centres, mu, kappa \/ rho,/'
's/K\[t\] += W\[t - 1\] + Cd\[t - 1\]/K[t] += W[t - 1] - Cd[t - 1]/'
's/Mmat = (Lnew + D)/Mmat = (Lnew - D)/'
's/Xnew = (phi \* Y + rho \* (Snew + Lnew - A)) \/ (phi \* phi + rho)/Xnew = (Y + rho * (Snew + Lnew - A)) \/ (phi * phi + rho)/'
)
for m in "${muts[@]}"; do
  rm -rf w; mkdir w; cp -r /root/repo/oracle /root/repo/tests w/
  sed -i "$m" w/oracle/rpca.py
  if cmp -s w/oracle/rpca.py /root/repo/oracle/rpca.py; then echo "MUTATION DID NOT APPLY: $m"; continue; fi
  (cd w && timeout 900 python -m pytest tests/test_rpca_pins.py -x -q -p no:cacheprovider 2>&1 | tail -1) | sed "s|^|[$m] |" | cut -c1-200
done
# signed split (admm_signed, signed_s_update)
muts2=(
's/    r2 = -u + km - lam_rho/    r2 = u + km - lam_rho/'
's/        Sn = Spn - Smn/        Sn = Spn + Smn/'
's/st.update(Bp=st\["Bp"\] + Zp - Spn\[:-1\], Cp=st\["Cp"\] + Wp - Spn\[1:\],/st.update(Bp=st["Bp"] + Zp - Spn[:-1], Cp=st["Cp"] + Wp - Smn[1:],/'
's/    ip = ((1.0 + m) \* r1 + r2) \/ det /    ip = ((1.0 + m) * r1 - r2) \/ det /'
)
for m in "${muts2[@]}"; do
  rm -rf w; mkdir w; cp -r /root/repo/oracle /root/repo/tests w/
  sed -i "$m" w/oracle/rpca.py
  if cmp -s w/oracle/rpca.py /root/repo/oracle/rpca.py; then echo "MUTATION DID NOT APPLY: $m"; continue; fi
  (cd w && timeout 900 python -m pytest tests/test_rpca_pins.py -x -q -p no:cacheprovider -k SG 2>&1 | tail -1) | sed "s|^|[$m] |" | cut -c1-200
done
