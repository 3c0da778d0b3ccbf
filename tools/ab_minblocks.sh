# A/B: __launch_bounds__(512, MB) for k_solve
for MB in 2 1; do
  sed -i "s/k_solve(const SolveParams P, const Ops ops_in)/k_solve(const SolveParams P, const Ops ops_in)/; s/__launch_bounds__(kSolveThreads, [0-9]) k_solve(/__launch_bounds__(kSolveThreads, $MB) k_solve(/" paper_2404_00270_b200/csrc/solve.cu
  python -m paper_2404_00270_b200.build > /dev/null 2>&1
  timeout 300 python tools/probe.py path20000 c2r c2u c4 c3p c3h --reps 1 | python tools/summ.py "mb=$MB"
done
