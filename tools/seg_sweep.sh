# z-segment A/B (dev): BP1 p-sweep at 10M DOFs and BP3 at 50M for a few HEXBP_SEG_WAVES values
for w in 0 1 2 4; do echo "== waves $w"; HEXBP_SEG_WAVES=$w timeout 300 python tools/sweep_time.py --bp 1 --ps 1,2,3,4,5,6,7,8 --dofs 1e7 2>&1 | grep p=; done
for w in 0 2; do echo "== bp3 waves $w"; HEXBP_SEG_WAVES=$w timeout 300 python tools/sweep_time.py --ps 2,3,4,5,6,8 --dofs 5e7 2>&1 | grep p=; done
