for i in 1 2; do for v in 1 0; do echo "== TOPK_GRID=$v"; SFFTB_TOPK_GRID=$v python tools/rep_cfg.py config5 config3; done; done
